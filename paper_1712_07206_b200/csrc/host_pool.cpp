// Packed-lower unpack on the host pool (see host_pool.hpp).
#include "host_pool.hpp"

#include "common.hpp"

namespace hsdla_b200 {

void unpack_lower(const double2* pk, double2* full, uint64_t n, uint64_t c0, uint64_t c1) {
  const uint64_t b0 = packed_col(n, c0);
  unpack_range(pk + b0, full, n, b0, packed_col(n, c1), false);
}

// Column holding global packed index b (packed_col(n, j) <= b < packed_col(n, j + 1)).
static uint64_t column_of(uint64_t n, uint64_t b) {
  uint64_t lo = 0, hi = n;  // invariant: packed_col(lo) <= b < packed_col(hi)
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    if (packed_col(n, mid) <= b)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// After the unpack has read a span of the pinned D2H stage, optionally push those lines out
// of the reading cores' private caches (cldemote: to the shared L3).  The next call's DMA
// writes into the stage, and lines still held in core L2s cost the PCIe writes a snoop
// each: with a 16 MB stage (C1) an 8 MB D2H ran at 6-8 GB/s instead of 55 and a pinned C1
// call took 2.7 ms instead of 1.3 (tools/small_probe.py).  A stage larger than the cores'
// L2s evicts itself, and the demote (~20 ns a line) then only costs: the caller decides.
static bool has_cldemote() {
#if HSDLA_B200_NT_STORES
  static const bool yes = [] {
    unsigned a = 0, b = 0, c = 0, d = 0;
    __asm__ volatile("cpuid" : "=a"(a), "=b"(b), "=c"(c), "=d"(d) : "a"(7), "c"(0));
    return ((c >> 25) & 1) != 0;
  }();
  return yes;
#else
  return false;
#endif
}
static void demote_lines(const void* p, size_t bytes) {
#if HSDLA_B200_NT_STORES
  const char* c = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(63));
  const char* end = static_cast<const char*>(p) + bytes;
  for (; c < end; c += 64) __asm__ volatile("cldemote %0" ::"m"(*c));
#else
  (void)p, (void)bytes;
#endif
}

void unpack_range(const double2* src, double2* full, uint64_t n, uint64_t b0, uint64_t b1, bool release) {
  if (b1 <= b0) return;
  HostPool& pool = HostPool::get();
  const uint64_t total = b1 - b0;
  // >= 256 KB per thread (a pool wake-up costs ~10-20 us)
  const unsigned nt = static_cast<unsigned>(std::min<uint64_t>(pool.width(), std::max<uint64_t>(1, total >> 14)));
  const bool demote = release && has_cldemote();
  pool.run(nt, [&](uint64_t t) {
    uint64_t p = b0 + total * t / nt;
    const uint64_t pe = b0 + total * (t + 1) / nt;
    if (p >= pe) return;
    uint64_t j = column_of(n, p);
    while (p < pe) {
      const uint64_t cb = packed_col(n, j), ce = packed_col(n, j + 1);
      const uint64_t e = std::min(pe, ce);
      // packed index p of column j is element (j + p - cb, j)
      copy_nt(full + j * n + j + (p - cb), src + (p - b0), (e - p) * sizeof(double2));
      p = e;
      ++j;
    }
    _mm_sfence();
    const uint64_t q0 = b0 + total * t / nt;
    if (demote) demote_lines(src + (q0 - b0), (pe - q0) * sizeof(double2));
  });
}

}  // namespace hsdla_b200
