// Packed-lower unpack on the host pool (see host_pool.hpp).
#include "host_pool.hpp"

#include "common.hpp"

namespace hsdla_b200 {

void unpack_lower(const double2* pk, double2* full, uint64_t n, uint64_t c0, uint64_t c1) {
  const uint64_t b0 = packed_col(n, c0);
  unpack_range(pk + b0, full, n, b0, packed_col(n, c1));
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

void unpack_range(const double2* src, double2* full, uint64_t n, uint64_t b0, uint64_t b1) {
  if (b1 <= b0) return;
  HostPool& pool = HostPool::get();
  const uint64_t total = b1 - b0;
  const unsigned nt = total < (1u << 18) ? 1u : pool.width();
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
  });
}

}  // namespace hsdla_b200
