// Host-side data movement of the drop-in: a persistent worker pool, streaming-store
// copies, and the packed-lower -> full-matrix unpack (all CPU-side byte movement; no
// arithmetic on H or S happens on the host).
#pragma once

#if defined(__x86_64__) || defined(__i386__)
#include <immintrin.h>
#define HSDLA_B200_NT_STORES 1
#else  // other hosts (e.g. Grace): plain copies, no fence needed
#define HSDLA_B200_NT_STORES 0
static inline void _mm_sfence() {}
#endif

#include <vector_types.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace hsdla_b200 {

// ---------------------------------------------------------------------------
// Host worker pool for the host-side data movement (packing pageable inputs into
// pinned slabs, unpacking packed triangles, page-cache reads): persistent threads,
// so a 64 MB slab does not pay ~16 thread creations.  run(n, f) executes f(0..n-1)
// on the workers and the calling thread and returns when all are done; calls from
// different host threads are serialised.
// ---------------------------------------------------------------------------
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  unsigned width() const { return static_cast<unsigned>(workers_.size()) + 1; }
  void run(uint64_t n, const std::function<void(uint64_t)>& f) {
    if (n == 0) return;
    if (n == 1 || workers_.empty()) {
      for (uint64_t i = 0; i < n; ++i) f(i);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);
    Job job;
    job.f = &f;
    job.n = n;
    {
      std::lock_guard<std::mutex> lk(mu_);
      cur_ = &job;
      job.users = 1;  // the caller
      ++gen_;
    }
    cv_.notify_all();
    process(job);
    std::unique_lock<std::mutex> lk(mu_);
    // the job lives on this stack frame: return only once no worker can touch it
    done_cv_.wait(lk, [&] { return job.done == job.n && job.users == 0; });
    cur_ = nullptr;
  }

 private:
  struct Job {
    const std::function<void(uint64_t)>* f = nullptr;
    uint64_t n = 0, done = 0;
    std::atomic<uint64_t> next{0};
    int users = 0;
  };
  HostPool() {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (unsigned t = 1; t < hw; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // Claim and run items of `job`; the caller of process() is one of job.users.
  void process(Job& job) {
    uint64_t d = 0;
    for (uint64_t i = job.next.fetch_add(1); i < job.n; i = job.next.fetch_add(1)) {
      (*job.f)(i);
      ++d;
    }
    std::lock_guard<std::mutex> lk(mu_);
    job.done += d;
    --job.users;
    if (job.done == job.n && job.users == 0) done_cv_.notify_all();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      Job* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && cur_ != nullptr); });
        if (stop_) return;
        seen = gen_;
        job = cur_;
        ++job->users;
      }
      process(*job);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  Job* cur_ = nullptr;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Host copy with non-temporal (streaming) stores: the destination lines are written without
// being read first (no read-for-ownership), so a pack into a pinned slab costs read +
// write of the bytes instead of read + read + write -- the host memory bandwidth the
// concurrent DMA also needs.  Callers fence (sfence) before publishing the data.
inline void copy_nt(void* dst, const void* src, size_t bytes) {
#if !HSDLA_B200_NT_STORES
  std::memcpy(dst, src, bytes);
#else
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  // head: up to the next 16-byte boundary of the destination
  const size_t head = std::min(bytes, (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
  std::memcpy(d, s, head);
  d += head;
  s += head;
  bytes -= head;
  size_t n = bytes / 16;
  __m128i* dv = reinterpret_cast<__m128i*>(d);
  const __m128i* sv = reinterpret_cast<const __m128i*>(s);
  for (; n >= 4; n -= 4, dv += 4, sv += 4) {
    const __m128i a = _mm_loadu_si128(sv), b = _mm_loadu_si128(sv + 1), c = _mm_loadu_si128(sv + 2),
                  e = _mm_loadu_si128(sv + 3);
    _mm_stream_si128(dv, a);
    _mm_stream_si128(dv + 1, b);
    _mm_stream_si128(dv + 2, c);
    _mm_stream_si128(dv + 3, e);
  }
  for (; n; --n, ++dv, ++sv) _mm_stream_si128(dv, _mm_loadu_si128(sv));
  std::memcpy(dv, sv, bytes & 15);
#endif
}

// fn(i) for i in [0, n), in `parts` contiguous ranges on the host pool when the work
// is large (>= 1 MB; >= 256 KB per part), else inline.
template <class F>
void par_for(uint64_t n, uint64_t bytes, F&& fn) {
  HostPool& pool = HostPool::get();
  const uint64_t parts = bytes < (size_t(1) << 20) ? 1 : std::min<uint64_t>({pool.width(), n, bytes >> 18});
  if (parts <= 1) {
    for (uint64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  pool.run(parts, [&](uint64_t t) {
    for (uint64_t i = n * t / parts; i < n * (t + 1) / parts; ++i) fn(i);
    _mm_sfence();  // streaming stores (copy_nt) visible before the job completes
  });
}

// Unpack columns [c0, c1) of a column-major packed lower triangle (pk = the whole
// packed array) into the lower triangle of an n x n matrix, over up to 16 threads
// with equal element counts.
void unpack_lower(const double2* pk, double2* full, uint64_t n, uint64_t c0, uint64_t c1);

// Unpack the global packed-lower index range [b0, b1) (it may start and end inside a
// column) into the lower triangle of the n x n column-major matrix `full`; src holds
// exactly those b1 - b0 elements.  Threads split the range by element count.  release:
// demote the source lines from the cores' private caches afterwards (host_pool.cpp).
void unpack_range(const double2* src, double2* full, uint64_t n, uint64_t b0, uint64_t b1, bool release);

}  // namespace hsdla_b200
