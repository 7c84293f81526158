// Cost of page-locking an ordinary (pageable, already touched) host buffer for the duration
// of one call: cudaHostRegister + cudaHostUnregister against the buffer size, next to a
// plain pageable H2D and a pinned H2D (development microbenchmark).
// Usage: ./register_cost [MB ...]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  CK(cudaFree(nullptr));
  for (int a = 1; a < (argc > 1 ? argc : 2); ++a) {
    const size_t mb = argc > 1 ? atoll(argv[a]) : 256, bytes = mb << 20;
    char* h = static_cast<char*>(aligned_alloc(4096, bytes));
    memset(h, 1, bytes);
    char* d;
    CK(cudaMalloc(&d, bytes));
    for (int rep = 0; rep < 3; ++rep) {
      double t0 = now_ms();
      CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
      const double pg = now_ms() - t0;
      t0 = now_ms();
      CK(cudaHostRegister(h, bytes, cudaHostRegisterDefault));
      const double reg = now_ms() - t0;
      t0 = now_ms();
      CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
      const double pin = now_ms() - t0;
      t0 = now_ms();
      CK(cudaHostUnregister(h));
      const double unreg = now_ms() - t0;
      printf("%zu MB: pageable H2D %.1f ms (%.1f GB/s) | register %.1f ms (%.1f GB/s) + pinned H2D %.1f ms "
             "(%.1f GB/s) + unregister %.1f ms\n",
             mb, pg, bytes / pg / 1e6, reg, bytes / reg / 1e6, pin, bytes / pin / 1e6, unreg);
    }
    CK(cudaFree(d));
    free(h);
  }
  return 0;
}
