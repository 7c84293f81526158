// Packed-lower (device) -> column-major lower triangle (pinned host) download, three ways
// (development microbenchmark):
//   (1) one contiguous D2H of the packed triangle + host unpack on 16 threads (the
//       drop-in's path);
//   (2) a gather kernel that writes the columns straight into the mapped pinned
//       destination over PCIe (zero-copy);
//   (3) one cudaMemcpyAsync per column into the destination.
// Usage: ./batch_d2h [n]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

static size_t pcol(size_t n, size_t j) { return j * (2 * n - j + 1) / 2; }

// one block per column j: rows j..n-1 of the packed column -> full + j*n + j
__global__ void gather_lower(const double2* __restrict__ pk, double2* full, size_t n, size_t c0) {
  const size_t j = c0 + blockIdx.x;
  const size_t base = j * (2 * n - j + 1) / 2, len = n - j;
  for (size_t i = threadIdx.x; i < len; i += blockDim.x) full[j * n + j + i] = pk[base + i];
}

// a DMMA-bound kernel (~1 ms) to time alone and next to a concurrent D2H
__global__ void busy(double* out, int iters) {
  double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7, c[8][2] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? atoll(argv[1]) : 3000, npk = n * (n + 1) / 2;
  char *dpk, *hpk, *hfull;
  CK(cudaMalloc(&dpk, npk * 16));
  CK(cudaMallocHost(&hpk, npk * 16));
  CK(cudaHostAlloc(&hfull, n * n * 16, cudaHostAllocMapped));
  void* dfull = nullptr;
  CK(cudaHostGetDevicePointer(&dfull, hfull, 0));
  CK(cudaMemset(dpk, 1, npk * 16));
  memset(hfull, 0, n * n * 16);
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  {
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    double* junk;
    CK(cudaMalloc(&junk, 4096 * 8));
    for (int mode = 0; mode < 4; ++mode) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, s));
      busy<<<148, 256, 0, s>>>(junk, 4000);
      CK(cudaEventRecord(e1, s));
      if (mode == 1) CK(cudaMemcpyAsync(hpk, dpk, 8 << 20, cudaMemcpyDeviceToHost, s2));        // 8 MB D2H, pinned
      if (mode == 2) CK(cudaMemcpyAsync(hpk, dpk, npk * 16, cudaMemcpyDeviceToHost, s2));       // whole packed D2H
      if (mode == 3) CK(cudaMemcpyAsync(dpk, hpk, npk * 16, cudaMemcpyHostToDevice, s2));       // H2D
      CK(cudaEventSynchronize(e1));
      CK(cudaDeviceSynchronize());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("busy kernel %s: %.3f ms\n", mode == 0 ? "alone" : mode == 1 ? "+ 8 MB D2H" : mode == 2 ? "+ packed D2H" : "+ packed H2D", ms);
    }
    // the drop-in's pattern: kernel 1; D2H (copy stream, after kernel 1) overlapping kernel 2;
    // the host waits for the D2H and unpacks it on 16 threads while kernel 2 runs
    cudaEvent_t k1, dd, e2a, e2b;
    CK(cudaEventCreate(&k1)); CK(cudaEventCreate(&dd)); CK(cudaEventCreate(&e2a)); CK(cudaEventCreate(&e2b));
    for (int mode = 0; mode < 6; ++mode) {
      CK(cudaDeviceSynchronize());
      busy<<<148, 256, 0, s>>>(junk, 1000);
      CK(cudaEventRecord(k1, s));
      CK(cudaEventRecord(e2a, s));
      busy<<<148, 256, 0, s>>>(junk, 4000);
      CK(cudaEventRecord(e2b, s));
      if (mode % 3 >= 1) {
        CK(cudaStreamWaitEvent(s2, k1, 0));
        CK(cudaMemcpyAsync(hpk, dpk, 8 << 20, cudaMemcpyDeviceToHost, s2));
        CK(cudaEventRecord(dd, s2));
      }
      if (mode % 3 == 2) {
        CK(cudaEventSynchronize(dd));
        std::vector<std::thread> th;
        for (int t = 0; t < 16; ++t)
          th.emplace_back([&, t] { memcpy(hfull + t * (1 << 20), hpk + t * (512 << 10), 512 << 10); });
        for (auto& x : th) x.join();
      }
      CK(cudaEventSynchronize(e2b));
      float ms;
      CK(cudaEventElapsedTime(&ms, e2a, e2b));
      printf("kernel 2 %s: %.3f ms\n", mode % 3 == 0 ? "alone" : mode % 3 == 1 ? "+ dependent D2H" : "+ D2H + host unpack", ms);
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0, s));
    CK(cudaMemcpyAsync(hpk, dpk, npk * 16, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms1;
    CK(cudaEventElapsedTime(&ms1, e0, e1));
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    const int T = 16;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (size_t j = t; j < n; j += T) memcpy(hfull + (j * n + j) * 16, hpk + pcol(n, j) * 16, (n - j) * 16);
      });
    for (auto& x : th) x.join();
    const double unpack = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();

    CK(cudaEventRecord(e0, s));
    gather_lower<<<static_cast<unsigned>(n), 256, 0, s>>>(reinterpret_cast<const double2*>(dpk),
                                                          static_cast<double2*>(dfull), n, 0);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms2;
    CK(cudaEventElapsedTime(&ms2, e0, e1));

    auto t1 = std::chrono::steady_clock::now();
    CK(cudaEventRecord(e0, s));
    for (size_t j = 0; j < n; ++j)
      CK(cudaMemcpyAsync(hfull + (j * n + j) * 16, dpk + pcol(n, j) * 16, (n - j) * 16, cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(e1, s));
    const double enq = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
    CK(cudaEventSynchronize(e1));
    float ms3;
    CK(cudaEventElapsedTime(&ms3, e0, e1));
    printf("n %zu (%.0f MB packed): D2H %.2f ms (%.1f GB/s) + unpack %.2f ms (%.1f GB/s, 16 thr) | zero-copy gather "
           "%.2f ms (%.1f GB/s) | %zu x cudaMemcpyAsync %.2f ms (%.1f GB/s), enqueue %.2f ms\n",
           n, npk * 16 / 1e6, ms1, npk * 16 / ms1 / 1e6, unpack, npk * 16 / unpack / 1e6, ms2, npk * 16 / ms2 / 1e6, n,
           ms3, npk * 16 / ms3 / 1e6, enq);
  }
  return 0;
}
