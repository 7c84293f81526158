// Does FP64 DADD work steal DMMA (mma.sync m8n8k4 f64) throughput on B200?
// Each warp issues 24 independent DMMAs per iteration (the 3M consumer's step) plus
// D FP64 adds (the 3M operand sums), or the same count of FP32 / integer adds.
// Usage: ./dmma_mix  -> one line per variant: DMMA TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int D, int KIND>  // KIND 0: f64 add, 1: f32 add, 2: int add
__global__ void __launch_bounds__(256) k_mix(double* out, int iters) {
  double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7;
  double c[24][2];
#pragma unroll
  for (int i = 0; i < 24; ++i) { c[i][0] = 0; c[i][1] = i; }
  double x[D > 0 ? D : 1];
  float xf[D > 0 ? D : 1];
  long long xi[D > 0 ? D : 1];
#pragma unroll
  for (int i = 0; i < (D > 0 ? D : 1); ++i) { x[i] = i; xf[i] = i; xi[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 24; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      if (i % 4 == 0) {
#pragma unroll
        for (int d = (i / 4) * D / 6; d < (i / 4 + 1) * D / 6; ++d) {
          if (KIND == 0) asm volatile("add.f64 %0, %0, %1;" : "+d"(x[d]) : "d"(a));
          if (KIND == 1) asm volatile("add.f32 %0, %0, %1;" : "+f"(xf[d]) : "f"(1.5f));
          if (KIND == 2) asm volatile("add.s64 %0, %0, %1;" : "+l"(xi[d]) : "l"(3ll));
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 24; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (D > 0 ? D : 1); ++i) s += x[i] + xf[i] + (double)xi[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int D, int KIND>
int run(const char* name, double* out, int sms) {
  const int iters = 20000, blocks = sms, threads = 256;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  k_mix<D, KIND><<<blocks, threads>>>(out, 100);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  k_mix<D, KIND><<<blocks, threads>>>(out, iters);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  const double flops = 2.0 * 256 * 24 * (double)iters * (threads / 32) * blocks;
  printf("%-28s D=%2d  %.2f TFLOP/s DMMA\n", name, D, flops / ms / 1e9);
  return 0;
}

int main() {
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  run<0, 0>("dmma only", out, sms);
  run<6, 0>("dmma + f64 add", out, sms);
  run<12, 0>("dmma + f64 add", out, sms);
  run<24, 0>("dmma + f64 add", out, sms);
  run<6, 1>("dmma + f32 add", out, sms);
  run<24, 1>("dmma + f32 add", out, sms);
  run<6, 2>("dmma + s64 add", out, sms);
  run<24, 2>("dmma + s64 add", out, sms);
  return 0;
}
