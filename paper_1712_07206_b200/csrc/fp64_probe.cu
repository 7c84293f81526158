// FP64 roofline probe: sustained DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4)
// throughput on all SMs.  Measured denominator for roofline.frac (MEASURED_PEAKS.json
// carries no FP64 figure).  Not on the H/S path.
#include <cuda_runtime.h>

#include <string>

#include "../../include/hsdla_b200.h"

namespace hsdla_b200 {
extern thread_local std::string g_last_error;
}

namespace {

__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

}  // namespace

extern "C" int hsdla_b200_fp64_peak(int device, double seconds, double* tflops) {
  auto fail = [](cudaError_t e) {
    (void)cudaGetLastError();
    hsdla_b200::g_last_error = std::string("fp64_peak: ") + cudaGetErrorString(e);
    return HSDLA_B200_CUDA_ERROR;
  };
  cudaError_t e;
  if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(e);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if ((e = cudaMalloc(&out, 4096)) != cudaSuccess) return fail(e);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 2, threads = 256, iters = 4000;
  const double flops = 2.0 * 256 * 8 * iters * (threads / 32) * static_cast<double>(blocks);
  dmma_loop<<<blocks, threads>>>(out, iters);  // warm-up
  cudaEventRecord(e0);
  int launches = 0;
  float ms = 0.f;
  do {
    dmma_loop<<<blocks, threads>>>(out, iters);
    ++launches;
    if (launches % 16 == 0) {
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
  } while (ms < seconds * 1e3 && launches < 100000);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return fail(e);
  if (tflops) *tflops = flops * launches / (ms * 1e-3) / 1e12;
  return HSDLA_B200_OK;
}
