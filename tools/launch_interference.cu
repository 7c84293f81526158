// Development microbenchmark: does a PCIe copy in flight on another stream slow a sequence of
// short kernel launches on the compute stream?  Streams of small kernels (param blocks of 64 B
// or ~1 KB, like CtnParams) timed alone, next to an H2D and a D2H copy, and as a CUDA graph.
// Usage: ./launch_interference [launches] [kernel_us]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

struct Small { double* out; long long spin; };
struct Big { double* out; long long spin; char pad[1008]; };

__device__ void spin_for(long long cycles, double* out) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  if (threadIdx.x == 0 && blockIdx.x == 0 && cycles < 0) out[0] = 1.0;
}
__global__ void k_small(const __grid_constant__ Small p) { spin_for(p.spin, p.out); }
__global__ void k_big(const __grid_constant__ Big p) { spin_for(p.spin, p.out); }

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 12;
  const double us = argc > 2 ? atof(argv[2]) : 30.0;
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const long long spin = static_cast<long long>(us * clk_khz / 1000.0);
  double* out;
  CK(cudaMalloc(&out, 64));
  const size_t bytes = 512ull << 20;
  void *h, *d;
  CK(cudaMallocHost(&h, bytes));
  CK(cudaMalloc(&d, bytes));
  cudaStream_t s, c;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  Small ps{out, spin};
  Big pb{};
  pb.out = out;
  pb.spin = spin;
  cudaEvent_t evs[64], evn[64];
  for (int i = 0; i < 64; ++i) {
    CK(cudaEventCreate(&evs[i]));
    CK(cudaEventCreateWithFlags(&evn[i], cudaEventDisableTiming));
  }
  int evmode = 0;  // 0 none, 1 a timing event after each launch, 2 a non-timing event
  auto seq = [&](bool big) {
    for (int i = 0; i < n; ++i) {
      if (big) k_big<<<148, 128, 0, s>>>(pb);
      else k_small<<<148, 128, 0, s>>>(ps);
      if (evmode == 1) CK(cudaEventRecord(evs[i], s));
      if (evmode == 2) CK(cudaEventRecord(evn[i], s));
    }
  };
  cudaGraphExec_t gx[2];
  for (int b = 0; b < 2; ++b) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    seq(b);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&gx[b], g, 0));
    CK(cudaGraphUpload(gx[b], s));
  }
  auto run = [&](const char* label, int copy, int big, bool graph) {
    float best = 1e9, sum = 0;
    const int reps = 7;
    for (int r = 0; r < reps; ++r) {
      CK(cudaDeviceSynchronize());
      if (copy == 1) CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c));
      if (copy == 2) CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c));
      CK(cudaEventRecord(e0, s));
      if (graph) CK(cudaGraphLaunch(gx[big], s));
      else seq(big);
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      sum += ms;
    }
    CK(cudaDeviceSynchronize());
    printf("%-28s %3d launches of %5.1f us: best %7.3f ms  mean %7.3f ms  (%.1f us per launch over the kernel)\n",
           label, n, us, best, sum / reps, (best * 1e3 - n * us) / n);
  };
  for (evmode = 1; evmode < 3; ++evmode)
    for (int copy = 0; copy < 3; ++copy) {
      char l[64];
      snprintf(l, sizeof l, "%s events %s", evmode == 1 ? "timing" : "no-timing",
               copy == 0 ? "alone" : copy == 1 ? "+H2D" : "+D2H");
      run(l, copy, 0, false);
    }
  evmode = 0;
  for (int big = 0; big < 2; ++big)
    for (int graph = 0; graph < 2; ++graph) {
      char l[64];
      for (int copy = 0; copy < 3; ++copy) {
        snprintf(l, sizeof l, "%s %s %s", big ? "1KB-params" : "64B-params", graph ? "graph " : "stream",
                 copy == 0 ? "alone" : copy == 1 ? "+H2D" : "+D2H");
        run(l, copy, big, graph);
      }
    }
  return 0;
}
