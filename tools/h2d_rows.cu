// Development microbenchmark: H2D throughput of a 2-D copy (pinned, contiguous source rows of
// `row` bytes -> device rows at a pitch of 83 KB, the chunk-row upload of the drop-in) against
// the row size, and of a plain 1-D copy of the same bytes.
#include <cuda_runtime.h>

#include <cstdio>

int main() {
  const size_t total = 64ull << 20, dpitch = 5184 * 16;
  void *h, *d;
  cudaMallocHost(&h, total);
  cudaMalloc(&d, dpitch * 20000);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t row : {1296ul, 2592ul, 6480ul, 12960ul, 25920ul, 40176ul, 82944ul}) {
    const size_t n = std::min<size_t>(total / row, 20000);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, s);
      cudaMemcpy2DAsync(d, dpitch, h, row, row, n, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    float best1 = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, s);
      cudaMemcpyAsync(d, h, row * n, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best1 = ms < best1 ? ms : best1;
    }
    float bestd = 1e9;  // device contiguous -> device pitched (copy engine)
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, s);
      cudaMemcpy2DAsync(d, dpitch, static_cast<char*>(d) + dpitch * 20000 - total, row, row, n,
                        cudaMemcpyDeviceToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      bestd = ms < bestd ? ms : bestd;
    }
    // pitched (83 KB) host source -> contiguous / pitched device (the pinned caller's strided rows)
    static char* hp = nullptr;
    if (!hp) cudaMallocHost(&hp, dpitch * 20000);
    float bs = 1e9, bss = 1e9;
    for (int r = 0; r < 5; ++r) {
      float ms;
      cudaEventRecord(e0, s);
      cudaMemcpy2DAsync(d, row, hp, dpitch, row, n, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      bs = ms < bs ? ms : bs;
      cudaEventRecord(e0, s);
      cudaMemcpy2DAsync(d, dpitch, hp, dpitch, row, n, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      bss = ms < bss ? ms : bss;
    }
    float bp1 = 1e9, bp2 = 1e9;  // small host pitches: row + 64 B, row rounded up to 4 KB
    for (int r = 0; r < 5; ++r) {
      float ms;
      const size_t p1 = row + 64, p2 = (row + 4095) / 4096 * 4096 + (row % 4096 == 0 ? 4096 : 0);
      const size_t m1 = std::min(n, dpitch * 20000 / p1), m2 = std::min(n, dpitch * 20000 / p2);
      cudaEventRecord(e0, s);
      cudaMemcpy2DAsync(d, dpitch, hp, p1, row, m1, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      bp1 = std::min(bp1, ms * n / m1);
      cudaEventRecord(e0, s);
      cudaMemcpy2DAsync(d, dpitch, hp, p2, row, m2, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      bp2 = std::min(bp2, ms * n / m2);
    }
    printf("  host pitch row+64 -> pitched %5.1f GB/s, host pitch 4K-rounded -> pitched %5.1f GB/s\n",
           row * n / bp1 / 1e6, row * n / bp2 / 1e6);
    printf("row %6zu B x %5zu rows (%5.1f MB): H2D contiguous->pitched %5.1f, pitched->contiguous %5.1f, "
           "pitched->pitched %5.1f, 1-D %5.1f GB/s; D2D 2-D %6.1f GB/s\n", row, n, row * n / 1e6,
           row * n / best / 1e6, row * n / bs / 1e6, row * n / bss / 1e6, row * n / best1 / 1e6, row * n / bestd / 1e6);
  }
  return 0;
}
