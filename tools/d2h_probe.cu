// D2H copy-rate probe (development helper): cudaMallocHost staging, halves / pieces / offsets.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t half = 8008000, total = 2 * half;
  char *h, *d;
  cudaMallocHost(&h, total);
  cudaMalloc(&d, total);
  cudaMemset(d, 1, total);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, size_t off, size_t bytes, size_t piece) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a, s);
      for (size_t o = 0; o < bytes; o += piece)
        cudaMemcpyAsync(h + off + o, d + off + o, (o + piece < bytes ? piece : bytes - o), cudaMemcpyDeviceToHost, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%-28s off %9zu bytes %9zu piece %9zu: %.3f ms (%.1f GB/s)\n", name, off, bytes, piece, ms, bytes / ms / 1e6);
    }
  };
  run("first half, one copy", 0, half, half);
  run("second half, one copy", half, half, half);
  run("second half, 1 MB pieces", half, half, 1 << 20);
  run("first half, 1 MB pieces", 0, half, 1 << 20);
  run("whole, one copy", 0, total, total);
  run("second half+64, one copy", half + 64, half - 64, half);
  // the CPU reads the landed bytes between copies (the unpack)
  volatile double sink = 0;
  auto cpu_read = [&](size_t off, size_t bytes) {
    double acc = 0;
    const double* p = reinterpret_cast<const double*>(h + off);
    for (size_t i = 0; i < bytes / 8; ++i) acc += p[i];
    sink = acc;
  };
  for (int rep = 0; rep < 3; ++rep) {
    cpu_read(0, total);
    run("after CPU read: second half", half, half, half);
    cpu_read(0, total);
    run("after CPU read: first half", 0, half, half);
  }
  // a wait on an event recorded on another stream first
  cudaStream_t s2;
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, s2);
  cudaStreamSynchronize(s2);
  cudaStreamWaitEvent(s, ev, 0);
  run("after a cross-stream wait", half, half, half);
  return 0;
}
