// Device-side launch timestamps for the engine's phase timing.
//
// A CUDA timing event recorded on the compute stream costs 30-55 us while a PCIe copy is in
// flight on another stream (3 us without; a non-timing event 5-9 us; tools/launch_interference.cu):
// the streamed drop-in, whose uploads and downloads overlap every chunk, paid ~0.4 ms per C2 call
// for its per-phase event brackets.  Instead every kernel of a timed phase stamps its own slot
// of 4 words with %globaltimer (ns):
//   slot[0] = start (CTA 0 at entry), slot[1] = end (the last CTA to finish),
//   slot[2] = CTA exit counter (reset to 0 by the last CTA, so a slot is reusable without a memset).
// The host reads the slots back at engine_sync (reduce.cpp) and sums each phase's span.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ctn_params.hpp"

namespace hsdla_b200 {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// every thread may call it; CTA (0,0,0)'s thread 0 writes the start
__device__ __forceinline__ void stamp_enter(unsigned long long* st) {
  if (st && threadIdx.x == 0 && threadIdx.y == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
    st[0] = globaltimer_ns();
}
// ONE thread per CTA, after every thread of its CTA finished its work
__device__ __forceinline__ void stamp_leave(unsigned long long* st) {
  if (!st) return;
  __threadfence();
  const unsigned n = gridDim.x * gridDim.y * gridDim.z;
  unsigned int* cnt = reinterpret_cast<unsigned int*>(st + 2);
  if (atomicAdd(cnt, 1u) == n - 1) {
    st[1] = globaltimer_ns();
    atomicExch(cnt, 0u);
  }
}

}  // namespace hsdla_b200
