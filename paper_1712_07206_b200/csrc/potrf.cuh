// Batched per-atom Cholesky try/fail of T_AA and the left-operand select of the
// original algorithm (Algorithm 1; reference pipeline.cpp:229-251).
//
// potrf_batched_kernel — kernels::potrf (kernels.cpp:417-436) for every atom block:
//   one CTA per atom, the reference's left-looking column order replayed with
//   explicitly rounded operations (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn /
//   __dsqrt_rn: no FMA contraction), so the factor and the failing pivot are
//   bit-identical to the reference's (tests/test_gpu_original.py pins it against
//   tests/golden/potrf_blocks.npz).  std::norm(z) = x*x + y*y (libstdc++
//   _Norm_helper<true>); l * conj(m) is the builtin complex product
//   (re = a c - b (-d), im = a (-d) + b c); s / l_jj is componentwise.
//   Output per atom, column-major N_L x N_L:
//     success: Q = L (lower factor, upper exactly 0), info = -1
//              -> the batched contraction Q^H A_a is the reference's
//                 trmm(Left, ConjTrans, L, A_a) (kernels.cpp:385-415);
//     failure: Q with Q^H = the hemm operator of T_AA's LOWER triangle (full(T_AA)
//              with the diagonal conjugated), info = pivot
//              -> Q^H A_a = T_AA A_a, the reference's hemm fallback.
//   O(N_L^3 / 3) flops per atom (0.3 GFLOP at config 4): latency-bound, negligible
//   next to the contractions; the block lives in L1/L2 (global scratch = Q itself).
//
// select_left_kernel — the left operand of the h_aa_update contraction:
//   W_a = Q_a^H A_a (in X1) and  Lft_a = W_a (HPD atom) | A_a (failed atom), so
//   H += Lft^H W = sum_hpd A^H L L^H A + sum_fail A^H T_AA A, lower triangle only —
//   the reference's herk(B_T) + lower(gemm(A_f, B_B)) (pipeline.cpp:253-276) as ONE
//   K-deep contraction without compacting the atoms.  HBM-bound copy.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "stamp.cuh"

namespace hsdla_b200 {

// n_fail (nullable) counts the atoms that did not factorise.
__global__ void __launch_bounds__(128) potrf_batched_kernel(const double2* __restrict__ taa, double2* __restrict__ q,
                                                            int32_t* __restrict__ info, int nl,
                                                            int* __restrict__ n_fail = nullptr,
                                                            unsigned long long* stamp = nullptr) {
  stamp_enter(stamp);
  const uint64_t blk = static_cast<uint64_t>(nl) * nl;
  const double2* T = taa + blockIdx.x * blk;
  double2* L = q + blockIdx.x * blk;
  __shared__ double s_ljj;
  __shared__ int s_fail;
  for (uint64_t idx = threadIdx.x; idx < blk; idx += blockDim.x) L[idx] = make_double2(0.0, 0.0);
  __syncthreads();
  int fail_at = -1;
  for (int j = 0; j < nl; ++j) {
    if (threadIdx.x == 0) {
      double d = T[j + static_cast<uint64_t>(j) * nl].x;
      for (int p = 0; p < j; ++p) {
        const double2 v = L[j + static_cast<uint64_t>(p) * nl];
        d = __dsub_rn(d, __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y)));
      }
      const int fail = !(d > 0.0) || !isfinite(d);
      s_fail = fail;
      if (!fail) {
        const double ljj = __dsqrt_rn(d);
        s_ljj = ljj;
        L[j + static_cast<uint64_t>(j) * nl] = make_double2(ljj, 0.0);
      }
    }
    __syncthreads();
    if (s_fail) {
      fail_at = j;
      break;
    }
    const double ljj = s_ljj;
    for (int i = j + 1 + threadIdx.x; i < nl; i += blockDim.x) {
      double2 s = T[i + static_cast<uint64_t>(j) * nl];
      for (int p = 0; p < j; ++p) {
        const double2 a = L[i + static_cast<uint64_t>(p) * nl];
        const double2 b = L[j + static_cast<uint64_t>(p) * nl];
        const double nbi = -b.y;
        const double tr = __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, nbi));
        const double ti = __dadd_rn(__dmul_rn(a.x, nbi), __dmul_rn(a.y, b.x));
        s.x = __dsub_rn(s.x, tr);
        s.y = __dsub_rn(s.y, ti);
      }
      L[i + static_cast<uint64_t>(j) * nl] = make_double2(__ddiv_rn(s.x, ljj), __ddiv_rn(s.y, ljj));
    }
    __syncthreads();
  }
  if (fail_at >= 0) {
    // hemm operand Q, Q^H = T_AA read from its lower triangle (kernels.cpp:152-167)
    for (uint64_t idx = threadIdx.x; idx < blk; idx += blockDim.x) {
      const int k = static_cast<int>(idx % nl), i = static_cast<int>(idx / nl);  // element (k, i)
      double2 v = k >= i ? T[k + static_cast<uint64_t>(i) * nl] : T[i + static_cast<uint64_t>(k) * nl];
      if (k <= i) v.y = -v.y;
      L[idx] = v;
    }
  }
  if (threadIdx.x == 0) {
    info[blockIdx.x] = fail_at;
    if (fail_at >= 0 && n_fail) atomicAdd(n_fail, 1);
  }
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) stamp_leave(stamp);
  }
}

// X2[r, j] = info[atom(r)] < 0 ? X1[r, j] : A[r, j] for the rows [0, Kc) of a chunk
// (pointers already offset to the chunk's first row; ld = K).
__global__ void select_left_kernel(const double2* __restrict__ X1, const double2* __restrict__ A,
                                   const int32_t* __restrict__ info, double2* __restrict__ X2, uint64_t Kc,
                                   uint64_t ld, uint64_t ng, int nl, unsigned long long* stamp = nullptr) {
  stamp_enter(stamp);
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < Kc) {
    const bool hpd = info[k / nl] < 0;
    const double2* src = hpd ? X1 : A;
    for (uint64_t j = blockIdx.y; j < ng; j += gridDim.y) X2[k + j * ld] = src[k + j * ld];
  }
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) stamp_leave(stamp);
  }
}

}  // namespace hsdla_b200
