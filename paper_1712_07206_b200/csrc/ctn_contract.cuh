// Complex-FP64 "conjugate-transpose x none" contraction engine for sm_100a.
//
//   C[i][j] = alpha * sum_s sum_k conj(L_s[k][i]) * R_s[k][j]  (+ beta * C_old)
//
// The one engine behind every product of the refined H/S construction
// (reference kernels.cpp:92-167 / pipeline.cpp:281-329):
//   * TRI mode: lower-triangular N_G x N_G output written to packed-lower storage
//     (ZHERK / ZHER2K / ZHERKX: herk_cols :104-117, her2k_cols :119-135,
//     herkx_cols :137-150).  Tiles enumerate the t(t+1)/2 lower tiles
//     (the idea of hybrid_dynamic.cpp:54-112), the strict upper triangle is never
//     touched and diagonal imaginary parts are forced to 0 (kernels.cpp:112).
//   * BATCH mode: per-atom rectangular products Z_a = T_AB^H A_a + 1/2 T_BB B_a and
//     X_a = T_AA A_a (compute_z pipeline.cpp:176-185 and the hemm_loop
//     :314-321) written straight into the stacked K x N_G buffers.
//
// B200 mapping (no tcgen05 kind::f64 exists; FP64 tensor work is warp-level DMMA):
//   * one elected producer lane streams 128-byte k-slabs of both operands with
//     TMA (cp.async.bulk.tensor, SWIZZLE_128B) into a STAGES-deep smem ring,
//     completion tracked by mbarrier transaction counts;
//   * 4 consumer warps each own a 32x32 complex output tile and run
//     mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Interleaved complex storage maps
//     straight onto real DMMA: for the 4 complex k of one quad, lane q loads the
//     whole complex number (re, im) with one LDS.128, and the k permutation
//     "step 0 = real parts, step 1 = imaginary parts" gives
//        Re += a_re b_re + a_im b_im,   Im += a_re b_im + a_im (-b_re)
//     i.e. exactly 8 real flops per complex MAC (the ledger convention,
//     flop_ledger.hpp) and no 3M trick (rounding stays plain).
//   * smem rows for mma row g are permuted (perm(g) = (g&1)<<2 | g>>1) so the
//     LDS.128 quarter-warps of the swizzled tile are bank-conflict free.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hsdla_b200 {

constexpr int kMaxSeg = 3;
constexpr int kChunkC = 8;  // complex k per TMA slab (128 B rows)

enum CtnMode { kTri = 0, kBatch = 1 };

struct alignas(64) CtnParams {
  CUtensorMap L[kMaxSeg];  // left operands (conjugated), 3-D maps
  CUtensorMap R[kMaxSeg];  // right operands
  int kchunks[kMaxSeg];    // 8-complex slabs per segment
  int l_row_z[kMaxSeg];    // 1: tile row coordinate in dim 2, atom in dim 1; 0: row in dim 1, atom in dim 2
  int r_row_z[kMaxSeg];
  int nseg;
  int n;                   // TRI: order N_G.  BATCH: number of output columns (N_G)
  int m_valid;             // BATCH: valid output rows per atom (N_L)
  int tiles;               // TRI: tiles per dimension
  double2* out;            // TRI: packed lower.  BATCH: column-major stacked buffer
  uint64_t ldo;            // BATCH: output leading dimension (complex elements)
  double alpha_re, alpha_im;
  double beta;             // real; 0 => C is never read
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Lower-tile index t -> (ti, tj), ti >= tj, tiles ordered row by row.
__device__ __forceinline__ void tri_tile(int t, int& ti, int& tj) {
  int r = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  while (r * (r + 1) / 2 > t) --r;
  ti = r;
  tj = t - r * (r + 1) / 2;
}

__device__ __forceinline__ uint64_t packed_index(uint64_t n, uint64_t i, uint64_t j) {
  // column-major packed lower ('L'): column j holds rows j..n-1
  return j * (2 * n - j + 1) / 2 + (i - j);
}

template <int MODE, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
struct CtnCfg {
  static constexpr int kConsumerWarps = WARPS_M * WARPS_N;
  static constexpr int kThreads = (kConsumerWarps + 1) * 32;
  static constexpr int kWM = BM / WARPS_M;
  static constexpr int kWN = BN / WARPS_N;
  static constexpr int kMB = kWM / 8;
  static constexpr int kNB = kWN / 8;
  static constexpr int kStageL = BM * 128;
  static constexpr int kStageR = BN * 128;
  static constexpr int kStageBytes = kStageL + kStageR;
  static constexpr int kSmemBytes = STAGES * kStageBytes + 1024 /*align*/ + 2 * STAGES * 8 + 64;
};

template <int MODE, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB = 1>
__global__ void __launch_bounds__(CtnCfg<MODE, BM, BN, WARPS_M, WARPS_N, STAGES>::kThreads, MINB)
    ctn_contract_kernel(const __grid_constant__ CtnParams P) {
  using Cfg = CtnCfg<MODE, BM, BN, WARPS_M, WARPS_N, STAGES>;
  constexpr int MB = Cfg::kMB, NB = Cfg::kNB;
  static_assert(BM % (8 * WARPS_M) == 0 && BN % (8 * WARPS_N) == 0, "tile shape");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- which output tile --------------------------------------------------
  int row0, col0, atom;
  if (MODE == kTri) {
    int ti, tj;
    tri_tile(blockIdx.x, ti, tj);
    row0 = ti * BM;
    col0 = tj * BN;
    atom = 0;
  } else {
    col0 = blockIdx.x * BN;
    row0 = blockIdx.y * BM;
    atom = blockIdx.z;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int total = 0;
#pragma unroll
  for (int s = 0; s < kMaxSeg; ++s)
    if (s < P.nseg) total += P.kchunks[s];

  if (warp == Cfg::kConsumerWarps) {
    // ===================== TMA producer (one lane) =========================
    if (lane == 0) {
      for (int s = 0; s < P.nseg; ++s) {
        prefetch_map(&P.L[s]);
        prefetch_map(&P.R[s]);
      }
      int seg = 0, kc = 0;
      for (int c = 0; c < total; ++c) {
        while (kc >= P.kchunks[seg]) {
          kc = 0;
          ++seg;
        }
        const int slot = c % STAGES;
        const uint32_t par = ((c / STAGES) & 1) ^ 1;
        mbar_wait(&empty[slot], par);
        uint8_t* sL = smem + slot * Cfg::kStageBytes;
        uint8_t* sR = sL + Cfg::kStageL;
        mbar_arrive_expect_tx(&full[slot], Cfg::kStageBytes);
        const int x = kc * 2 * kChunkC;
        if (P.l_row_z[seg])
          tma_load_3d(sL, &P.L[seg], x, atom, row0, &full[slot]);
        else
          tma_load_3d(sL, &P.L[seg], x, row0, atom, &full[slot]);
        if (P.r_row_z[seg])
          tma_load_3d(sR, &P.R[seg], x, atom, col0, &full[slot]);
        else
          tma_load_3d(sR, &P.R[seg], x, col0, atom, &full[slot]);
        ++kc;
      }
    }
    return;
  }

  // ======================= DMMA consumers =================================
  const int wm = warp % WARPS_M;
  const int wn = warp / WARPS_M;
  const int g = lane >> 2;
  const int q = lane & 3;
  const int pg = ((g & 1) << 2) | (g >> 1);  // smem row permutation (bank-conflict-free LDS.128)

  uint32_t offL[MB], offR[NB], offK[2];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) offL[mb] = (wm * Cfg::kWM + 8 * mb + pg) * 128;
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) offR[nb] = Cfg::kStageL + (wn * Cfg::kWN + 8 * nb + pg) * 128;
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) offK[kk] = ((4 * kk + q) ^ pg) << 4;

  double cre[MB][NB][2], cim[MB][NB][2];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      cre[mb][nb][0] = cre[mb][nb][1] = 0.0;
      cim[mb][nb][0] = cim[mb][nb][1] = 0.0;
    }

  for (int c = 0; c < total; ++c) {
    const int slot = c % STAGES;
    mbar_wait(&full[slot], (c / STAGES) & 1);
    const uint8_t* st = smem + slot * Cfg::kStageBytes;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      double2 a[MB], b[NB];
      double nbr[NB];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) a[mb] = *reinterpret_cast<const double2*>(st + offL[mb] + offK[kk]);
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        b[nb] = *reinterpret_cast<const double2*>(st + offR[nb] + offK[kk]);
        nbr[nb] = -b[nb].x;
      }
      // Four independent sweeps so consecutive DMMAs never share an accumulator.
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma(cre[mb][nb][0], cre[mb][nb][1], a[mb].x, b[nb].x);
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma(cim[mb][nb][0], cim[mb][nb][1], a[mb].x, b[nb].y);
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma(cre[mb][nb][0], cre[mb][nb][1], a[mb].y, b[nb].y);
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma(cim[mb][nb][0], cim[mb][nb][1], a[mb].y, nbr[nb]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }

  // ---- epilogue -------------------------------------------------------------
  const double ar = P.alpha_re, ai = P.alpha_im, beta = P.beta;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const int i = row0 + wm * Cfg::kWM + 8 * mb + pg;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = col0 + wn * Cfg::kWN + 8 * nb + (e ? 4 + q : q);
        const double xr = cre[mb][nb][e], xi = cim[mb][nb][e];
        double vr = ar * xr - ai * xi;
        double vi = ar * xi + ai * xr;
        if (MODE == kTri) {
          if (i < P.n && j < P.n && i >= j) {
            if (i == j) vi = 0.0;
            double2* dst = P.out + packed_index(P.n, i, j);
            if (beta != 0.0) {
              const double2 o = *dst;
              vr += beta * o.x;
              vi += beta * o.y;
            }
            *dst = make_double2(vr, vi);
          }
        } else {
          if (i < P.m_valid && j < P.n) {
            double2* dst = P.out + (static_cast<uint64_t>(atom) * P.m_valid + i) + static_cast<uint64_t>(j) * P.ldo;
            if (beta != 0.0) {
              const double2 o = *dst;
              vr += beta * o.x;
              vi += beta * o.y;
            }
            *dst = make_double2(vr, vi);
          }
        }
      }
    }
  }
}

}  // namespace hsdla_b200
