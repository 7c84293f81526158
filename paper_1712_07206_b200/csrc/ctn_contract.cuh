// Complex-FP64 "conjugate-transpose x none" contraction engine for sm_100a.
//
//   C[i][j] = alpha * sum_s sum_k conj(L_s[k][i]) * R_s[k][j]  (+ beta * C_old)
//
// The one engine behind every product of the refined H/S construction
// (reference kernels.cpp:92-167 / pipeline.cpp:281-329):
//   * TRI modes: lower-triangular N_G x N_G output written to packed-lower storage
//     (ZHERK / ZHER2K / ZHERKX: herk_cols :104-117, her2k_cols :119-135,
//     herkx_cols :137-150).  Tiles enumerate the lower tiles (the idea of
//     hybrid_dynamic.cpp:54-112); the strict upper triangle is never touched and
//     diagonal imaginary parts are forced to 0 (kernels.cpp:112).  kTri covers the
//     strictly-lower tiles (or every lower tile, `with_diag`), kTriDiag the diagonal
//     tiles and kTriRow a ragged last tile row, each with its own warp assignment
//     (launch_tri_kernel in contract.cu issues them).
//   * BATCH mode (persistent: CTAs loop over column x row x atom tiles, so the next
//     tile's TMA loads overlap the current tile's epilogue): per-atom rectangular
//     products Z_a = T_AB^H A_a + 1/2 T_BB B_a, X_a = T_AA A_a (compute_z
//     pipeline.cpp:176-185 and the hemm_loop :314-321) and the merged algorithm's
//     [W_A; W_B] = M_a Y_a, written straight into the stacked K x N_G buffers.
//
// B200 mapping (no tcgen05 kind::f64 exists; FP64 tensor work is warp-level DMMA):
//   * one elected producer lane streams 128-byte k-slabs of both operands with
//     TMA (cp.async.bulk.tensor, SWIZZLE_128B) into a STAGES-deep smem ring,
//     completion tracked by mbarrier transaction counts;
//   * 8 consumer warps (two warpgroups) each own a 32x16 complex output tile and
//     run mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); the producer has a warpgroup of its
//     own so setmaxnreg can hand its registers to the consumers (232 each).
//     Interleaved complex storage maps straight onto real DMMA: for the 4 complex k
//     of one quad, lane q loads the whole complex number (re, im) with one LDS.128.
//     4M (G3M = 0): Re += a_re b_re + a_im b_im, Im += a_re b_im + a_im (-b_re):
//     8 real flops per complex MAC, the ledger convention (flop_ledger.hpp).
//     3M (G3M = 1, default): Gauss's product, 3 real DMMAs (6 flops) per complex MAC.
//   * smem rows for mma row g are permuted (perm(g) = (g&1)<<2 | g>>1) so the
//     LDS.128 quarter-warps of the swizzled tile are bank-conflict free.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "ctn_params.hpp"
#include "stamp.cuh"

namespace hsdla_b200 {

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
// the same on shared-window addresses (hoisted conversions in the consumers' k-loop)
__device__ __forceinline__ void mbar_arrive_u(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
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

__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Lower-tile index t -> (ti, tj), ti >= tj, in an L2-friendly grouped order:
// tile rows are taken in bands of kBand rows (kBand = 1: plain row-by-row order) (band b holds the same tiles as rows
// [b*kBand, (b+1)*kBand) of the row-by-row order, so the band start is the
// row-major prefix), and inside a band the tiles go column by column.  One wave of
// 148 persistent CTAs then covers ~kBand row blocks x ~148/kBand column blocks of
// the operands instead of 1 x 148, so each k-slab of an operand block is fetched
// from HBM once per wave and re-served from L2 to the other CTAs of its band.
__device__ __forceinline__ void tri_tile(int t, int tiles, int kBand, int& ti, int& tj) {
  int r = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);  // row in the row-by-row order
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  while (r * (r + 1) / 2 > t) --r;
  const int r0 = (r / kBand) * kBand;
  const int h = min(kBand, tiles - r0);  // rows in this band
  int u = t - r0 * (r0 + 1) / 2;         // index inside the band
  if (u < r0 * h) {                      // rectangular part: columns 0 .. r0-1, h tiles each
    tj = u / h;
    ti = r0 + (u - tj * h);
    return;
  }
  u -= r0 * h;  // triangular part: column c (tj = r0 + c) holds rows r0+c .. r0+h-1
  int c = 0;
  while (u >= h - c) {
    u -= h - c;
    ++c;
  }
  tj = r0 + c;
  ti = r0 + c + u;
}

// Tile t of the lower tiles (diagonal included) restricted to tile columns [c0, c1): the triangle
// of rows c0 .. c1-1 first (row by row), then the full-width rows c1 .. (w = c1 - c0 tiles each).
// A column band of tiles covers a contiguous range of packed-lower storage, so a build's final H
// contraction can run band by band with each band's download overlapping the next band's compute.
__device__ __forceinline__ void tri_tile_cols(int t, int c0, int c1, int& ti, int& tj) {
  const int w = c1 - c0, tri = w * (w + 1) / 2;
  if (t < tri) {
    int r = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    ti = c0 + r;
    tj = c0 + t - r * (r + 1) / 2;
  } else {
    const int u = t - tri;
    ti = c1 + u / w;
    tj = c0 + u % w;
  }
}

// Tile t of the STRICTLY lower tiles (ti > tj) restricted to tile columns [c0, c1) (c1 == 0:
// all T columns, grouped order of tri_tile): the triangle of rows c0+1 .. c1-1, then the full
// rows c1 .. (w = c1 - c0 tiles each).  The diagonal tiles run in a launch of their own.
__device__ __forceinline__ void tri_tile_strict(int t, int T, int c0, int c1, int kBand, int& ti, int& tj) {
  if (c1 <= 0) {  // the whole triangle: the lower tiles of the (T-1)-grid, one row down
    tri_tile(t, T - 1, kBand, ti, tj);
    ++ti;
    return;
  }
  const int w = c1 - c0, tri = w * (w - 1) / 2;
  if (t < tri) {
    int r = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);  // row r + 1 of the window triangle
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    ti = c0 + 1 + r;
    tj = c0 + t - r * (r + 1) / 2;
  } else {
    const int u = t - tri;
    ti = c1 + u / w;
    tj = c0 + u % w;
  }
}

__device__ __forceinline__ uint64_t packed_index(uint64_t n, uint64_t i, uint64_t j) {
  // column-major packed lower ('L'): column j holds rows j..n-1
  return j * (2 * n - j + 1) / 2 + (i - j);
}

// KSUB: 128-byte k-slabs (8 complex) per pipeline stage; one full/empty mbarrier
// handshake per stage, so KSUB > 1 amortises the synchronisation over more DMMAs.
// PW: producer warps.  4: the producer is a warpgroup of its own (one TMA lane, three idle
// warps) and setmaxnreg moves registers from it to the consumers at run time; ptxas still
// compiles the consumers against the 384-thread launch bound (168 registers).  1: a single
// producer warp, no setmaxnreg; the 288-thread launch bound lets ptxas give every thread
// up to 224 registers, room for larger warp tiles.
template <int MODE, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int KSUB = 1, int PW = 4>
struct CtnCfg {
  static constexpr int kConsumerWarps = WARPS_M * WARPS_N;
  static constexpr int kProducerWarps = PW;
  static constexpr int kThreads = (kConsumerWarps + kProducerWarps) * 32;
  static constexpr int kProducerRegs = 40;
  static constexpr int kConsumerRegs =
      ((65536 / kThreads / 8 * 8) * kThreads - kProducerRegs * kProducerWarps * 32) / (kConsumerWarps * 32) / 8 * 8;
  static constexpr int kWM = BM / WARPS_M;
  static constexpr int kWN = BN / WARPS_N;
  static constexpr int kMB = kWM / 8;
  static constexpr int kNB = kWN / 8;
  static constexpr int kSubL = BM * 128;  // one k-slab of the left operand tile
  static constexpr int kSubR = BN * 128;
  static constexpr int kStageL = KSUB * kSubL;
  static constexpr int kStageR = KSUB * kSubR;
  static constexpr int kStageBytes = kStageL + kStageR;
  static constexpr int kSmemBytes = STAGES * kStageBytes + 1024 /*align*/ + 2 * STAGES * 8 + 64;
};

// ---------------------------------------------------------------------------
// Work decomposition.  BATCH: persistent CTAs, whole tiles blockIdx.x, +gridDim.x, ...
// TRI: persistent CTAs (grid = #SMs) with a data-parallel + stream-K split:
// all full waves but the last are whole tiles (tile b, b+G, ...); the remaining
// tiles' k-iterations are divided evenly over the G CTAs, so the last wave has no
// idle SMs.  A tile cut between CTAs is finished by its OWNER (the CTA holding its
// k = 0 piece, processed LAST in that CTA's range); the other contributors process
// their piece FIRST, park the partial accumulators in a workspace slot and publish
// a per-CTA flag (release/acquire).  The owner adds partials in a fixed order,
// so the result is bitwise deterministic run to run.
// ---------------------------------------------------------------------------
struct Piece {
  int tile, k0, k1;
  int kind;  // 0 whole tile, 1 owner (k0 == 0, k1 < I), 2 contributor (k0 > 0)
};

struct TriSched {
  int G, b, I, dp_tiles, dp_next;
  long long sk_total, sk_pos, sk_end;
  __device__ TriSched(int tiles, int iters, int grid, int block) : G(grid), b(block), I(iters) {
    dp_tiles = (tiles % grid == 0) ? tiles : max(0, tiles / grid - 1) * grid;
    sk_total = static_cast<long long>(tiles - dp_tiles) * iters;
    sk_pos = start(block);
    sk_end = start(block + 1);
    dp_next = block;
  }
  __device__ long long start(int cta) const { return sk_total * cta / G; }
  __device__ bool next(Piece& p) {
    if (dp_next < dp_tiles) {
      p.tile = dp_next;
      p.k0 = 0;
      p.k1 = I;
      p.kind = 0;
      dp_next += G;
      return true;
    }
    if (sk_pos < sk_end) {
      const int t = static_cast<int>(sk_pos / I);
      p.k0 = static_cast<int>(sk_pos - static_cast<long long>(t) * I);
      const long long rem = sk_end - sk_pos;
      p.k1 = static_cast<int>(p.k0 + rem < I ? p.k0 + rem : I);
      p.tile = dp_tiles + t;
      p.kind = (p.k0 == 0 && p.k1 == I) ? 0 : (p.k0 == 0 ? 1 : 2);
      sk_pos += p.k1 - p.k0;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Fragment masks of a warp tile (bit mb * NB + nb: the 8 x 8 fragment (mb, nb) is computed).
__host__ __device__ constexpr bool frag_on(unsigned m, int mb, int nb, int NB) { return (m >> (mb * NB + nb)) & 1u; }
__host__ __device__ constexpr bool row_on(unsigned m, int mb, int NB) {
  return ((m >> (mb * NB)) & ((1u << NB) - 1u)) != 0;
}
__host__ __device__ constexpr bool col_on(unsigned m, int nb, int MB, int NB) {
  for (int mb = 0; mb < MB; ++mb)
    if (frag_on(m, mb, nb, NB)) return true;
  return false;
}
// Diagonal TRI tiles (64 x 64, 8 warps of 32 x 16): of the 8 x 8 fragments only the 36 on or below
// the diagonal carry output.  Roles by warp tile (wm, wn): (1,0), (1,1) all 8 fragments; (0,0),
// (1,2) the 7 with mb >= nb; (0,1), (1,3) the 3 with mb >= nb + 2; (0,2), (0,3) none.  The warps
// are re-assigned so the two warps of each SM sub-partition (w, w + 4) carry 8 / 8 / 10 / 10
// fragments instead of 7 / 15 / 3 / 11: the tile takes 10 / 16 of a full tile's DMMA time.
constexpr unsigned kMaskFull = 0xFFu, kMaskTri7 = 0xFDu, kMaskTri3 = 0xD0u, kMaskNone = 0u;

// G3M = 0: four real DMMAs per complex MAC (8 flops, plain FP64 rounding).
// G3M = 1: Gauss's three-multiplication complex product (the ZGEMM3M scheme, 6 executed
//   flops per complex MAC): per k, t1 += a_r b_r, t2 += a_i b_i, t3 += (a_r - a_i)(b_r + b_i),
//   then Re(conj(a) b) = t1 + t2 and Im = t3 - t1 + t2.  Still all-FP64; the imaginary
//   part's rounding error bound grows by a small constant factor.
template <int MODE, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB = 1, int G3M = 0, int KSUB = 1,
          int PW = 4>
__global__ void __launch_bounds__(CtnCfg<MODE, BM, BN, WARPS_M, WARPS_N, STAGES, KSUB, PW>::kThreads, MINB)
    ctn_contract_kernel(const __grid_constant__ CtnParams P) {
  using Cfg = CtnCfg<MODE, BM, BN, WARPS_M, WARPS_N, STAGES, KSUB, PW>;
  constexpr int MB = Cfg::kMB, NB = Cfg::kNB;
  constexpr int NCT = Cfg::kConsumerWarps * 32;  // consumer threads
  constexpr int NS = G3M ? 3 : 2;                // accumulator sets per output element
  constexpr int NACC = MB * NB * 2 * NS;         // accumulator doubles per consumer thread
  static_assert(BM % (8 * WARPS_M) == 0 && BN % (8 * WARPS_N) == 0, "tile shape");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  stamp_enter(P.stamp);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int iters = 0;
#pragma unroll
  for (int s = 0; s < kMaxSeg; ++s)
    if (s < P.nseg) iters += P.kchunks[s];

  // tile coordinates of a piece
  constexpr bool kTriLike = MODE != kBatch;
  auto tile_origin = [&](int tile, int& row0, int& col0, int& atom) {
    if (MODE == kTriDiag) {
      row0 = col0 = (P.diag_t0 + tile) * BM;
      atom = 0;
    } else if (MODE == kTriRow) {
      row0 = P.row_ti * BM;
      col0 = (P.diag_t0 + tile) * BN;
      atom = 0;
    } else if (MODE == kTri) {
      int ti, tj;
      if (P.with_diag) {
        if (P.col_t1 > 0)
          tri_tile_cols(tile, P.col_t0, P.col_t1, ti, tj);
        else
          tri_tile(tile, P.tiles, P.band, ti, tj);
      } else {
        tri_tile_strict(tile, P.tiles, P.col_t0, P.col_t1, P.band, ti, tj);
      }
      row0 = ti * BM;
      col0 = tj * BN;
      atom = 0;
    } else {
      // persistent BATCH: tile = (column tile fastest, then row tile, then atom)
      const int tx = tile % P.bat_tx, rest = tile / P.bat_tx;
      col0 = tx * BN;
      row0 = (rest % P.bat_ty) * BM;
      atom = rest / P.bat_ty;
    }
  };

  static_assert(PW == 1 || Cfg::kConsumerWarps % 4 == 0, "consumer warps must form whole warpgroups");
  if (warp >= Cfg::kConsumerWarps) {
    // ===================== TMA producer (one lane) =========================
    if (PW == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::kProducerRegs) : "memory");
    if (warp == Cfg::kConsumerWarps && lane == 0) {
      for (int s = 0; s < P.nseg; ++s) {
        prefetch_map(&P.L[s]);
        prefetch_map(&P.R[s]);
      }
      TriSched sched(P.tiles_total, iters, gridDim.x, blockIdx.x);
      Piece pc;
      int bt = blockIdx.x;  // BATCH: tiles blockIdx.x, + gridDim.x, ...
      bool have = kTriLike ? sched.next(pc) : bt < P.bat_tiles;
      if (!kTriLike) pc = Piece{bt, 0, iters, 0};
      int it = 0;
      while (have) {
        int row0, col0, atom;
        tile_origin(pc.tile, row0, col0, atom);
        int seg = 0, kc = pc.k0;
        while (seg < P.nseg - 1 && kc >= P.kchunks[seg]) kc -= P.kchunks[seg++];
        for (int c = pc.k0; c < pc.k1; c += KSUB, ++it) {
          const int n = min(KSUB, pc.k1 - c);  // k-slabs in this stage
          const int slot = it % STAGES;
          mbar_wait(&empty[slot], ((it / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[slot], n * (Cfg::kSubL + Cfg::kSubR));
          for (int u = 0; u < n; ++u) {
            while (kc >= P.kchunks[seg]) {
              kc = 0;
              ++seg;
            }
            uint8_t* sL = smem + slot * Cfg::kStageBytes + u * Cfg::kSubL;
            uint8_t* sR = smem + slot * Cfg::kStageBytes + Cfg::kStageL + u * Cfg::kSubR;
            const int x = kc * 2 * kChunkC;
            // TRI: operand columns are held from global column g0 on (column windows)
            const int lr = kTriLike ? row0 - P.g0 : row0, lc = kTriLike ? col0 - P.g0 : col0;
            if (P.l_row_z[seg])
              tma_load_3d(sL, &P.L[seg], x, atom, lr, &full[slot]);
            else
              tma_load_3d(sL, &P.L[seg], x, lr, atom, &full[slot]);
            if (P.r_row_z[seg])
              tma_load_3d(sR, &P.R[seg], x, atom, lc, &full[slot]);
            else
              tma_load_3d(sR, &P.R[seg], x, lc, atom, &full[slot]);
            ++kc;
          }
        }
        if (kTriLike) {
          have = sched.next(pc);
        } else {
          bt += gridDim.x;
          have = bt < P.bat_tiles;
          pc = Piece{bt, 0, iters, 0};
        }
      }
    }
    return;
  }

  // ======================= DMMA consumers =================================
  if (PW == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::kConsumerRegs) : "memory");
  const int ctid = threadIdx.x;  // 0 .. NCT-1
  const int g = lane >> 2;
  const int q = lane & 3;
  const int pg = ((g & 1) << 2) | (g >> 1);  // smem row permutation (bank-conflict-free LDS.128)
  constexpr bool kDiagRemap = MODE == kTriDiag && WARPS_M == 2 && WARPS_N == 4 && MB == 4 && NB == 2;
  // Ragged last tile row (rows 64 (T-1) .. N_G-1, v valid fragment rows of 8): warps w and w + 4
  // (one SM sub-partition) take the two row halves of column block w % 4, so the sub-partitions
  // share the valid rows evenly; each warp runs the k-loop of its first min(4, v - 4 wm) rows.
  constexpr bool kRowRemap = MODE == kTriRow && WARPS_M == 2 && WARPS_N == 4 && MB == 4 && NB == 2;

  uint32_t offL[MB], offR[NB], offK[2];
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) offK[kk] = ((4 * kk + q) ^ pg) << 4;

  // BATCH: the k-slab index of each segment's half-padded last slab (-1: none), hoisted out of
  // the k-loop (evaluated per slab it cost ~9 % of the W producer's issue slots)
  int half_slab[kMaxSeg];
  {
    int end = 0;
#pragma unroll
    for (int s = 0; s < kMaxSeg; ++s) {
      end += s < P.nseg ? P.kchunks[s] : 0;
      half_slab[s] = (s < P.nseg && P.half_last[s]) ? end - 1 : -1;
    }
  }
  // shared-window address of the ring (one generic->shared conversion per kernel, not per k-step)
  // (aligned in the shared window from the symbol's own address: a constant the compiler can
  // rematerialise without reading the window base, SR_SWINHI, inside the loop)
  const uint32_t sring = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sfull = sring + STAGES * Cfg::kStageBytes, sempty = sfull + 8 * STAGES;

  TriSched sched(P.tiles_total, iters, gridDim.x, blockIdx.x);
  Piece pc;
  int bt = blockIdx.x;
  bool have = kTriLike ? sched.next(pc) : bt < P.bat_tiles;
  if (!kTriLike) pc = Piece{bt, 0, iters, 0};
  int it = 0;
  while (have) {
    // this tile's warp tile (wm, wn) and fragment role (0 all, 1 / 2 / 3: the diagonal-tile masks)
    int wm = warp % WARPS_M, wn = warp / WARPS_M, role = 0;
    if (kDiagRemap) {
      {
        // warp -> (wm, wn, role) = w0 (1,0,full) w1 (1,1,full) w2 (0,0,tri7) w3 (1,2,tri7)
        // w4 (0,2,none) w5 (0,3,none) w6 (0,1,tri3) w7 (1,3,tri3); warps w and w + 4 share an SM
        // sub-partition.  Bit-packed tables (an indexed constant array would live in local memory).
        wm = (0x8Bu >> warp) & 1u;
        wn = (0xDE84u >> (2 * warp)) & 3u;
        role = (0xAF50u >> (2 * warp)) & 3u;
      }
    }
    if (kRowRemap) {
      wm = warp >> 2;
      wn = warp & 3;
      const int rows = min(4, max(0, P.row_v - 4 * wm));
      role = rows == 4 ? 0 : 4 + rows;  // 4: none, 5 / 6 / 7: the first 1 / 2 / 3 fragment rows
    }
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) offL[mb] = (wm * Cfg::kWM + 8 * mb + pg) * 128;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) offR[nb] = Cfg::kStageL + (wn * Cfg::kWN + 8 * nb + pg) * 128;  // sub-slab 0
    double acc[MB][NB][2][NS];  // [mb][nb][e][re, im] or [t1, t2, t3]
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int r = 0; r < NS; ++r) acc[mb][nb][e][r] = 0.0;

    // Software-pipelined main loop: the fragments of step s+1 (next kk, or the next
    // stage's first kk) are loaded before the 32 DMMAs of step s issue, so LDS latency
    // and the stage-full wait hide behind the tensor pipe.
    struct Frag {
      double2 a[MB], b[NB];
      double sa[G3M ? MB : 1], sb[G3M ? NB : 1];  // 3M: a_r - a_i, b_r + b_i
    };
    // BATCH: k-slab c is the last of a segment whose length leaves <= 4 valid k in it
    auto half_pad = [&](int c) {
      bool h = false;
#pragma unroll
      for (int s = 0; s < kMaxSeg; ++s) h |= c == half_slab[s];
      return h;
    };
    // The k-loop of one piece for fragment mask M (compile time: the loads, operand sums and
    // DMMAs of fragments outside M are not emitted; a warp with no fragments still takes part in
    // the stage handshake).
    auto kloop = [&](auto maskc) {
      constexpr unsigned M = decltype(maskc)::value;
      auto load_frag = [&](Frag& f, uint32_t st, int u, int kk) {
        const uint32_t base = st + offK[kk];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
          if (row_on(M, mb, NB)) f.a[mb] = lds128(base + u * Cfg::kSubL + offL[mb]);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
          if (col_on(M, nb, MB, NB)) f.b[nb] = lds128(base + u * Cfg::kSubR + offR[nb]);
      };
      // 3M operand sums, formed one step ahead of their use (off the DMMA issue path)
      auto sum_frag = [&](Frag& f) {
        if (G3M) {
#pragma unroll
          for (int mb = 0; mb < MB; ++mb)
            if (row_on(M, mb, NB)) f.sa[mb] = f.a[mb].x - f.a[mb].y;
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
            if (col_on(M, nb, MB, NB)) f.sb[nb] = f.b[nb].x + f.b[nb].y;
        }
      };
      auto mma_frag = [&](const Frag& f) {
        if (G3M) {
          // three independent sweeps (t3, t1, t2) so consecutive DMMAs never share an
          // accumulator; the operand sums were formed one step ahead (sum_frag)
#pragma unroll
          for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
              if (frag_on(M, mb, nb, NB)) dmma(acc[mb][nb][0][NS - 1], acc[mb][nb][1][NS - 1], f.sa[mb], f.sb[nb]);
#pragma unroll
          for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
              if (frag_on(M, mb, nb, NB)) dmma(acc[mb][nb][0][0], acc[mb][nb][1][0], f.a[mb].x, f.b[nb].x);
#pragma unroll
          for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
              if (frag_on(M, mb, nb, NB)) dmma(acc[mb][nb][0][1], acc[mb][nb][1][1], f.a[mb].y, f.b[nb].y);
          return;
        }
        // Four independent sweeps so consecutive DMMAs never share an accumulator.
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
            if (frag_on(M, mb, nb, NB)) dmma(acc[mb][nb][0][0], acc[mb][nb][1][0], f.a[mb].x, f.b[nb].x);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
            if (frag_on(M, mb, nb, NB)) dmma(acc[mb][nb][0][1], acc[mb][nb][1][1], f.a[mb].x, f.b[nb].y);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
            if (frag_on(M, mb, nb, NB)) dmma(acc[mb][nb][0][0], acc[mb][nb][1][0], f.a[mb].y, f.b[nb].y);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb)
#pragma unroll
          for (int nb = 0; nb < NB; ++nb)
            if (frag_on(M, mb, nb, NB)) dmma(acc[mb][nb][0][1], acc[mb][nb][1][1], f.a[mb].y, -f.b[nb].x);
      };
      if (pc.k1 > pc.k0) {
        Frag f0, f1;
        {
          const int slot = it % STAGES;
          mbar_wait_u(sfull + 8 * slot, (it / STAGES) & 1);
          load_frag(f0, sring + slot * Cfg::kStageBytes, 0, 0);
          sum_frag(f0);
        }
        for (int c = pc.k0; c < pc.k1; c += KSUB, ++it) {
          const int n = min(KSUB, pc.k1 - c);
          const int slot = it % STAGES;
          const uint32_t st = sring + slot * Cfg::kStageBytes;
          if (MODE == kBatch && KSUB == 1 && half_pad(c)) {
            // the segment's last slab holds <= 4 valid k: its second half (kk = 1) is TMA
            // zero-fill, so only the first half's DMMAs issue (N_L = 81: 84 of 88 k per segment)
            mma_frag(f0);
            if (c + 1 < pc.k1) {
              const int nslot = (it + 1) % STAGES;
              mbar_wait_u(sfull + 8 * nslot, ((it + 1) / STAGES) & 1);
              load_frag(f0, sring + nslot * Cfg::kStageBytes, 0, 0);
              sum_frag(f0);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_u(sempty + 8 * slot);
            continue;
          }
#pragma unroll
          for (int u = 0; u < KSUB; ++u) {
            if (u < n) {
              load_frag(f1, st, u, 1);
              mma_frag(f0);
              sum_frag(f1);
              // the next step's fragments: sub-slab u+1 of this stage, or the next stage
              const bool more = u + 1 < n || c + KSUB < pc.k1;
              if (u + 1 < n) {
                load_frag(f0, st, u + 1, 0);
              } else if (c + KSUB < pc.k1) {
                const int nslot = (it + 1) % STAGES;
                mbar_wait_u(sfull + 8 * nslot, ((it + 1) / STAGES) & 1);
                load_frag(f0, sring + nslot * Cfg::kStageBytes, 0, 0);
              }
              mma_frag(f1);
              if (more) sum_frag(f0);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_u(sempty + 8 * slot);
        }
      }
    };
    if constexpr (kDiagRemap) {
      if (role == 0)
        kloop(std::integral_constant<unsigned, kMaskFull>{});
      else if (role == 1)
        kloop(std::integral_constant<unsigned, kMaskTri7>{});
      else if (role == 2)
        kloop(std::integral_constant<unsigned, kMaskTri3>{});
      else
        kloop(std::integral_constant<unsigned, kMaskNone>{});
    } else if constexpr (kRowRemap) {
      if (role == 0)
        kloop(std::integral_constant<unsigned, kMaskFull>{});
      else if (role == 5)
        kloop(std::integral_constant<unsigned, 0x03u>{});  // fragment row 0
      else if (role == 6)
        kloop(std::integral_constant<unsigned, 0x0Fu>{});  // rows 0-1
      else if (role == 7)
        kloop(std::integral_constant<unsigned, 0x3Fu>{});  // rows 0-2
      else
        kloop(std::integral_constant<unsigned, kMaskNone>{});
    } else {
      kloop(std::integral_constant<unsigned, (1u << (MB * NB)) - 1u>{});
    }

    if (kTriLike && pc.kind == 2) {
      // contributor: park the partial, publish the flag
      double* ws = P.sk_ws + static_cast<size_t>(blockIdx.x) * NACC * NCT;
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int r = 0; r < NS; ++r)
              __stcg(ws + ((((mb * NB + nb) * 2 + e) * NS + r) * NCT + ctid), acc[mb][nb][e][r]);
      __threadfence();
      consumer_bar(NCT);
      if (ctid == 0) st_release_u32(P.sk_flags + blockIdx.x, P.epoch);
    } else {
      if (kTriLike && pc.kind == 1) {
        // owner: add the later pieces of this tile, in CTA order (deterministic)
        const long long tile_end = static_cast<long long>(pc.tile - sched.dp_tiles + 1) * sched.I;
        for (int b2 = blockIdx.x + 1; b2 < static_cast<int>(gridDim.x) && sched.start(b2) < tile_end; ++b2) {
          if (sched.start(b2 + 1) == sched.start(b2)) continue;  // empty range
          if (ctid == 0)
            while (ld_acquire_u32(P.sk_flags + b2) != P.epoch) __nanosleep(64);
          consumer_bar(NCT);
          const double* ws = P.sk_ws + static_cast<size_t>(b2) * NACC * NCT;
#pragma unroll
          for (int mb = 0; mb < MB; ++mb)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
#pragma unroll
              for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int r = 0; r < NS; ++r)
                  acc[mb][nb][e][r] += __ldcg(ws + ((((mb * NB + nb) * 2 + e) * NS + r) * NCT + ctid));
        }
      }
      // ---- epilogue ---------------------------------------------------------
      int row0, col0, atom;
      tile_origin(pc.tile, row0, col0, atom);
      const double ar = P.alpha_re, ai = P.alpha_im, beta = P.beta;
      const bool keep_di = kTriLike && P.keep_diag_imag != nullptr && *P.keep_diag_imag != 0;
      // destination of accumulator element (mb, nb, e); nullptr outside the output
      auto dst_of = [&](int mb, int nb, int e) -> double2* {
        const int i = row0 + wm * Cfg::kWM + 8 * mb + pg;
        const int j = col0 + wn * Cfg::kWN + 8 * nb + (e ? 4 + q : q);
        if (kTriLike) return (i < P.n && j < P.n && i >= j) ? P.out + (packed_index(P.n, i, j) - P.pk0) : nullptr;
        if (i >= P.m_valid || j >= P.n) return nullptr;
        const int mr = P.m_row ? P.m_row : P.m_valid;
        const bool hi = i >= mr;  // stacked W: rows [m_row, m_valid) are W_B's, in out2
        return (hi ? P.out2 : P.out) + (static_cast<uint64_t>(atom) * mr + (hi ? i - mr : i)) +
               static_cast<uint64_t>(j) * P.ldo;
      };
      // Fold the accumulator sets into (Re, Im) first (3M: frees a third of them).  With
      // beta != 0 the old values are gathered MG row blocks at a time (MG x NB x 2 loads in
      // flight together; all MB at once would exceed the 168 registers ptxas allocates
      // under the 384-thread launch bound), then combined and stored.
      double2 x[MB][NB][2];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            x[mb][nb][e] = G3M ? make_double2(acc[mb][nb][e][0] + acc[mb][nb][e][1],
                                              acc[mb][nb][e][NS - 1] - acc[mb][nb][e][0] + acc[mb][nb][e][1])
                               : make_double2(acc[mb][nb][e][0], acc[mb][nb][e][1]);
      constexpr int MG = MB % 2 == 0 ? 2 : 1;
#pragma unroll
      for (int m0 = 0; m0 < MB; m0 += MG) {
        double2 old[MG][NB][2];
        if (beta != 0.0) {
#pragma unroll
          for (int u = 0; u < MG; ++u)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const double2* d = dst_of(m0 + u, nb, e);
                old[u][nb][e] = d ? __ldcg(d) : make_double2(0.0, 0.0);
              }
        }
#pragma unroll
        for (int u = 0; u < MG; ++u) {
          const int mb = m0 + u;
          const int i = row0 + wm * Cfg::kWM + 8 * mb + pg;
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              double2* d = dst_of(mb, nb, e);
              if (!d) continue;
              const int j = col0 + wn * Cfg::kWN + 8 * nb + (e ? 4 + q : q);
              const double xr = x[mb][nb][e].x, xi = x[mb][nb][e].y;
              double vr = ar * xr - ai * xi;
              double vi = ar * xi + ai * xr;
              if (kTriLike && i == j && !keep_di) vi = 0.0;
              if (beta != 0.0) {
                vr += beta * old[u][nb][e].x;
                vi += beta * old[u][nb][e].y;
              }
              *d = make_double2(vr, vi);
            }
          }
        }
      }
    }
    if (kTriLike) {
      have = sched.next(pc);
    } else {
      bt += gridDim.x;
      have = bt < P.bat_tiles;
      pc = Piece{bt, 0, iters, 0};
    }
  }
  if (P.stamp) {  // the producer warps returned after their last TMA issue
    consumer_bar(NCT);
    if (ctid == 0) stamp_leave(P.stamp);
  }
}

}  // namespace hsdla_b200
