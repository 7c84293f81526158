// Host-side interface to every kernel of libhsdla_b200.so: the contraction engine
// (contract.cu) and the elementwise / batched helpers (elementwise.cu).  Host code
// builds CtnParams blocks and calls these launchers; no other TU launches kernels
// except lapw.cu (LAPW setup) and kernel_layer.cu (its private helpers).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "ctn_params.hpp"

namespace hsdla_b200 {

// ---- contraction engine (contract.cu) ---------------------------------------
// kernel shapes (tools/tune_tri.cu sweep): TRI 64x64 tiles, 8 consumer warps of
// 32x16; BATCH 32x128 tiles, 8 consumer warps of 32x16.
constexpr int kTriBM = 64;
constexpr int kBatBM = 32, kBatBN = 128;
// merged build: ONE BATCH launch W = M Y per atom over the stacked 2 N_L rows
// (W_A; W_B), 24-row tiles (162 rows -> 7 tiles = 168, against 2 x 96 with 32-row tiles)
constexpr int kBatWBM = 24, kBatWBN = 192;  // (or kBatBN = 128 columns when that pads N_G less)
// stream-K partial-accumulator slot per CTA: 64 x 64 outputs x 3 sets (3M) doubles
constexpr uint64_t kSkSlot = uint64_t(kTriBM) * kTriBM * 3;

extern std::atomic<int> g_default_arith;  // hsdla_b200_set_default_arith

// 3-D FP64 tensor map; dims/strides in elements (doubles), box rows of 16 doubles
// (128 B) with the 128-byte swizzle the consumer's LDS.128 pattern expects.
void make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
              uint32_t b1, uint32_t b2);
// Dynamic shared-memory opt-in of the contraction kernels on the current device.
void set_kernel_attributes();
// Launch the TRI (lower-triangular, packed output) / BATCH (per-atom rectangular)
// contraction with arith HSDLA_B200_ARITH_3M / _4M on `s`.
// Returns the number of kernels launched (the strictly-lower and the diagonal launch, or one).
int launch_tri_kernel(int arith, const dim3& grid, const CtnParams& P, cudaStream_t s);
void launch_bat_kernel(int arith, const dim3& grid, const CtnParams& P, cudaStream_t s);
// The W producer with bn = kBatWBN (warp tiles 24 x 24) or kBatBN (24 x 16) output columns per tile.
void launch_batw_kernel(int arith, int bn, const dim3& grid, const CtnParams& P, cudaStream_t s);

inline int chunks_of(uint64_t kcomplex) { return static_cast<int>((kcomplex + kChunkC - 1) / kChunkC); }
// Tile-row band of the TRI tile order (ctn_contract.cuh tri_tile); HSDLA_B200_TRI_BAND
// overrides it for tuning experiments.
int tri_band();

// ---- elementwise / batched helpers (elementwise.cu) ------------------------------
// `stamp` (optional, every launcher): the launch timestamp slot of the engine's phase timing
// (stamp.cuh).  The contraction launchers take it in CtnParams::stamp.  These return whether they
// launched (false for an empty range: the slot was not written).
// X = diag(u) B for rows [0, Kc) of a K-strided stack (kernels.cpp:438-450).
bool launch_diag_scale(const double2* B, const double* u, double2* X, uint64_t Kc, uint64_t ld, uint64_t ng,
                       cudaStream_t s, unsigned long long* stamp = nullptr);
// Counter-based synthetic fill ~ U(lo, hi) (timing sweeps; not the reference generator).
void launch_fill_uniform(double* p, uint64_t n, uint64_t seed, double lo, double hi, unsigned grid, cudaStream_t s);
// Operator expansion from the lower triangles (see elementwise.cu).
// wl != nullptr (merged algorithm): only the stacked left operand of W = M Y is written,
// per atom [Paa | Tab] (k over A rows) then [Pab | Pbb] (k over B rows), 4 N_L^2 complex.
bool launch_expand_hermitian(const double2* taa, const double2* tbb, double2* paa, double2* pbb, int nl,
                             uint64_t total, double bscale, const double2* tab, double2* wl, cudaStream_t s,
                             unsigned long long* stamp = nullptr);
// kernels::potrf for nb blocks (potrf.cuh); n_fail nullable.
bool launch_potrf_batched(const double2* taa, double2* q, int32_t* info, int nl, uint64_t nb, int* n_fail,
                          cudaStream_t s, unsigned long long* stamp = nullptr);
// X2 = info < 0 ? X1 : A, rows [0, Kc) (potrf.cuh).
bool launch_select_left(const double2* X1, const double2* A, const int32_t* info, double2* X2, uint64_t Kc,
                        uint64_t ld, uint64_t ng, int nl, cudaStream_t s, unsigned long long* stamp = nullptr);
// out[i] = sum_r in[r][i] for i in [0, n) (r = 0 .. nin-1 in order; out may alias an input):
// the owner's sum of the partial packed H/S of engines that share one device.
void launch_sum_partials(double2* out, const double2* const* in, int nin, uint64_t n, cudaStream_t s);

}  // namespace hsdla_b200
