// The contraction-engine instantiations (ctn_contract.cuh) and their host launchers.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>

#include "common.hpp"
#include "ctn_contract.cuh"
#include "device.hpp"

namespace hsdla_b200 {

std::atomic<int> g_default_arith{HSDLA_B200_ARITH_3M};

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw Fail{HSDLA_B200_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable"};
  return fn;
}

void make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
              uint32_t b1, uint32_t b2) {
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1 * 8, s2 * 8};
  cuuint32_t box[3] = {16, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Fail{HSDLA_B200_CUDA_ERROR,
               "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")"};
}

constexpr int kTriStages = 8;  // power of two: slot / phase are bit ops in the loop
using TriCfg = CtnCfg<kTri, kTriBM, kTriBM, 2, 4, kTriStages>;
constexpr int kBatStages = 4;
using BatCfg = CtnCfg<kBatch, kBatBM, kBatBN, 1, 8, kBatStages>;
// the merged build's stacked W = M Y producer: 24-row tiles (2 N_L = 162 rows -> 168), 192 or 128
// columns.  (Measured at C2: 1.15 ms per launch with 24 x 192 tiles (warp tiles 24 x 24), 1.18 ms
// with 24 x 128; a single producer warp, which ptxas still compiles against 168 registers since 9
// warps put 3 on one SM sub-partition: 1.19 ms, and 24 x 192 under it spills: 1.44 ms.)
constexpr int kBatWStages = 8;
using BatWCfg = CtnCfg<kBatch, kBatWBM, kBatWBN, 1, 8, kBatWStages>;
static decltype(&ctn_contract_kernel<kBatch, kBatWBM, kBatWBN, 1, 8, kBatWStages>) const batw_kernels[2] = {
    ctn_contract_kernel<kBatch, kBatWBM, kBatWBN, 1, 8, kBatWStages, 1, 1>,
    ctn_contract_kernel<kBatch, kBatWBM, kBatWBN, 1, 8, kBatWStages, 1, 0>};
using BatW128Cfg = CtnCfg<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages>;
static decltype(&ctn_contract_kernel<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages>) const batw128_kernels[2] = {
    ctn_contract_kernel<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages, 1, 1>,
    ctn_contract_kernel<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages, 1, 0>};


// [arith]: HSDLA_B200_ARITH_3M (Gauss, 3 real DMMAs per complex MAC) / _4M (4 DMMAs)
static decltype(&ctn_contract_kernel<kTri, kTriBM, kTriBM, 2, 4, kTriStages>) const tri_kernels[2] = {
    ctn_contract_kernel<kTri, kTriBM, kTriBM, 2, 4, kTriStages, 1, 1>,
    ctn_contract_kernel<kTri, kTriBM, kTriBM, 2, 4, kTriStages, 1, 0>};
static decltype(&ctn_contract_kernel<kBatch, kBatBM, kBatBN, 1, 8, kBatStages>) const bat_kernels[2] = {
    ctn_contract_kernel<kBatch, kBatBM, kBatBN, 1, 8, kBatStages, 1, 1>,
    ctn_contract_kernel<kBatch, kBatBM, kBatBN, 1, 8, kBatStages, 1, 0>};

// diagonal tiles: their own launch with the warp remapping (ctn_contract.cuh kDiagRemap)
static decltype(&ctn_contract_kernel<kTriDiag, kTriBM, kTriBM, 2, 4, kTriStages>) const diag_kernels[2] = {
    ctn_contract_kernel<kTriDiag, kTriBM, kTriBM, 2, 4, kTriStages, 1, 1>,
    ctn_contract_kernel<kTriDiag, kTriBM, kTriBM, 2, 4, kTriStages, 1, 0>};
// a ragged last tile row: its own launch with the row remapping (kRowRemap)
static decltype(&ctn_contract_kernel<kTriRow, kTriBM, kTriBM, 2, 4, kTriStages>) const row_kernels[2] = {
    ctn_contract_kernel<kTriRow, kTriBM, kTriBM, 2, 4, kTriStages, 1, 1>,
    ctn_contract_kernel<kTriRow, kTriBM, kTriBM, 2, 4, kTriStages, 1, 0>};

void set_kernel_attributes() {
  for (int a = 0; a < 2; ++a) {
    HS_CUDA(cudaFuncSetAttribute(tri_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, TriCfg::kSmemBytes));
    HS_CUDA(cudaFuncSetAttribute(diag_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, TriCfg::kSmemBytes));
    HS_CUDA(cudaFuncSetAttribute(row_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, TriCfg::kSmemBytes));
    HS_CUDA(cudaFuncSetAttribute(bat_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, BatCfg::kSmemBytes));
    HS_CUDA(cudaFuncSetAttribute(batw_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, BatWCfg::kSmemBytes));
    HS_CUDA(cudaFuncSetAttribute(batw128_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 BatW128Cfg::kSmemBytes));
  }
}

// One lower-triangular contraction = up to three launches on `s`: the strictly-lower tiles, the
// diagonal tiles (warp-remapped: a diagonal tile costs 10 / 16 of a full one) and, when N_G leaves
// the last tile row with v <= 6 of its 8 fragment rows, that row's tiles (remapped so the valid
// rows are spread over the SM sub-partitions: about v / 8 of a full row).  Small triangles run as
// ONE launch over every lower tile.  P describes the whole set (tiles_total counts the diagonal);
// grid.x bounds every grid.  Each launch gets its own stream-K flag generation (4 epoch + i).
int launch_tri_kernel(int arith, const dim3& grid, const CtnParams& P, cudaStream_t s) {
  int iters = 0;
  for (int sg = 0; sg < P.nseg; ++sg) iters += P.kchunks[sg];
  const int T = P.tiles;
  const int t0 = P.col_t1 > 0 ? P.col_t0 : 0, ndiag = P.col_t1 > 0 ? P.col_t1 - P.col_t0 : T;
  const int nstrict = P.tiles_total - ndiag;
  // launch k (in issue order) stamps slot P.stamp + k * kStampWords
  auto slot = [&](int k) { return P.stamp ? P.stamp + k * kStampWords : nullptr; };
  auto grid_of = [&](int tiles) {
    return dim3(static_cast<unsigned>(std::max<long long>(1, std::min<long long>(grid.x, 1LL * tiles * iters))));
  };
  // A separate diagonal launch saves 6/16 of the diagonal tiles' work, ~0.375 x ndiag x iters
  // k-slabs over the GPU, and costs a launch (~10 us): below ~8000 tile-slabs (C1: 16 x 196) the
  // triangle runs as ONE launch over every lower tile (measured: C1 0.42 ms in one launch, 0.46 split;
  // C2 17.96 -> 17.77 ms split)
  const double split_min = env_double("HSDLA_B200_DIAG_SPLIT_MIN", 8000);  // read per call (tests vary it)
  if (1.0 * ndiag * iters < split_min) {
    CtnParams q = P;
    q.with_diag = 1;
    q.epoch = 4 * P.epoch;
    q.stamp = slot(0);
    tri_kernels[arith]<<<grid_of(P.tiles_total), TriCfg::kThreads, TriCfg::kSmemBytes, s>>>(q);
    HS_CUDA(cudaGetLastError());
    return 1;
  }
  // the ragged last row: tiles (T-1, c) for c in [t0, min(t1, T-1)), v valid fragment rows
  const int v = static_cast<int>((P.n - static_cast<long long>(T - 1) * kTriBM + 7) / 8);
  const int c1 = P.col_t1 > 0 ? std::min(P.col_t1, T - 1) : T - 1;
  // worth its launch when the skipped rows' work, nrow x iters x (8 - v) / 8 k-slabs over the GPU,
  // exceeds ~15 us, and v <= 6 (C2's v = 7 measured 17.79 ms either way)
  const double row_min = env_double("HSDLA_B200_ROW_SPLIT_MIN", 24000);
  const int nrow0 = T >= 2 && v <= 6 ? std::max(0, c1 - t0) : 0;
  const int nrow = 1.0 * nrow0 * iters * (8 - v) >= row_min ? nrow0 : 0;
  int n = 0;
  if (nstrict - nrow > 0) {
    CtnParams q = P;
    q.tiles_total = nstrict - nrow;
    q.with_diag = 0;
    // the whole triangle without its last row: the strictly-lower tiles of the (T-1)-grid (the
    // grouped order interleaves the last rows, so the grid shrinks); a window's last row comes
    // last in its enumeration, so the count alone excludes it
    if (nrow > 0 && P.col_t1 <= 0) q.tiles = T - 1;
    q.epoch = 4 * P.epoch;
    q.stamp = slot(n);
    tri_kernels[arith]<<<grid_of(q.tiles_total), TriCfg::kThreads, TriCfg::kSmemBytes, s>>>(q);
    HS_CUDA(cudaGetLastError());
    ++n;
  }
  if (nrow > 0) {
    CtnParams r = P;
    r.tiles_total = nrow;
    r.row_ti = T - 1;
    r.row_v = v;
    r.diag_t0 = t0;
    r.epoch = 4 * P.epoch + 2;
    r.stamp = slot(n);
    row_kernels[arith]<<<grid_of(nrow), TriCfg::kThreads, TriCfg::kSmemBytes, s>>>(r);
    HS_CUDA(cudaGetLastError());
    ++n;
  }
  CtnParams d = P;
  d.tiles_total = ndiag;
  d.diag_t0 = t0;
  d.epoch = 4 * P.epoch + 1;
  d.stamp = slot(n);
  diag_kernels[arith]<<<grid_of(ndiag), TriCfg::kThreads, TriCfg::kSmemBytes, s>>>(d);
  HS_CUDA(cudaGetLastError());
  return n + 1;
}

void launch_bat_kernel(int arith, const dim3& grid, const CtnParams& P, cudaStream_t s) {
  bat_kernels[arith]<<<grid, BatCfg::kThreads, BatCfg::kSmemBytes, s>>>(P);
  HS_CUDA(cudaGetLastError());
}

void launch_batw_kernel(int arith, int bn, const dim3& grid, const CtnParams& P, cudaStream_t s) {
  if (bn == kBatWBN)
    batw_kernels[arith]<<<grid, BatWCfg::kThreads, BatWCfg::kSmemBytes, s>>>(P);
  else
    batw128_kernels[arith]<<<grid, BatW128Cfg::kThreads, BatW128Cfg::kSmemBytes, s>>>(P);
  HS_CUDA(cudaGetLastError());
}

int tri_band() {
  static int band = [] {
    const char* v = std::getenv("HSDLA_B200_TRI_BAND");
    const int b = v ? std::atoi(v) : 8;
    return b >= 1 ? b : 1;
  }();
  return band;
}

}  // namespace hsdla_b200
