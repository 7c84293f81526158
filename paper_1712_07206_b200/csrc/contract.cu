// The contraction-engine instantiations (ctn_contract.cuh) and their host launchers.
#include <cudaTypedefs.h>

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
// the merged build's stacked W = M Y producer: 24-row tiles (2 N_L = 162 rows -> 168).
// (Measured at C2: 1.18 ms per launch; 24 x 192 tiles with warp tiles 24 x 24: 1.15 ms; a
// single producer warp, which ptxas still compiles against 168 registers since 9 warps put
// 3 on one SM sub-partition: 1.19 ms, and 24 x 192 under it spills: 1.44 ms.)
constexpr int kBatWStages = 8;
using BatWCfg = CtnCfg<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages>;
static decltype(&ctn_contract_kernel<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages>) const batw_kernels[2] = {
    ctn_contract_kernel<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages, 1, 1>,
    ctn_contract_kernel<kBatch, kBatWBM, kBatBN, 1, 8, kBatWStages, 1, 0>};


// [arith]: HSDLA_B200_ARITH_3M (Gauss, 3 real DMMAs per complex MAC) / _4M (4 DMMAs)
static decltype(&ctn_contract_kernel<kTri, kTriBM, kTriBM, 2, 4, kTriStages>) const tri_kernels[2] = {
    ctn_contract_kernel<kTri, kTriBM, kTriBM, 2, 4, kTriStages, 1, 1>,
    ctn_contract_kernel<kTri, kTriBM, kTriBM, 2, 4, kTriStages, 1, 0>};
static decltype(&ctn_contract_kernel<kBatch, kBatBM, kBatBN, 1, 8, kBatStages>) const bat_kernels[2] = {
    ctn_contract_kernel<kBatch, kBatBM, kBatBN, 1, 8, kBatStages, 1, 1>,
    ctn_contract_kernel<kBatch, kBatBM, kBatBN, 1, 8, kBatStages, 1, 0>};

void set_kernel_attributes() {
  for (int a = 0; a < 2; ++a) {
    HS_CUDA(cudaFuncSetAttribute(tri_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, TriCfg::kSmemBytes));
    HS_CUDA(cudaFuncSetAttribute(bat_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, BatCfg::kSmemBytes));
    HS_CUDA(cudaFuncSetAttribute(batw_kernels[a], cudaFuncAttributeMaxDynamicSharedMemorySize, BatWCfg::kSmemBytes));
  }
}

void launch_tri_kernel(int arith, const dim3& grid, const CtnParams& P, cudaStream_t s) {
  tri_kernels[arith]<<<grid, TriCfg::kThreads, TriCfg::kSmemBytes, s>>>(P);
  HS_CUDA(cudaGetLastError());
}

void launch_bat_kernel(int arith, const dim3& grid, const CtnParams& P, cudaStream_t s) {
  bat_kernels[arith]<<<grid, BatCfg::kThreads, BatCfg::kSmemBytes, s>>>(P);
  HS_CUDA(cudaGetLastError());
}

void launch_batw_kernel(int arith, const dim3& grid, const CtnParams& P, cudaStream_t s) {
  batw_kernels[arith]<<<grid, BatWCfg::kThreads, BatWCfg::kSmemBytes, s>>>(P);
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
