// Development harness: times the merged build's W producer ([W_A; W_B] = M_a [A_a; B_a], the
// stacked BATCH launch of engine.cpp make_chunk) on synthetic data.  Not part of the product.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//        -o tune_batw tune_batw.cu -lcuda
//   ./tune_batw [n_atoms] [n_l] [n_g]                      (default: C2, 64 81 3000)
//
// With the per-tile clock instrumentation (tools/tile_clock.patch applied to a copy of
// ctn_contract.cuh, -DHSDLA_EXP_TILE_CLOCK -I<that copy>) it also prints the mean k-loop,
// epilogue and inter-tile gap per tile in SM cycles.
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ctn_contract.cuh"
using namespace hsdla_b200;

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static void make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                     uint64_t s2, uint32_t b1, uint32_t b2) {
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1 * 8, s2 * 8};
  cuuint32_t box[3] = {16, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) {
    printf("encode failed %d\n", r);
    exit(1);
  }
}

__global__ void fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995;
    x ^= x >> 15;
    p[i] = (x & 0xffffff) / 16777216.0 - 0.5;
  }
}

#ifdef HSDLA_EXP_TILE_CLOCK
static void tile_report() {
  static long long h[148][64][4];
  cudaMemcpyFromSymbol(h, g_tclk, sizeof(h));
  double kl = 0, ep = 0, gap = 0;
  int n = 0, ng = 0;
  for (int b = 0; b < 148; ++b)
    for (int i = 0; i < 64; ++i) {
      if (h[b][i][0] == 0 || h[b][i][2] < h[b][i][0]) break;
      kl += h[b][i][1] - h[b][i][0];
      ep += h[b][i][2] - h[b][i][1];
      ++n;
      if (i + 1 < 64 && h[b][i + 1][0] > h[b][i][2]) {
        gap += h[b][i + 1][0] - h[b][i][2];
        ++ng;
      }
    }
  printf("  per tile (%d tiles, %lld k-slabs): k-loop %.0f clk, epilogue %.0f clk, gap %.0f clk\n", n,
         h[0][0][3] % 100000000LL, kl / n, ep / n, ng ? gap / ng : 0.0);
}
#endif

template <int BN, int ST = 8, int KSUB = 1>
static void run(uint64_t na, uint64_t nl, uint64_t ng) {
  constexpr int BM = 24, PW = 4;
  using Cfg = CtnCfg<kBatch, BM, BN, 1, 8, ST, KSUB, PW>;
  auto kern = ctn_contract_kernel<kBatch, BM, BN, 1, 8, ST, 1, 1, KSUB, PW>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
  const uint64_t K = na * nl, blk = nl * nl;
  double2 *A, *B, *Wl, *X1, *X2;
  cudaMalloc(&A, K * ng * 16);
  cudaMalloc(&B, K * ng * 16);
  cudaMalloc(&Wl, 4 * na * blk * 16);
  cudaMalloc(&X1, K * ng * 16);
  cudaMalloc(&X2, K * ng * 16);
  fill<<<1024, 256>>>((double*)A, 2 * K * ng, 1);
  fill<<<1024, 256>>>((double*)B, 2 * K * ng, 2);
  fill<<<1024, 256>>>((double*)Wl, 8 * na * blk, 3);
  CtnParams P;
  std::memset(&P, 0, sizeof(P));
  // the same maps as engine.cpp make_chunk (cp.w)
  make_map(&P.L[0], Wl, 2 * nl, 2 * nl, na, 2 * nl, 8 * blk, BM, 1);
  make_map(&P.L[1], Wl + 2 * blk, 2 * nl, 2 * nl, na, 2 * nl, 8 * blk, BM, 1);
  make_map(&P.R[0], A, 2 * nl, na, ng, 2 * nl, 2 * K, 1, BN);
  make_map(&P.R[1], B, 2 * nl, na, ng, 2 * nl, 2 * K, 1, BN);
  P.kchunks[0] = P.kchunks[1] = static_cast<int>((nl + 7) / 8);
  P.half_last[0] = P.half_last[1] = nl % 8 >= 1 && nl % 8 <= 4;
  P.r_row_z[0] = P.r_row_z[1] = 1;
  P.nseg = 2;
  P.n = static_cast<int>(ng);
  P.m_valid = static_cast<int>(2 * nl);
  P.m_row = static_cast<int>(nl);
  P.out = X1;
  P.out2 = X2;
  P.ldo = K;
  P.alpha_re = 1.0;
  P.bat_tx = static_cast<int>((ng + BN - 1) / BN);
  P.bat_ty = static_cast<int>((2 * nl + BM - 1) / BM);
  P.bat_tiles = P.bat_tx * P.bat_ty * static_cast<int>(na);
  const char* g = getenv("TUNE_GRID");  // fewer persistent CTAs than SMs (L2-bandwidth probe)
  const dim3 grid(static_cast<unsigned>(std::min(P.bat_tiles, g ? atoi(g) : 148)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(P);
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(P);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaError_t err = cudaGetLastError();
  // useful flops at 6 per complex MAC (3M): (2 N_L)^2 N_G per atom
  const double useful = 6.0 * 4.0 * nl * nl * ng * na;
  printf("W 24x%d stages %d ksub %d: %d tiles  %.3f ms  useful %.2f TF/s (%.3f of 37.0)  %s\n", BN, ST, KSUB,
         P.bat_tiles, best,
         useful / best / 1e9, useful / best / 1e9 / 37.0, err ? cudaGetErrorString(err) : "");
  {  // bitwise comparison against the first variant's output
    static std::vector<double> ref;
    std::vector<double> h(2 * K * ng);
    cudaMemcpy(h.data(), X1, h.size() * 8, cudaMemcpyDeviceToHost);
    if (ref.empty()) ref = h;
    size_t nd = 0;
    for (size_t i = 0; i < h.size(); ++i) nd += h[i] != ref[i];
    printf("  differing elements vs the first variant: %zu\n", nd);
  }
#ifdef HSDLA_EXP_TILE_CLOCK
  tile_report();
#endif
  for (void* p : {(void*)A, (void*)B, (void*)Wl, (void*)X1, (void*)X2}) cudaFree(p);
}

int main(int argc, char** argv) {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const uint64_t na = argc > 1 ? atoll(argv[1]) : 64, nl = argc > 2 ? atoll(argv[2]) : 81,
                 ng = argc > 3 ? atoll(argv[3]) : 3000;
  printf("N_A %lu N_L %lu N_G %lu\n", na, nl, ng);
  run<192>(na, nl, ng);
  run<128>(na, nl, ng);
  if (getenv("TUNE_VARIANTS")) {
    run<192, 6>(na, nl, ng);
    run<192, 7>(na, nl, ng);
    run<192, 4, 2>(na, nl, ng);
    run<128, 6, 2>(na, nl, ng);
  }
  return 0;
}
