// Development harness: times TRI-mode contraction configs on a C2-sized S product
// (2 segments, K = 5184, N_G = 3000) with random data.  Not part of the product.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>
#include "../paper_1712_07206_b200/csrc/ctn_contract.cuh"
using namespace hsdla_b200;

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static std::vector<double> ref3m;  // first 3M variant's output (all 3M variants must match it bitwise)
static void make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                     uint64_t s2, uint32_t b1, uint32_t b2) {
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1 * 8, s2 * 8};
  cuuint32_t box[3] = {16, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) { printf("encode failed %d\n", r); exit(1); }
}

__global__ void fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995; x ^= x >> 15;
    p[i] = (x & 0xffffff) / 16777216.0 - 0.5;
  }
}

template <int BM, int WM, int WN, int ST, int MINB, int G3M = 0, int KSUB = 1>
void run(const char* name, double2* A, double2* B, double2* out, uint64_t K, uint64_t ng, int nseg) {
  using Cfg = CtnCfg<kTri, BM, BM, WM, WN, ST, KSUB>;
  auto kern = ctn_contract_kernel<kTri, BM, BM, WM, WN, ST, MINB, G3M, KSUB>;       // strictly-lower tiles
  auto dkern = ctn_contract_kernel<kTriDiag, BM, BM, WM, WN, ST, MINB, G3M, KSUB>;  // diagonal tiles
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
  cudaFuncSetAttribute(dkern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
  CtnParams P;
  memset(&P, 0, sizeof(P));
  CUtensorMap mA, mB;
  make_map(&mA, A, 2 * K, ng, 1, 2 * K, 2 * K * ng, BM, 1);
  make_map(&mB, B, 2 * K, ng, 1, 2 * K, 2 * K * ng, BM, 1);
  for (int s = 0; s < nseg; ++s) {
    P.L[s] = (s & 1) ? mB : mA;
    P.R[s] = (s & 1) ? mA : mB;
    P.kchunks[s] = (int)((K + 7) / 8);
  }
  P.nseg = nseg;
  P.n = (int)ng;
  int tiles = (int)((ng + BM - 1) / BM);
  P.tiles = tiles;
  P.tiles_total = tiles * (tiles - 1) / 2;  // kTri launch (with_diag 0): strictly lower; the kTriDiag launch: `tiles`
  P.band = 8;
  P.out = out;
  P.alpha_re = 1.0;
  static double* ws = nullptr;
  static uint32_t* flags = nullptr;
  if (!ws) {
    cudaMalloc(&ws, 4 * 148ull * 128 * 128 * 2 * 8);
    cudaMalloc(&flags, 4 * 148 * 4);
    cudaMemset(flags, 0, 4 * 148 * 4);
  }
  P.sk_ws = ws;
  P.sk_flags = flags;
  static uint32_t epoch = 0;
  const char* gs = getenv("TUNE_GRID");  // fewer persistent CTAs than SMs (memory-system probe)
  int grid = gs ? atoi(gs) : 148 * MINB;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::kThreads, Cfg::kSmemBytes);
  auto launch2 = [&] {
    CtnParams d = P;
    d.tiles_total = tiles;
    d.diag_t0 = 0;
    d.epoch = P.epoch | 0x40000000u;
    static const char* only = getenv("TUNE_ONLY");  // "strict" | "diag": one of the two launches
    if (!only || only[0] != 'd') kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(P);
    if (!only || only[0] != 's') dkern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(d);
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  P.epoch = ++epoch;
  launch2();
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    P.epoch = ++epoch;
    launch2();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaError_t err = cudaGetLastError();
  double flops = 4.0 * nseg * K * (double)ng * ng;
  // bitwise comparison against the first 3M variant's output (same sums, same DMMA order)
  std::vector<double> h(ng * (ng + 1));
  cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
  size_t ndiff = 0;
  if (G3M) {
    if (ref3m.empty()) ref3m = h;
    for (size_t i = 0; i < h.size(); ++i) ndiff += h[i] != ref3m[i];
  }
#ifdef HSDLA_EXP_TILE_CLOCK
  {  // per-tile SM clocks of the last launch (tools/tile_clock.patch): whole tiles only
    static long long h[148][64][4];
    cudaMemcpyFromSymbol(h, g_tclk, sizeof(h));
    double kl = 0, ep = 0, gap = 0;
    int nt = 0, ng2 = 0;
    for (int b = 0; b < 148; ++b)
      for (int i = 0; i < 64; ++i) {
        if (h[b][i][0] == 0 || h[b][i][2] < h[b][i][0]) break;
        if (h[b][i][3] / 100000000LL != 0) continue;
        kl += h[b][i][1] - h[b][i][0];
        ep += h[b][i][2] - h[b][i][1];
        ++nt;
        if (i + 1 < 64 && h[b][i + 1][0] > h[b][i][2]) {
          gap += h[b][i + 1][0] - h[b][i][2];
          ++ng2;
        }
      }
    printf("  per whole tile (%d tiles, %d k-slabs): k-loop %.0f clk, epilogue %.0f clk, gap %.0f clk\n", nt,
           2 * (int)((K + 7) / 8), kl / nt, ep / nt, ng2 ? gap / ng2 : 0.0);
  }
#endif
  printf("%-34s occ %d grid %6d  %8.3f ms  %6.2f TF/s(ledger)  diff-vs-3M %zu  %s\n", name, occ, grid, best,
         flops / best / 1e9, ndiff, err ? cudaGetErrorString(err) : "");
}

int main(int argc, char** argv) {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  uint64_t K = argc > 1 ? atoll(argv[1]) : 5184, ng = argc > 2 ? atoll(argv[2]) : 3000;
  int nseg = argc > 3 ? atoi(argv[3]) : 2;
  double2 *A, *B, *out;
  cudaMalloc(&A, K * ng * 16); cudaMalloc(&B, K * ng * 16); cudaMalloc(&out, ng * (ng + 1) / 2 * 16);
  fill<<<1024, 256>>>((double*)A, 2 * K * ng, 1);
  fill<<<1024, 256>>>((double*)B, 2 * K * ng, 2);
  printf("K %lu N_G %lu nseg %d\n", K, ng, nseg);
  run<64, 2, 4, 8, 1, 0, 1>("4M st8 ksub1", A, B, out, K, ng, nseg);
  run<64, 2, 4, 4, 1, 0, 2>("4M st4 ksub2", A, B, out, K, ng, nseg);
  run<64, 2, 4, 8, 1, 1, 1>("3M st8 ksub1 [current]", A, B, out, K, ng, nseg);
  run<64, 2, 4, 4, 1, 1, 2>("3M st4 ksub2", A, B, out, K, ng, nseg);
  run<64, 2, 4, 8, 1, 1, 1>("3M st8 ksub1 [current]", A, B, out, K, ng, nseg);
  return 0;
}
