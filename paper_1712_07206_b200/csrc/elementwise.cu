// Elementwise (HBM-bound) and batched helper kernels of the engine, with their host
// launchers (declared in device.hpp).
#include "common.hpp"
#include "device.hpp"
#include "potrf.cuh"
#include "stamp.cuh"

namespace hsdla_b200 {

// ---------------------------------------------------------------------------
// elementwise kernels (HBM-bound)
// ---------------------------------------------------------------------------

// X = diag(u) B for rows [0, Kc) of a K-strided stack (kernels.cpp:438-450);
// coalesced along K, columns strided over blockIdx.y.
static __global__ void diag_scale_kernel(const double2* __restrict__ B, const double* __restrict__ u,
                                  double2* __restrict__ X, uint64_t Kc, uint64_t ld, uint64_t ng,
                                  unsigned long long* stamp) {
  stamp_enter(stamp);
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < Kc) {
    const double s = u[k];
    for (uint64_t j = blockIdx.y; j < ng; j += gridDim.y) {
      const double2 b = B[k + j * ld];
      X[k + j * ld] = make_double2(s * b.x, s * b.y);
    }
  }
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) stamp_leave(stamp);
  }
}

// Counter-based synthetic fill (splitmix64 of (seed, index)) -> U(lo, hi): device-side
// inputs for the large-N scaling sweep, where host generation of 10-50 GB would
// dominate.  Not the reference generator (generate_problem is bit-identical on the
// host); contraction timing does not depend on the values.
static __global__ void fill_uniform_kernel(double* __restrict__ p, uint64_t n, uint64_t seed, double lo, double hi) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ULL + i + 0x632BE59BD9B4E019ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    p[i] = lo + (hi - lo) * static_cast<double>(z >> 11) * 0x1.0p-53;
  }
}

// Left operands P with P^H = the reference's hemm operator, from the LOWER triangle
// only (kernels.cpp:152-167 uses h(i,l) for l <= i — the diagonal as stored — and
// conj(h(l,i)) for l > i).  The contraction computes P^H R, so
//   P(k,i) = conj(T(i,k)) for k <= i,  T(k,i) for k > i
// (= full(T) with the diagonal conjugated; identical for a real diagonal).
//   Pbb[a] = bscale * P(T_BB[a]),  Paa[a] = P(T_AA[a])  (bscale 1/2)
// Merged algorithm (wl != nullptr): the stacked left operand of W = M Y per atom instead,
//   wl[a] = [Paa | Tab] then [Pab | Pbb]  (column i of each N_L x 2 N_L half holds k = 0 .. N_L-1)
// with Pab(k, i) = conj(T_AB(i, k)) (Pab^H B = T_AB B) and Pbb = full(T_BB) (bscale 1).
static __device__ __forceinline__ void expand_one(const double2* __restrict__ taa, const double2* __restrict__ tbb,
                                                  double2* __restrict__ paa, double2* __restrict__ pbb, int nl,
                                                  double bscale, const double2* __restrict__ tab,
                                                  double2* __restrict__ wl, uint64_t idx);
static __global__ void expand_hermitian_kernel(const double2* __restrict__ taa, const double2* __restrict__ tbb,
                                        double2* __restrict__ paa, double2* __restrict__ pbb, int nl,
                                        uint64_t total, double bscale, const double2* __restrict__ tab,
                                        double2* __restrict__ wl, unsigned long long* stamp) {
  stamp_enter(stamp);
  const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < total) expand_one(taa, tbb, paa, pbb, nl, bscale, tab, wl, idx);
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) stamp_leave(stamp);
  }
}
static __device__ __forceinline__ void expand_one(const double2* __restrict__ taa, const double2* __restrict__ tbb,
                                                  double2* __restrict__ paa, double2* __restrict__ pbb, int nl,
                                                  double bscale, const double2* __restrict__ tab,
                                                  double2* __restrict__ wl, uint64_t idx) {
  const uint64_t blk = static_cast<uint64_t>(nl) * nl;
  const uint64_t a = idx / blk;
  const int r = static_cast<int>(idx - a * blk);
  const int k = r % nl, i = r / nl;  // element (k, i) of the column-major block
  const uint64_t lo =
      a * blk + (k >= i ? (k + static_cast<uint64_t>(i) * nl) : (i + static_cast<uint64_t>(k) * nl));
  double2 vaa = taa[lo], vbb = tbb[lo];
  if (k <= i) {
    vaa.y = -vaa.y;
    vbb.y = -vbb.y;
  }
  if (!wl) {
    paa[idx] = vaa;
    pbb[idx] = make_double2(bscale * vbb.x, bscale * vbb.y);
    return;
  }
  // merged: B^H T_BB B stands for the reference's Z^H B + B^H Z share
  // 1/2 B^H (T_BB + T_BB^H) B (hemm reads T_BB's diagonal as stored, kernels.cpp:152-167),
  // i.e. T_BB with its diagonal's imaginary part dropped
  if (k == i) vbb.y = 0.0;
  const double2 v = tab[a * blk + i + static_cast<uint64_t>(k) * nl];
  double2* w = wl + 4 * a * blk + k;
  w[static_cast<uint64_t>(i) * nl] = vaa;                      // [Paa | .]
  w[static_cast<uint64_t>(nl + i) * nl] = tab[idx];            // [. | Tab]
  w[2 * blk + static_cast<uint64_t>(i) * nl] = make_double2(v.x, -v.y);  // [Pab | .]
  w[2 * blk + static_cast<uint64_t>(nl + i) * nl] = make_double2(bscale * vbb.x, bscale * vbb.y);  // [. | Pbb]
}

// out[i] = sum_r in[r][i], ranks in order (bitwise deterministic); out may alias one of
// the inputs (each element is read from every input before it is written).
constexpr int kMaxSumIn = 16;
struct SumIn {
  const double2* p[kMaxSumIn];
};
__global__ void sum_partials_kernel(double2* __restrict__ out, const SumIn in, int nin, uint64_t n) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double2 acc = in.p[0][i];
    for (int r = 1; r < nin; ++r) {
      const double2 v = in.p[r][i];
      acc.x += v.x;
      acc.y += v.y;
    }
    out[i] = acc;
  }
}

bool launch_diag_scale(const double2* B, const double* u, double2* X, uint64_t Kc, uint64_t ld, uint64_t ng,
                       cudaStream_t s, unsigned long long* stamp) {
  if (!Kc || !ng) return false;
  const dim3 g(static_cast<unsigned>((Kc + 255) / 256), static_cast<unsigned>(std::min<uint64_t>(ng, 2048)));
  diag_scale_kernel<<<g, 256, 0, s>>>(B, u, X, Kc, ld, ng, stamp);
  HS_CUDA(cudaGetLastError());
  return true;
}

void launch_fill_uniform(double* p, uint64_t n, uint64_t seed, double lo, double hi, unsigned grid, cudaStream_t s) {
  fill_uniform_kernel<<<grid, 256, 0, s>>>(p, n, seed, lo, hi);
  HS_CUDA(cudaGetLastError());
}

bool launch_expand_hermitian(const double2* taa, const double2* tbb, double2* paa, double2* pbb, int nl,
                             uint64_t total, double bscale, const double2* tab, double2* wl, cudaStream_t s,
                             unsigned long long* stamp) {
  if (!total) return false;
  expand_hermitian_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(taa, tbb, paa, pbb, nl, total,
                                                                                      bscale, tab, wl, stamp);
  HS_CUDA(cudaGetLastError());
  return true;
}

bool launch_potrf_batched(const double2* taa, double2* q, int32_t* info, int nl, uint64_t nb, int* n_fail,
                          cudaStream_t s, unsigned long long* stamp) {
  if (!nb) return false;
  potrf_batched_kernel<<<static_cast<unsigned>(nb), 128, 0, s>>>(taa, q, info, nl, n_fail, stamp);
  HS_CUDA(cudaGetLastError());
  return true;
}

bool launch_select_left(const double2* X1, const double2* A, const int32_t* info, double2* X2, uint64_t Kc,
                        uint64_t ld, uint64_t ng, int nl, cudaStream_t s, unsigned long long* stamp) {
  if (!Kc || !ng) return false;
  const dim3 g(static_cast<unsigned>((Kc + 255) / 256), static_cast<unsigned>(std::min<uint64_t>(ng, 2048)));
  select_left_kernel<<<g, 256, 0, s>>>(X1, A, info, X2, Kc, ld, ng, nl, stamp);
  HS_CUDA(cudaGetLastError());
  return true;
}

void launch_sum_partials(double2* out, const double2* const* in, int nin, uint64_t n, cudaStream_t s) {
  if (!n || nin < 1) return;
  if (nin > kMaxSumIn) throw Fail{HSDLA_B200_CONFIG_ERROR, "more than 16 engines share one device"};
  int dev = 0, sms = 148;
  HS_CUDA(cudaGetDevice(&dev));
  HS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sms) * 8));
  SumIn a{};
  for (int r = 0; r < nin; ++r) a.p[r] = in[r];
  sum_partials_kernel<<<grid, 256, 0, s>>>(out, a, nin, n);
  HS_CUDA(cudaGetLastError());
}

}  // namespace hsdla_b200
