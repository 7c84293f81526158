// LAPW matching-coefficient setup (north_star subsystem 1): host side of the kernels in
// lapw_setup.cuh, the engine's in-HBM setup of A, B, U and the operator-only upload.
#include <cmath>
#include <cstring>
#include <vector>

#include "engine.hpp"
#include "lapw_setup.cuh"

namespace hsdla_b200 {

// ---------------------------------------------------------------------------
// LAPW matching-coefficient setup
// ---------------------------------------------------------------------------
static void check_lapw(const hsdla_b200_lapw* sys) {
  if (!sys || !sys->gvec || !sys->tau || !sys->atom_type || !sys->rmt || !sys->u || !sys->du || !sys->udot ||
      !sys->dudot || !sys->udot_norm)
    throw Fail{HSDLA_B200_DIMENSION_ERROR, "lapw: null pointer"};
  if (sys->n_atoms < 1 || sys->n_types < 1 || sys->n_g < 1 || sys->lmax < 0 || sys->lmax > kLapwMaxL)
    throw Fail{HSDLA_B200_DIMENSION_ERROR, "lapw: need n_atoms, n_types, n_g >= 1 and 0 <= lmax <= 20"};
  if (!(sys->omega > 0.0)) throw Fail{HSDLA_B200_DIMENSION_ERROR, "lapw: omega must be > 0"};
  for (uint64_t a = 0; a < sys->n_atoms; ++a)
    if (sys->atom_type[a] < 0 || static_cast<uint64_t>(sys->atom_type[a]) >= sys->n_types)
      throw Fail{HSDLA_B200_DIMENSION_ERROR, "lapw: atom_type out of range"};
  const int nlv = sys->lmax + 1;
  for (uint64_t t = 0; t < sys->n_types; ++t) {
    if (!(sys->rmt[t] > 0.0)) throw Fail{HSDLA_B200_DIMENSION_ERROR, "lapw: rmt must be > 0"};
    for (int l = 0; l < nlv; ++l) {
      const size_t i = t * nlv + l;
      if (sys->u[i] * sys->dudot[i] - sys->udot[i] * sys->du[i] == 0.0)
        throw Fail{HSDLA_B200_DIMENSION_ERROR, "lapw: singular radial matching system (u udot' - udot u' == 0)"};
    }
  }
}

// Bytes of device scratch the LAPW inputs and per-G tables of `na` atoms need.
static size_t lapw_tables_bytes(const hsdla_b200_lapw* sys, uint64_t na) {
  const size_t nlv = sys->lmax + 1;
  return sys->n_g * (nlv * nlv + sys->n_types * nlv + na) * sizeof(double2);
}
static size_t lapw_inputs_bytes(const hsdla_b200_lapw* sys, uint64_t na) {
  const size_t nlv = sys->lmax + 1;
  return ((sys->n_g * 3 + na * 3 + sys->n_types * nlv * 4 + sys->n_types + sys->n_types * nlv + 4 * nlv * nlv) *
              sizeof(double) +
          ((na * sizeof(int32_t) + 7) & ~size_t(7)) + 255) & ~size_t(255);
}
static size_t lapw_scratch_size(const hsdla_b200_lapw* sys, uint64_t na) {
  return lapw_inputs_bytes(sys, na) + lapw_tables_bytes(sys, na);
}

// Compute A, B (ld = ldo rows) and U for atoms [a0, a0+na) of sys on stream s.
// `scratch` (lapw_scratch_size bytes, device) receives the inputs and the per-G tables.
static void lapw_enqueue(const hsdla_b200_lapw* sys, uint64_t a0, uint64_t na, double2* A, double2* B, uint64_t ldo,
                         double* U, void* scratch, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                         cudaEvent_t ev_mid = nullptr) {
  const int nlv = sys->lmax + 1, nl = nlv * nlv;
  // pack [gvec | tau | radial(u,u',udot,udot') | rmt | udot_norm | ylm coefficients | type] into one host block
  const size_t n_g3 = sys->n_g * 3, n_t3 = na * 3, n_rad = sys->n_types * nlv * 4, n_un = sys->n_types * nlv;
  const size_t n_yc = 4 * static_cast<size_t>(nl);
  std::vector<double> h(n_g3 + n_t3 + n_rad + sys->n_types + n_un + n_yc + (na * sizeof(int32_t) + 7) / 8);
  double* hp = h.data();
  std::memcpy(hp, sys->gvec, n_g3 * sizeof(double));
  std::memcpy(hp + n_g3, sys->tau + 3 * a0, n_t3 * sizeof(double));
  double* rad = hp + n_g3 + n_t3;
  for (uint64_t t = 0; t < sys->n_types; ++t)
    for (int l = 0; l < nlv; ++l) {
      const size_t i = t * nlv + l;
      rad[4 * i + 0] = sys->u[i];
      rad[4 * i + 1] = sys->du[i];
      rad[4 * i + 2] = sys->udot[i];
      rad[4 * i + 3] = sys->dudot[i];
    }
  std::memcpy(rad + n_rad, sys->rmt, sys->n_types * sizeof(double));
  std::memcpy(rad + n_rad + sys->n_types, sys->udot_norm, n_un * sizeof(double));
  ylm_coefficients(sys->lmax, rad + n_rad + sys->n_types + n_un);
  std::memcpy(rad + n_rad + sys->n_types + n_un + n_yc, sys->atom_type + a0, na * sizeof(int32_t));
  HS_CUDA(cudaMemcpyAsync(scratch, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  HS_CUDA(cudaStreamSynchronize(s));  // h is pageable and goes out of scope
  double* d = static_cast<double*>(scratch);
  LapwDevParams P;
  P.gvec = d;
  P.tau = d + n_g3;
  P.radial = d + n_g3 + n_t3;
  P.rmt = d + n_g3 + n_t3 + n_rad;
  const double* d_un = P.rmt + sys->n_types;
  P.ylm_coef = d_un + n_un;
  P.type = reinterpret_cast<const int32_t*>(d_un + n_un + n_yc);
  P.kx = sys->kpt[0];
  P.ky = sys->kpt[1];
  P.kz = sys->kpt[2];
  P.pref = 4.0 * M_PI / std::sqrt(sys->omega);
  P.n_atoms = static_cast<int>(na);
  P.n_types = static_cast<int>(sys->n_types);
  P.lmax = sys->lmax;
  P.n_g = static_cast<int>(sys->n_g);
  P.A = A;
  P.B = B;
  P.ldo = ldo;
  double2* tabY = reinterpret_cast<double2*>(static_cast<char*>(scratch) + lapw_inputs_bytes(sys, na));
  double2* tabF = tabY + sys->n_g * nl;
  double2* tabS = tabF + sys->n_g * sys->n_types * nlv;
  int dev = 0, sms = 148;
  HS_CUDA(cudaGetDevice(&dev));
  HS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t items = sys->n_g * (nlv + sys->n_types + na);
  const unsigned tgrid = static_cast<unsigned>(std::min<uint64_t>((items + 255) / 256, static_cast<uint64_t>(sms) * 16));
  if (ev0) HS_CUDA(cudaEventRecord(ev0, s));
  lapw_tables_kernel<<<tgrid, 256, 0, s>>>(P, tabY, tabF, tabS);
  HS_CUDA(cudaGetLastError());
  if (ev_mid) HS_CUDA(cudaEventRecord(ev_mid, s));
  constexpr int kRows = 4;
  const uint64_t K = na * nl;
  const uint64_t row_blocks = (K + 256 * kRows - 1) / (256 * kRows);
  if (row_blocks > 65535) throw Fail{HSDLA_B200_SIZING_ERROR, "lapw: too many rows (atoms x N_L) per GPU shard"};
  const dim3 sgrid(static_cast<unsigned>(sys->n_g), static_cast<unsigned>(row_blocks));
  lapw_stream_kernel<kRows><<<sgrid, 256, 0, s>>>(P, tabY, tabF, tabS);
  HS_CUDA(cudaGetLastError());
  if (ev1) HS_CUDA(cudaEventRecord(ev1, s));
  const int rows = static_cast<int>(na * nl);
  lapw_u_kernel<<<(rows + 255) / 256, 256, 0, s>>>(P.type, d_un, sys->lmax, static_cast<int>(na), U);
  HS_CUDA(cudaGetLastError());
}

static void engine_setup_lapw(hsdla_b200_engine* e, const hsdla_b200_lapw* sys, uint64_t a0) {
  check_lapw(sys);
  const uint64_t nlv = sys->lmax + 1;
  if (nlv * nlv != e->nl || sys->n_g != e->ng || a0 + e->na > sys->n_atoms)
    throw Fail{HSDLA_B200_DIMENSION_ERROR, "lapw system does not match the engine shard"};
  HS_CUDA(cudaSetDevice(e->device));
  // the engine's operand columns [c0, N_G): the G vectors from c0 on
  hsdla_b200_lapw wsys = *sys;
  wsys.gvec = sys->gvec + 3 * e->c0;
  wsys.n_g = e->ncol;
  sys = &wsys;
  const size_t need = lapw_scratch_size(sys, e->na);
  if (need > e->lapw_scratch_bytes) {
    HS_CUDA(cudaStreamSynchronize(e->stream));
    if (e->lapw_scratch) HS_CUDA(cudaFree(e->lapw_scratch));
    e->lapw_scratch = nullptr;
    e->lapw_scratch_bytes = 0;
    HS_CUDA(cudaMalloc(&e->lapw_scratch, need));
    e->lapw_scratch_bytes = need;
  }
  lapw_enqueue(sys, a0, e->na, e->A(0), e->B(0), e->K, e->U, e->lapw_scratch, e->stream, e->ev_setup0,
               e->ev_setup1, e->ev_setup_mid);
  e->setup_bytes = 2 * e->K * e->ncol * sizeof(double2);
}

static void engine_upload_operators(hsdla_b200_engine* e, const double* taa, const double* tab, const double* tbb,
                                    uint64_t a0) {
  if (!taa || !tab || !tbb) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null operator pointer"};
  HS_CUDA(cudaSetDevice(e->device));
  const uint64_t blk = e->nl * e->nl;
  const size_t bytes = e->na * blk * sizeof(double2);
  // on the copy stream, so the next build's S contraction (which needs no operator) runs
  // while they travel; the build waits for ev_ops before its operator expansion
  cudaStream_t cs = e->copy_stream;
  // after everything already on the compute stream: the previous build (done with T) and any
  // earlier upload into T (engine_upload copies on the compute stream; a pageable copy may still
  // be in flight when it returns, and landing after this one would restore the old operators)
  copy_after_compute(e);
  HS_CUDA(cudaMemcpyAsync(e->Taa, reinterpret_cast<const double2*>(taa) + a0 * blk, bytes, cudaMemcpyHostToDevice, cs));
  HS_CUDA(cudaMemcpyAsync(e->Tab, reinterpret_cast<const double2*>(tab) + a0 * blk, bytes, cudaMemcpyHostToDevice, cs));
  HS_CUDA(cudaMemcpyAsync(e->Tbb, reinterpret_cast<const double2*>(tbb) + a0 * blk, bytes, cudaMemcpyHostToDevice, cs));
  HS_CUDA(cudaEventRecord(e->ev_ops, cs));
  e->ops_pending = true;
}

}  // namespace hsdla_b200

using namespace hsdla_b200;

extern "C" {

int hsdla_b200_lapw_coefficients(int device, const hsdla_b200_lapw* sys, double* A, double* B, double* U) {
  return guarded([&] {
    check_lapw(sys);
    if (!A || !B || !U) throw Fail{HSDLA_B200_DIMENSION_ERROR, "null output"};
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
      (void)cudaGetLastError();
      throw Fail{HSDLA_B200_CONFIG_ERROR, "no such CUDA device (the B200 path has no CPU fallback)"};
    }
    HS_CUDA(cudaSetDevice(device));
    const uint64_t nlv = sys->lmax + 1, K = sys->n_atoms * nlv * nlv;
    check_dims(sys->n_atoms, nlv * nlv, sys->n_g);
    struct Buf {
      void* p = nullptr;
      ~Buf() {
        if (p) cudaFree(p);
      }
    } dA, dB, dU, dS;
    HS_CUDA(cudaMalloc(&dS.p, lapw_scratch_size(sys, sys->n_atoms)));
    HS_CUDA(cudaMalloc(&dA.p, K * sys->n_g * sizeof(double2)));
    HS_CUDA(cudaMalloc(&dB.p, K * sys->n_g * sizeof(double2)));
    HS_CUDA(cudaMalloc(&dU.p, K * sizeof(double)));
    cudaStream_t s = 0;
    lapw_enqueue(sys, 0, sys->n_atoms, static_cast<double2*>(dA.p), static_cast<double2*>(dB.p), K,
                 static_cast<double*>(dU.p), dS.p, s, nullptr, nullptr);
    HS_CUDA(cudaMemcpy(A, dA.p, K * sys->n_g * sizeof(double2), cudaMemcpyDeviceToHost));
    HS_CUDA(cudaMemcpy(B, dB.p, K * sys->n_g * sizeof(double2), cudaMemcpyDeviceToHost));
    HS_CUDA(cudaMemcpy(U, dU.p, K * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int hsdla_b200_engine_setup_lapw(hsdla_b200_engine* e, const hsdla_b200_lapw* sys, uint64_t atom_begin) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_setup_lapw(e, sys, atom_begin);
  });
}

int hsdla_b200_engine_upload_operators(hsdla_b200_engine* e, const double* T_AA, const double* T_AB,
                                       const double* T_BB, uint64_t atom_begin) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    engine_upload_operators(e, T_AA, T_AB, T_BB, atom_begin);
  });
}

int hsdla_b200_engine_setup_time(hsdla_b200_engine* e, double* ms, uint64_t* bytes, double* ms_stream) {
  return guarded([&] {
    if (!e) throw Fail{HSDLA_B200_CONFIG_ERROR, "null engine"};
    if (!e->setup_bytes) throw Fail{HSDLA_B200_CONFIG_ERROR, "no setup_lapw has run"};
    HS_CUDA(cudaEventSynchronize(e->ev_setup1));
    if (ms) *ms = ev_ms(e->ev_setup0, e->ev_setup1);
    if (ms_stream) *ms_stream = ev_ms(e->ev_setup_mid, e->ev_setup1);
    if (bytes) *bytes = e->setup_bytes;
  });
}

}  // extern "C"
