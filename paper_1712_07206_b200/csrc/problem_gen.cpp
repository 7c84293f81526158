// Synthetic problem generator: hsdla::generate_problem (reference
// proj/src/problem.cpp:79-142) re-implemented for the C-ABI.  Bit-identical to
// the reference by construction: std::mt19937_64 has a standard-specified output
// sequence and the double mapping below is the reference's (problem.cpp:13-24);
// tests/test_host.py pins it against the golden fixtures.
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/hsdla_b200.h"

namespace hsdla_b200 {
extern thread_local std::string g_last_error;
}

namespace {

using cplx = std::complex<double>;

struct Rng {
  explicit Rng(uint64_t seed) : eng(seed) {}
  double uniform01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  cplx symmetric() {
    const double re = uniform(-1.0, 1.0);
    const double im = uniform(-1.0, 1.0);
    return {re, im};
  }
  std::mt19937_64 eng;
};

void fill(cplx* m, uint64_t n, Rng& rng) {
  for (uint64_t i = 0; i < n; ++i) m[i] = rng.symmetric();
}

// Largest eigenvalue of Hermitian PSD g by 50 power iterations (problem.cpp:50-69).
double lambda_max(const cplx* g, uint64_t n) {
  std::vector<cplx> v(n, cplx(1.0, 0.0)), w(n);
  double lambda = 0.0;
  for (int it = 0; it < 50; ++it) {
    for (uint64_t i = 0; i < n; ++i) {
      cplx s = 0.0;
      for (uint64_t j = 0; j < n; ++j) s += g[i + j * n] * v[j];
      w[i] = s;
    }
    double norm = 0.0;
    for (uint64_t i = 0; i < n; ++i) norm += std::norm(w[i]);
    norm = std::sqrt(norm);
    if (norm == 0.0) break;
    lambda = norm;
    for (uint64_t i = 0; i < n; ++i) v[i] = w[i] / norm;
  }
  return lambda;
}

// The generator stream restricted to atoms [lo, hi): A and B rows of those atoms (leading
// dimension (hi - lo) n_l), their operator blocks, U and hpd flags.  Draws of other atoms are
// skipped (discarded), so the output is bit-identical to the same rows of a full generation.
void generate(uint64_t na, uint64_t nl, uint64_t ng, uint64_t seed, uint64_t n_not_hpd, uint64_t lo, uint64_t hi,
              double* A, double* B, double* T_AA, double* T_AB, double* T_BB, double* U, uint8_t* hpd) {
  Rng rng(seed);
  const uint64_t K = na * nl, blk = nl * nl, r0 = lo * nl, r1 = hi * nl, Ks = r1 - r0;
  for (double* M : {A, B}) {  // column-major K x N_G, each complex = 2 draws (problem.cpp:97-98)
    cplx* m = reinterpret_cast<cplx*>(M);
    for (uint64_t j = 0; j < ng; ++j) {
      rng.eng.discard(2 * r0);
      fill(m + j * Ks, Ks, rng);
      rng.eng.discard(2 * (K - r1));
    }
  }
  std::vector<cplx> m(blk), r(blk);
  for (uint64_t a = 0; a < na; ++a) {
    if (a < lo || a >= hi) {  // M, T_AB, R blocks and the U row of an atom outside the shard
      rng.eng.discard(6 * blk + nl);
      continue;
    }
    const uint64_t al = a - lo;
    fill(m.data(), blk, rng);
    cplx* g = reinterpret_cast<cplx*>(T_AA) + al * blk;
    for (uint64_t j = 0; j < nl; ++j)  // G = M^H M
      for (uint64_t i = 0; i < nl; ++i) {
        cplx s = 0.0;
        for (uint64_t k = 0; k < nl; ++k) s += std::conj(m[k + i * nl]) * m[k + j * nl];
        g[i + j * nl] = s;
      }
    const bool is_hpd = a < na - n_not_hpd;
    hpd[al] = is_hpd ? 1 : 0;
    if (is_hpd) {
      for (uint64_t i = 0; i < nl; ++i) g[i + i * nl] += 1.0;
    } else {
      const double shift = 1.05 * lambda_max(g, nl) + 1.0;
      for (uint64_t i = 0; i < nl; ++i) g[i + i * nl] -= shift;
    }
    fill(reinterpret_cast<cplx*>(T_AB) + al * blk, blk, rng);
    fill(r.data(), blk, rng);
    cplx* t = reinterpret_cast<cplx*>(T_BB) + al * blk;
    for (uint64_t j = 0; j < nl; ++j)
      for (uint64_t i = 0; i < nl; ++i) t[i + j * nl] = 0.5 * (r[i + j * nl] + std::conj(r[j + i * nl]));
    for (uint64_t i = 0; i < nl; ++i) U[al * nl + i] = rng.uniform(0.5, 1.5);
  }
}

int check_args(uint64_t na, uint64_t nl, uint64_t ng, uint64_t n_not_hpd, const void* const* outs, int nouts) {
  if (na < 1 || nl < 1 || ng < 1 || n_not_hpd > na) {
    hsdla_b200::g_last_error = "generate_problem: all dims must be >= 1 and n_not_hpd <= n_atoms";
    return HSDLA_B200_DIMENSION_ERROR;
  }
  for (int i = 0; i < nouts; ++i)
    if (!outs[i]) {
      hsdla_b200::g_last_error = "generate_problem: null output";
      return HSDLA_B200_DIMENSION_ERROR;
    }
  return HSDLA_B200_OK;
}

}  // namespace

extern "C" int hsdla_b200_generate_problem(uint64_t na, uint64_t nl, uint64_t ng, uint64_t seed, uint64_t n_not_hpd,
                                           double* A, double* B, double* T_AA, double* T_AB, double* T_BB,
                                           double* U, uint8_t* hpd) {
  const void* outs[] = {A, B, T_AA, T_AB, T_BB, U, hpd};
  if (const int rc = check_args(na, nl, ng, n_not_hpd, outs, 7)) return rc;
  generate(na, nl, ng, seed, n_not_hpd, 0, na, A, B, T_AA, T_AB, T_BB, U, hpd);
  return HSDLA_B200_OK;
}

extern "C" int hsdla_b200_generate_problem_shard(uint64_t na, uint64_t nl, uint64_t ng, uint64_t seed,
                                                 uint64_t n_not_hpd, uint64_t lo, uint64_t hi, double* A, double* B,
                                                 double* T_AA, double* T_AB, double* T_BB, double* U, uint8_t* hpd) {
  const void* outs[] = {A, B, T_AA, T_AB, T_BB, U, hpd};
  if (const int rc = check_args(na, nl, ng, n_not_hpd, outs, 7)) return rc;
  if (lo >= hi || hi > na) {
    hsdla_b200::g_last_error = "generate_problem_shard: need atom_begin < atom_end <= n_atoms";
    return HSDLA_B200_DIMENSION_ERROR;
  }
  generate(na, nl, ng, seed, n_not_hpd, lo, hi, A, B, T_AA, T_AB, T_BB, U, hpd);
  return HSDLA_B200_OK;
}
