// LAPW matching-coefficient setup on sm_100a (north_star subsystem 1).
//
// Builds the stacked coefficient matrices A, B ((N_A N_L) x N_G, column-major,
// row a*N_L + lm, lm = l(l+1)+m) that the reference takes as INPUT
// (problem.hpp:16-27; SPEC.md:89-90 lists their construction as a non-goal, so
// this subsystem has no reference implementation: its parity oracle is the
// self-authored C restatement oracle/hsdla_oracle.c:orc_lapw_coefficients,
// itself pinned against scipy's Y_lm and j_l).
//
// Paper Eq. (basis): inside muffin tin a,
//   phi_G(k, r) = sum_lm [A^{a,G}_lm u_l(r) + B^{a,G}_lm udot_l(r)] Y_lm(r_a^)
// matched in value and radial derivative at r = R_a to the plane wave
// Omega^{-1/2} e^{i K.r}, K = k + G.  With the Rayleigh expansion
//   e^{iK.r} = e^{iK.tau_a} 4 pi sum_lm i^l j_l(K r_a) Y*_lm(K^) Y_lm(r_a^)
// and c_lm = 4 pi Omega^{-1/2} e^{iK.tau_a} i^l Y*_lm(K^), the 2x2 matching
// system gives (det = u udot' - udot u')
//   A = c [ j_l(KR) udot'_l - K j_l'(KR) udot_l ] / det
//   B = c [ K j_l'(KR) u_l  - j_l(KR) u'_l     ] / det.
// Y_lm: orthonormal complex spherical harmonics with the Condon-Shortley phase
// (scipy.special.sph_harm_y convention), Y_{l,-m} = (-1)^m conj(Y_lm).
//
// Two passes.  lapw_tables_kernel computes, fully parallel over independent
// items, the per-G tables Y_lm(K^) (one thread per (G, m): stable normalised-
// Legendre recursion), the matching factors (one thread per (G, type): j_l / K j_l'
// by series / upward / Miller downward recursion) and the structure factors
// e^{iK.tau_a} (one thread per (G, atom)).  lapw_stream_kernel then writes the
// 2 * N_A * N_L complex outputs of every column with coalesced 16-byte streaming
// stores, one thread per (row, column) — the HBM-write-bound pass (roofline: 32 B
// per (atom, lm, G) written; table reads < 2 % of that, L2-resident).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hsdla_b200 {

constexpr int kLapwMaxL = 20;  // lmax <= 20 (N_L <= 441)
constexpr int kLapwMaxTypes = 32;

struct LapwDevParams {
  const double* gvec;       // n_g x 3
  const double* tau;        // n_atoms x 3 (this shard's atoms)
  const int32_t* type;      // n_atoms
  const double* radial;     // n_types x (lmax+1) x 4: u, u', udot, udot'
  const double* rmt;        // n_types
  const double* ylm_coef;   // 4 (lmax+1)^2: ylm_coefficients()
  double kx, ky, kz;
  double pref;              // 4 pi / sqrt(Omega)
  int n_atoms, n_types, lmax, n_g;
  double2* A;               // output, ld = ldo (rows a*N_L + lm)
  double2* B;
  uint64_t ldo;
};

// j_l(x) for l = 0..lmax (x >= 0), written to j[0..lmax].
// Series only for x < 1e-3 (converges in 2-3 terms there); Miller / upward recurrence
// otherwise, with 1/x hoisted out of the recurrences (no division on the chain).
__host__ __device__ inline void sph_bessel(int lmax, double x, double* j) {
  if (x < 1e-3) {  // power series: j_l(x) = x^l/(2l+1)!! sum_k (-x^2/2)^k / (k! (2l+3)(2l+5)...(2l+2k+1))
    double xl = 1.0, df = 1.0;  // x^l, (2l+1)!!
    for (int l = 0; l <= lmax; ++l) {
      if (l > 0) {
        xl *= x;
        df *= (2.0 * l + 1.0);
      }
      double term = 1.0, sum = 1.0;
      const double y = -0.5 * x * x;
      for (int k = 1; k < 30; ++k) {
        term *= y / (k * (2.0 * l + 2.0 * k + 1.0));
        sum += term;
        if (fabs(term) < 1e-17 * fabs(sum)) break;
      }
      j[l] = xl / df * sum;
    }
    return;
  }
  double s, c;
  sincos(x, &s, &c);
  const double ix = 1.0 / x;
  const double j0 = s * ix;
  if (x > lmax) {  // upward recurrence is stable for x > l
    j[0] = j0;
    if (lmax >= 1) j[1] = (j0 - c) * ix;
    for (int l = 1; l < lmax; ++l) j[l + 1] = (2.0 * l + 1.0) * ix * j[l] - j[l - 1];
    return;
  }
  // Miller downward recurrence from well above lmax.  Normalised by whichever of
  // j_0 = sin x / x and j_1 = (sin x / x - cos x) / x is larger in magnitude: they never
  // vanish together, so the normalisation keeps full precision next to the zeros of j_0
  // (x = n pi, where normalising by j_0 alone loses every digit).  In the Miller range
  // (1e-3 <= x <= lmax) j_1 is chosen only for |j_1| > |j_0|, i.e. x > 2, where its
  // formula has no cancellation.
  const int top = lmax + 30 + static_cast<int>(x);
  double jp1 = 0.0, jl = 1e-300, m1 = 0.0;  // m1: the unnormalised j_1
  for (int l = top; l >= 1; --l) {
    const double jm1 = (2.0 * l + 1.0) * ix * jl - jp1;
    jp1 = jl;
    jl = jm1;  // now j_{l-1}
    if (l - 1 <= lmax) j[l - 1] = jl;
    if (l - 1 == 1) m1 = jl;
    if (fabs(jl) > 1e250) {  // rescale everything computed so far
      const double f = 1e-250;
      jl *= f;
      jp1 *= f;
      m1 *= f;
      for (int m = l - 1; m <= lmax; ++m) j[m] *= f;
    }
  }
  const double j1 = (j0 - c) * ix;
  const double norm = fabs(j1) > fabs(j0) ? j1 / m1 : j0 / jl;
  for (int l = 0; l <= lmax; ++l) j[l] *= norm;
}

// Y_lm(theta, phi) for one m >= 0 and all l in [m, lmax], as the complex values
// Y_{l,m} stored at lm = l(l+1)+m, plus Y_{l,-m} = (-1)^m conj(Y_lm).  x = cos(theta),
// sth = sin(theta), (cph, sph) = (cos phi, sin phi).
__host__ __device__ inline void ylm_column(int lmax, int m, double x, double sth, double cph, double sph, double2* Y) {
  const double inv4pi = 0.07957747154594767;  // 1/(4 pi)
  // normalised P_m^m with Condon-Shortley phase: P_0^0 = 1/sqrt(4pi); P_m^m = -sqrt((2m+1)/(2m)) sth P_{m-1}^{m-1}
  double pmm = sqrt(inv4pi);
  for (int k = 1; k <= m; ++k) pmm *= -sqrt((2.0 * k + 1.0) / (2.0 * k)) * sth;
  // e^{i m phi}
  double er = 1.0, ei = 0.0;
  for (int k = 0; k < m; ++k) {
    const double t = er * cph - ei * sph;
    ei = er * sph + ei * cph;
    er = t;
  }
  const double sgn = (m & 1) ? -1.0 : 1.0;
  double p_lm2 = 0.0, p_lm1 = pmm;
  for (int l = m; l <= lmax; ++l) {
    double p;
    if (l == m) {
      p = pmm;
    } else if (l == m + 1) {
      p = sqrt(2.0 * m + 3.0) * x * pmm;
    } else {
      const double a = sqrt((4.0 * l * l - 1.0) / (static_cast<double>(l) * l - static_cast<double>(m) * m));
      const double b = sqrt((static_cast<double>(l - 1) * (l - 1) - static_cast<double>(m) * m) /
                            (4.0 * (l - 1) * (l - 1) - 1.0));
      p = a * (x * p_lm1 - b * p_lm2);
    }
    if (l > m) {
      p_lm2 = p_lm1;
      p_lm1 = p;
    }
    const int lm = l * (l + 1);
    Y[lm + m] = make_double2(p * er, p * ei);
    if (m > 0) Y[lm - m] = make_double2(sgn * p * er, -sgn * p * ei);
  }
}

// The l-recurrence coefficients of ylm_column, tabulated once on the host (the same
// correctly rounded sqrt / division results): index l*(lmax+1)+m.
//   C[0][l*(lmax+1)+m] = a_lm = sqrt((4l^2-1)/(l^2-m^2))          (l >= m+2)
//   C[1][l*(lmax+1)+m] = b_lm = sqrt(((l-1)^2-m^2)/(4(l-1)^2-1))   (l >= m+2)
//   C[2][m]            = sqrt(2m+3)
//   C[3][k]            = sqrt((2k+1)/(2k))                          (k >= 1)
inline void ylm_coefficients(int lmax, double* C) {
  const int n = (lmax + 1) * (lmax + 1);
  for (int i = 0; i < 4 * n; ++i) C[i] = 0.0;
  for (int m = 0; m <= lmax; ++m) {
    C[2 * n + m] = sqrt(2.0 * m + 3.0);
    if (m >= 1) C[3 * n + m] = sqrt((2.0 * m + 1.0) / (2.0 * m));
    for (int l = m + 2; l <= lmax; ++l) {
      C[l * (lmax + 1) + m] = sqrt((4.0 * l * l - 1.0) / (static_cast<double>(l) * l - static_cast<double>(m) * m));
      C[n + l * (lmax + 1) + m] = sqrt((static_cast<double>(l - 1) * (l - 1) - static_cast<double>(m) * m) /
                                       (4.0 * (l - 1) * (l - 1) - 1.0));
    }
  }
}

// ylm_column with the tabulated coefficients (no sqrt / division on the device).
__device__ inline void ylm_column_tab(int lmax, int m, double x, double sth, double cph, double sph, double2* Y,
                                      const double* __restrict__ C) {
  const int n = (lmax + 1) * (lmax + 1);
  double pmm = 0.28209479177387814;  // sqrt(1/(4 pi))
  for (int k = 1; k <= m; ++k) pmm *= -C[3 * n + k] * sth;
  double er = 1.0, ei = 0.0;
  for (int k = 0; k < m; ++k) {
    const double t = er * cph - ei * sph;
    ei = er * sph + ei * cph;
    er = t;
  }
  const double sgn = (m & 1) ? -1.0 : 1.0;
  double p_lm2 = 0.0, p_lm1 = pmm;
  for (int l = m; l <= lmax; ++l) {
    double p;
    if (l == m) {
      p = pmm;
    } else if (l == m + 1) {
      p = C[2 * n + m] * x * pmm;
    } else {
      p = C[l * (lmax + 1) + m] * (x * p_lm1 - C[n + l * (lmax + 1) + m] * p_lm2);
    }
    if (l > m) {
      p_lm2 = p_lm1;
      p_lm1 = p;
    }
    const int lm = l * (l + 1);
    Y[lm + m] = make_double2(p * er, p * ei);
    if (m > 0) Y[lm - m] = make_double2(sgn * p * er, -sgn * p * ei);
  }
}

// Direction of K: cos(theta), sin(theta), cos(phi), sin(phi); K = 0 -> z axis.
__host__ __device__ inline void k_direction(double kx, double ky, double kz, double& kn, double& x, double& sth,
                                            double& cph, double& sph) {
  const double rho = sqrt(kx * kx + ky * ky);
  kn = sqrt(rho * rho + kz * kz);
  if (kn == 0.0) {
    x = 1.0;
    sth = 0.0;
    cph = 1.0;
    sph = 0.0;
    return;
  }
  x = kz / kn;
  sth = rho / kn;
  if (rho == 0.0) {
    cph = 1.0;
    sph = 0.0;
  } else {
    cph = kx / rho;
    sph = ky / rho;
  }
}

// ---- pass 1: per-G tables (one thread per independent item) ----------------
//   Y[g][lm]      = Y_lm(K_g^)                     (one item per (g, m >= 0))
//   F[g][t][l]    = (fa, fb) matching factors         (one item per (g, type))
//   SF[g][a]      = pref * e^{i K_g . tau_a}          (one item per (g, atom))
// Item ranges are contiguous per kind so warps stay convergent.
__global__ void __launch_bounds__(256) lapw_tables_kernel(const LapwDevParams P, double2* __restrict__ tabY,
                                                          double2* __restrict__ tabF, double2* __restrict__ tabS) {
  const int nlv = P.lmax + 1, nl = nlv * nlv;
  const uint64_t ng = P.n_g;
  const uint64_t nY = ng * nlv, nF = ng * P.n_types, nS = ng * P.n_atoms;
  for (uint64_t it = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; it < nY + nF + nS;
       it += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t g;
    int sub;
    if (it < nY) {
      g = it / nlv;
      sub = static_cast<int>(it - g * nlv);
    } else if (it < nY + nF) {
      g = (it - nY) / P.n_types;
      sub = static_cast<int>(it - nY - g * P.n_types);
    } else {
      g = (it - nY - nF) / P.n_atoms;
      sub = static_cast<int>(it - nY - nF - g * P.n_atoms);
    }
    const double kx = P.kx + P.gvec[3 * g], ky = P.ky + P.gvec[3 * g + 1], kz = P.kz + P.gvec[3 * g + 2];
    if (it < nY) {
      double kn, x, sth, cph, sph;
      k_direction(kx, ky, kz, kn, x, sth, cph, sph);
      ylm_column_tab(P.lmax, sub, x, sth, cph, sph, tabY + g * nl, P.ylm_coef);
    } else if (it < nY + nF) {
      const int t = sub;
      const double kn = sqrt(kx * kx + ky * ky + kz * kz);
      double jl[kLapwMaxL + 2];
      const double xr = kn * P.rmt[t];
      sph_bessel(P.lmax + 1, xr, jl);
      for (int l = 0; l <= P.lmax; ++l) {
        // K j_l'(KR) = K [ l/x j_l - j_{l+1} ]  (recurrence valid for all l, x > 0); 0 at K = 0
        const double kjd = xr > 0.0 ? kn * (l / xr * jl[l] - jl[l + 1]) : 0.0;
        const double* r = P.radial + (static_cast<size_t>(t) * nlv + l) * 4;
        const double u = r[0], du = r[1], ud = r[2], dud = r[3];
        const double det = u * dud - ud * du;
        tabF[(g * P.n_types + t) * nlv + l] = make_double2((jl[l] * dud - kjd * ud) / det, (kjd * u - jl[l] * du) / det);
      }
    } else {
      const int a = sub;
      const double ph = kx * P.tau[3 * a] + ky * P.tau[3 * a + 1] + kz * P.tau[3 * a + 2];
      double sn, cs;
      sincos(ph, &sn, &cs);
      tabS[g * P.n_atoms + a] = make_double2(P.pref * cs, P.pref * sn);
    }
  }
}

// ---- pass 2: the HBM-write-bound stream --------------------------------------
// One thread per (row r = a*N_L + lm, column g) pair, rows fastest (coalesced
// 16-byte streaming stores into both A and B); the tables are L2-resident reads
// (< 2 % of the bytes written).  Each thread writes
// ROWS rows 256 apart.  grid = (n_g, ceil(K / 256 / ROWS)).
template <int ROWS>
__global__ void __launch_bounds__(256) lapw_stream_kernel(const LapwDevParams P, const double2* __restrict__ tabY,
                                                          const double2* __restrict__ tabF,
                                                          const double2* __restrict__ tabS) {
  const int nlv = P.lmax + 1, nl = nlv * nlv;
  const uint64_t K = static_cast<uint64_t>(P.n_atoms) * nl;
  const uint64_t g = blockIdx.x;
  const double2* Y = tabY + g * nl;
  const double2* F = tabF + g * P.n_types * nlv;
  const double2* SF = tabS + g * P.n_atoms;
  double2* colA = P.A + g * P.ldo;
  double2* colB = P.B + g * P.ldo;
#pragma unroll
  for (int k = 0; k < ROWS; ++k) {
    const uint64_t r = (static_cast<uint64_t>(blockIdx.y) * ROWS + k) * blockDim.x + threadIdx.x;
    if (r >= K) return;
    const int a = static_cast<int>(r / nl);
    const int lm = static_cast<int>(r - static_cast<uint64_t>(a) * nl);
    int l = static_cast<int>(sqrt(static_cast<double>(lm)));
    l -= (l * l > lm);
    l += ((l + 1) * (l + 1) <= lm);
    const double2 y = __ldg(Y + lm), s = __ldg(SF + a), fl = __ldg(F + __ldg(P.type + a) * nlv + l);
    // c = s * i^l * conj(y)
    double cr = s.x * y.x + s.y * y.y;  // s * conj(y)
    double ci = s.y * y.x - s.x * y.y;
    switch (l & 3) {  // multiply by i^l
      case 1: { const double tr = -ci; ci = cr; cr = tr; } break;
      case 2: cr = -cr; ci = -ci; break;
      case 3: { const double tr = ci; ci = -cr; cr = tr; } break;
      default: break;
    }
    __stcs(colA + r, make_double2(cr * fl.x, ci * fl.x));
    __stcs(colB + r, make_double2(cr * fl.y, ci * fl.y));
  }
}

// U rows: U[a*N_L + lm] = ||udot_l|| of atom a's type.
__global__ void lapw_u_kernel(const int32_t* type, const double* udot_norm, int lmax, int n_atoms, double* U) {
  const int nl = (lmax + 1) * (lmax + 1);
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_atoms * nl) return;
  const int a = r / nl, lm = r - a * nl;
  int l = 0;
  while ((l + 1) * (l + 1) <= lm) ++l;
  U[r] = udot_norm[type[a] * (lmax + 1) + l];
}

}  // namespace hsdla_b200
