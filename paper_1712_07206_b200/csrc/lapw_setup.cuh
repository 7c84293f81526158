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
// Kernel shape: one CTA per G column.  Per column the CTA computes Y_lm(K^)
// (one lane per m, stable normalised-Legendre recursion), j_l / K j_l' per atom
// type (series / upward / Miller downward recursion), e^{iK.tau_a} per atom and
// the per-(type, l) matching factors into shared memory, then streams the
// column's 2 * N_A * N_L complex outputs with coalesced 16-byte stores — an
// HBM-write-bound kernel (roofline: 32 B per (atom, lm, G) written).
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
  double kx, ky, kz;
  double pref;              // 4 pi / sqrt(Omega)
  int n_atoms, n_types, lmax, n_g;
  double2* A;               // output, ld = ldo (rows a*N_L + lm)
  double2* B;
  uint64_t ldo;
};

// j_l(x) for l = 0..lmax (x >= 0), written to j[0..lmax].
__host__ __device__ inline void sph_bessel(int lmax, double x, double* j) {
  if (x < 1.0) {  // power series: j_l(x) = x^l/(2l+1)!! sum_k (-x^2/2)^k / (k! (2l+3)(2l+5)...(2l+2k+1))
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
  const double j0 = s / x;
  if (x > lmax) {  // upward recurrence is stable for x > l
    j[0] = j0;
    if (lmax >= 1) j[1] = s / (x * x) - c / x;
    for (int l = 1; l < lmax; ++l) j[l + 1] = (2.0 * l + 1.0) / x * j[l] - j[l - 1];
    return;
  }
  // Miller downward recurrence from well above lmax, normalised by j_0
  const int top = lmax + 30 + static_cast<int>(x);
  double jp1 = 0.0, jl = 1e-300, scale = 1.0;
  for (int l = top; l >= 1; --l) {
    const double jm1 = (2.0 * l + 1.0) / x * jl - jp1;
    jp1 = jl;
    jl = jm1;  // now j_{l-1}
    if (l - 1 <= lmax) j[l - 1] = jl;
    if (fabs(jl) > 1e250) {  // rescale everything computed so far
      const double f = 1e-250;
      jl *= f;
      jp1 *= f;
      for (int m = l - 1; m <= lmax; ++m) j[m] *= f;
      scale *= f;
    }
  }
  const double norm = j0 / jl;
  for (int l = 0; l <= lmax; ++l) j[l] *= norm;
  (void)scale;
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

__global__ void __launch_bounds__(256) lapw_setup_kernel(const LapwDevParams P) {
  extern __shared__ double2 sh[];
  const int nl = (P.lmax + 1) * (P.lmax + 1);
  const int nlv = P.lmax + 1;
  double2* Y = sh;                           // nl
  double2* sf = Y + nl;                      // n_atoms: pref * e^{iK.tau}
  double2* fab = sf + P.n_atoms;             // n_types * nlv: (fa, fb)
  int8_t* lof = reinterpret_cast<int8_t*>(fab + P.n_types * nlv);  // l of each lm

  const int g = blockIdx.x;
  const double kx = P.kx + P.gvec[3 * g], ky = P.ky + P.gvec[3 * g + 1], kz = P.kz + P.gvec[3 * g + 2];
  double kn, x, sth, cph, sph;
  k_direction(kx, ky, kz, kn, x, sth, cph, sph);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    for (int m = lane; m <= P.lmax; m += 32) ylm_column(P.lmax, m, x, sth, cph, sph, Y);
  } else if (warp == 1) {
    for (int t = lane; t < P.n_types; t += 32) {
      double jl[kLapwMaxL + 2];
      const double R = P.rmt[t];
      const double xr = kn * R;
      sph_bessel(P.lmax + 1, xr, jl);
      for (int l = 0; l <= P.lmax; ++l) {
        // K j_l'(KR) = K [ l/x j_l - j_{l+1} ]  (recurrence valid for all l, x > 0); 0 at K = 0
        const double kjd = xr > 0.0 ? kn * (l / xr * jl[l] - jl[l + 1]) : 0.0;
        const double* r = P.radial + (static_cast<size_t>(t) * nlv + l) * 4;
        const double u = r[0], du = r[1], ud = r[2], dud = r[3];
        const double det = u * dud - ud * du;
        fab[t * nlv + l] = make_double2((jl[l] * dud - kjd * ud) / det, (kjd * u - jl[l] * du) / det);
      }
    }
  }
  for (int lm = tid; lm < nl; lm += blockDim.x) {
    int l = 0;
    while ((l + 1) * (l + 1) <= lm) ++l;
    lof[lm] = static_cast<int8_t>(l);
  }
  for (int a = tid; a < P.n_atoms; a += blockDim.x) {
    const double ph = kx * P.tau[3 * a] + ky * P.tau[3 * a + 1] + kz * P.tau[3 * a + 2];
    double s, c;
    sincos(ph, &s, &c);
    sf[a] = make_double2(P.pref * c, P.pref * s);
  }
  __syncthreads();

  // stream the column: one warp per atom block of N_L rows (contiguous in memory)
  double2* colA = P.A + static_cast<uint64_t>(g) * P.ldo;
  double2* colB = P.B + static_cast<uint64_t>(g) * P.ldo;
  const int nwarps = blockDim.x >> 5;
  for (int a = warp; a < P.n_atoms; a += nwarps) {
    const double2 s = sf[a];
    const int t = P.type[a];
    const double2* f = fab + t * nlv;
    for (int lm = lane; lm < nl; lm += 32) {
      const int l = lof[lm];
      const double2 y = Y[lm];
      // c = s * i^l * conj(y)
      double cr = s.x * y.x + s.y * y.y;   // s * conj(y)
      double ci = s.y * y.x - s.x * y.y;
      switch (l & 3) {  // multiply by i^l
        case 1: { const double tr = -ci; ci = cr; cr = tr; } break;
        case 2: cr = -cr; ci = -ci; break;
        case 3: { const double tr = ci; ci = -cr; cr = tr; } break;
        default: break;
      }
      const double2 fl = f[l];
      const uint64_t row = static_cast<uint64_t>(a) * nl + lm;
      __stcs(colA + row, make_double2(cr * fl.x, ci * fl.x));
      __stcs(colB + row, make_double2(cr * fl.y, ci * fl.y));
    }
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
