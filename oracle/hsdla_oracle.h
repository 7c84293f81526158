/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the HSDLA H/S construction.
 *
 * Plain-C restatement of the reference algorithm (arXiv 1712.07206, refined
 * pipeline, /root/reference/proj).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, as the CHECKER.  The product path
 * (paper_1712_07206_b200/) never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here BIT-FOR-BIT
 * against golden vectors produced by the unmodified reference library
 * (tests/golden/make_golden.py over oracle/_ref/libhsdla_ref.so).
 *
 * Storage: complex numbers are interleaved (re, im) doubles; matrices are
 * column-major (proj/include/hsdla/complex_matrix.hpp:11-31).  Per-atom N_L x N_L
 * operator blocks are contiguous, atom-major.
 */
#ifndef HSDLA_ORACLE_H
#define HSDLA_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/src/problem.cpp:79-142 */
int orc_generate_problem(uint64_t na, uint64_t nl, uint64_t ng, uint64_t seed, uint64_t n_not_hpd,
                         double* A, double* B, double* T_AA, double* T_AB, double* T_BB, double* U,
                         uint8_t* hpd);

/* proj/src/pipeline.cpp:281-329 with the kernels of proj/src/kernels.cpp
 * (Variant::Reference order).  H, S: n_g x n_g column-major; the caller zeroes
 * them (HermitianView(ng) is zero-initialised, pipeline.cpp:287-288).  ledger[9]
 * in the key order gemm, hemm, her2k, herk, scaling, herkx, potrf, trmm, total. */
int orc_build_hs_refined(uint64_t na, uint64_t nl, uint64_t ng, const double* A, const double* B,
                         const double* T_AA, const double* T_AB, const double* T_BB,
                         const double* U, double* H, double* S, uint64_t* ledger);

/* proj/src/pipeline.cpp:189-279 (Algorithm 1, Variant::Reference kernels).
 * n_hpd_out (may be NULL): atoms whose T_AA passed potrf. */
int orc_build_hs_original(uint64_t na, uint64_t nl, uint64_t ng, const double* A, const double* B,
                          const double* T_AA, const double* T_AB, const double* T_BB,
                          const double* U, double* H, double* S, uint64_t* ledger, uint64_t* n_hpd_out);

/* proj/src/kernels.cpp:417-436: Cholesky of the lower triangle of a (n x n).
 * l: full n x n factor (upper 0).  Returns -1 on success, else the failing pivot. */
int64_t orc_potrf(uint64_t n, const double* a, double* l);

/* proj/src/pipeline.cpp:336-364 */
void orc_flop_model(int variant, uint64_t na, uint64_t nl, uint64_t ng, uint64_t n_hpd,
                    uint64_t* ledger);

/* proj/src/oracle.cpp:72-126 (which: 0 direct_H, 1 direct_S, 2 direct_H_grouped);
 * out: full n_g x n_g.  Refuses n_g > 512 (oracle.hpp:9) with return 3. */
int orc_direct(int which, uint64_t na, uint64_t nl, uint64_t ng, const double* A, const double* B,
               const double* T_AA, const double* T_AB, const double* T_BB, const double* U,
               double* out);

/* Principal-submatrix sampling (SURVEY §7 hard part 3): H[J,J], S[J,J] for the
 * column subset J (|J| = nj) by the refined pipeline on the J-sliced problem.
 * Hs, Ss: nj x nj column-major (lower authoritative). */
int orc_build_hs_sampled(uint64_t na, uint64_t nl, uint64_t ng, const double* A, const double* B,
                         const double* T_AA, const double* T_AB, const double* T_BB,
                         const double* U, const uint64_t* J, uint64_t nj, double* Hs, double* Ss);

/* ---- LAPW matching-coefficient setup (north_star subsystem 1) -------------
 * NO REFERENCE IMPLEMENTATION exists (SPEC.md:89-90 makes A, B synthetic inputs);
 * this is a self-authored restatement of the standard LAPW matching (paper Eq.
 * basis), "parity self-pinned": orc_ylm / orc_sph_bessel are
 * checked against scipy.special.sph_harm_y / spherical_jn in tests/test_lapw.py.
 * Algorithms deliberately differ from the GPU's (unnormalised Legendre recurrence
 * + lgamma normalisation; Miller recurrence for every x >= 1e-3). */
void orc_ylm(int lmax, double kx, double ky, double kz, double* Y /* 2*(lmax+1)^2 */);
void orc_sph_bessel(int lmax, double x, double* j /* lmax+1 */);
/* A, B: (n_atoms*(lmax+1)^2) x n_g complex, column-major; U: n_atoms*(lmax+1)^2.
 * radial arrays are n_types x (lmax+1), row-major [t*(lmax+1)+l]. */
int orc_lapw_coefficients(uint64_t n_atoms, uint64_t n_types, int lmax, uint64_t n_g, const double* kpt,
                          const double* gvec, const double* tau, const int32_t* type, const double* rmt,
                          const double* u, const double* du, const double* udot, const double* dudot,
                          const double* udot_norm, double omega, double* A, double* B, double* U);

/* proj/src/complex_matrix.cpp:106-118 */
double orc_rel_frobenius_error_lower(uint64_t n, const double* x, const double* y);

#ifdef __cplusplus
}
#endif
#endif
