/* TEST INFRASTRUCTURE ONLY — CPU oracle (restatement) of the reference HSDLA
 * refined H/S construction.  See hsdla_oracle.h for the contract and for who may
 * call this.  Every function cites the reference file:line it restates
 * (paths under /root/reference/proj).  The arithmetic replicates the reference's
 * operation order exactly (std::complex<double> semantics written out by hand,
 * no FMA contraction: build with -ffp-contract=off), so results are bit-identical
 * to the reference's Variant::Reference kernels; tests/test_oracle.py pins that
 * against golden vectors produced by the unmodified reference.
 */
#include "hsdla_oracle.h"

#define _GNU_SOURCE
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cx;

static inline cx cx_make(double r, double i) {
  cx z = {r, i};
  return z;
}
/* std::complex<double> operator* (builtin complex multiply, finite inputs). */
static inline cx cx_mul(cx a, cx b) { return cx_make(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re); }
static inline cx cx_add(cx a, cx b) { return cx_make(a.re + b.re, a.im + b.im); }
static inline cx cx_conj(cx a) { return cx_make(a.re, -a.im); }
static inline cx cx_scale(double s, cx a) { return cx_make(s * a.re, s * a.im); }

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the standard-specified engine) + the reference's mapping  */
/* to doubles (proj/src/problem.cpp:13-24).                                   */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = ~0ULL << 31, lower = (1ULL << 31) - 1;
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* problem.cpp:18-20 */
static double rng_uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
static double rng_uniform(mt64* g, double lo, double hi) { return lo + (hi - lo) * rng_uniform01(g); }
static cx rng_cplx(mt64* g) {
  const double r = rng_uniform(g, -1.0, 1.0); /* braced init: real drawn first */
  const double i = rng_uniform(g, -1.0, 1.0);
  return cx_make(r, i);
}

/* problem.cpp:26-31: column-major fill order is part of the contract. */
static void fill_random(cx* m, size_t n, mt64* g) {
  for (size_t i = 0; i < n; ++i) m[i] = rng_cplx(g);
}

/* problem.cpp:34-47: G = M^H M (full). */
static void gram(const cx* m, size_t n, cx* g) {
  for (size_t j = 0; j < n; ++j)
    for (size_t i = 0; i < n; ++i) {
      cx s = cx_make(0.0, 0.0);
      for (size_t k = 0; k < n; ++k) s = cx_add(s, cx_mul(cx_conj(m[k + i * n]), m[k + j * n]));
      g[i + j * n] = s;
    }
}

/* problem.cpp:50-69: power-iteration estimate of lambda_max. */
static double lambda_max_estimate(const cx* g, size_t n) {
  cx* v = malloc(n * sizeof(cx));
  cx* w = malloc(n * sizeof(cx));
  for (size_t i = 0; i < n; ++i) v[i] = cx_make(1.0, 0.0);
  double lambda = 0.0;
  for (int it = 0; it < 50; ++it) {
    for (size_t i = 0; i < n; ++i) {
      cx s = cx_make(0.0, 0.0);
      for (size_t j = 0; j < n; ++j) s = cx_add(s, cx_mul(g[i + j * n], v[j]));
      w[i] = s;
    }
    double norm = 0.0;
    for (size_t i = 0; i < n; ++i) norm += w[i].re * w[i].re + w[i].im * w[i].im;
    norm = sqrt(norm);
    if (norm == 0.0) break;
    lambda = norm;
    for (size_t i = 0; i < n; ++i) v[i] = cx_make(w[i].re / norm, w[i].im / norm);
  }
  free(v);
  free(w);
  return lambda;
}

int orc_generate_problem(uint64_t na, uint64_t nl, uint64_t ng, uint64_t seed, uint64_t n_not_hpd,
                         double* A, double* B, double* T_AA, double* T_AB, double* T_BB, double* U,
                         uint8_t* hpd) {
  if (na < 1 || nl < 1 || ng < 1) return 1; /* problem.cpp:82-84 DimensionError */
  if (n_not_hpd > na) return 1;             /* problem.cpp:85-87 */
  mt64* g = malloc(sizeof(mt64));
  mt64_seed(g, seed);
  const size_t K = na * nl;
  fill_random((cx*)A, K * ng, g); /* problem.cpp:97 */
  fill_random((cx*)B, K * ng, g); /* problem.cpp:98 */
  const size_t blk = nl * nl;
  cx* m = malloc(blk * sizeof(cx));
  cx* r = malloc(blk * sizeof(cx));
  const uint64_t n_hpd = na - n_not_hpd;
  for (size_t a = 0; a < na; ++a) { /* problem.cpp:108-140 */
    fill_random(m, blk, g);
    cx* taa = (cx*)T_AA + a * blk;
    gram(m, nl, taa);
    const int is_hpd = a < n_hpd;
    hpd[a] = (uint8_t)is_hpd;
    if (is_hpd) {
      for (size_t i = 0; i < nl; ++i) taa[i + i * nl].re += 1.0;
    } else {
      const double s = 1.05 * lambda_max_estimate(taa, nl) + 1.0;
      for (size_t i = 0; i < nl; ++i) taa[i + i * nl].re -= s;
    }
    fill_random((cx*)T_AB + a * blk, blk, g);
    fill_random(r, blk, g);
    cx* tbb = (cx*)T_BB + a * blk;
    for (size_t j = 0; j < nl; ++j)
      for (size_t i = 0; i < nl; ++i) tbb[i + j * nl] = cx_scale(0.5, cx_add(r[i + j * nl], cx_conj(r[j + i * nl])));
    for (size_t i = 0; i < nl; ++i) U[a * nl + i] = rng_uniform(g, 0.5, 1.5);
  }
  free(m);
  free(r);
  free(g);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Kernels (proj/src/kernels.cpp, Variant::Reference order).                 */
/* ------------------------------------------------------------------------ */

/* kernels.cpp:59-82: conj(a).b with two split accumulator pairs. */
static cx dotc(size_t k, const cx* a, const cx* b) {
  const double* pa = (const double*)a;
  const double* pb = (const double*)b;
  double cr0 = 0.0, ci0 = 0.0, cr1 = 0.0, ci1 = 0.0;
  size_t l = 0;
  for (; l + 1 < k; l += 2) {
    const double ar0 = pa[2 * l], ai0 = pa[2 * l + 1];
    const double br0 = pb[2 * l], bi0 = pb[2 * l + 1];
    cr0 += ar0 * br0 + ai0 * bi0;
    ci0 += ar0 * bi0 - ai0 * br0;
    const double ar1 = pa[2 * l + 2], ai1 = pa[2 * l + 3];
    const double br1 = pb[2 * l + 2], bi1 = pb[2 * l + 3];
    cr1 += ar1 * br1 + ai1 * bi1;
    ci1 += ar1 * bi1 - ai1 * br1;
  }
  for (; l < k; ++l) {
    const double ar = pa[2 * l], ai = pa[2 * l + 1];
    const double br = pb[2 * l], bi = pb[2 * l + 1];
    cr0 += ar * br + ai * bi;
    ci0 += ar * bi - ai * br;
  }
  return cx_make(cr0 + cr1, ci0 + ci1);
}

/* kernels.cpp:86-90 (beta is complex here; beta == 0 never reads C). */
static cx combine(cx alpha, cx prod, cx beta, const cx* old) {
  cx v = cx_mul(alpha, prod);
  if (!(beta.re == 0.0 && beta.im == 0.0)) v = cx_add(v, cx_mul(beta, *old));
  return v;
}

/* kernels.cpp:92-102 + gemm(..., ConjTrans, ..., None) (:245-283): C = alpha A^H B + beta C. */
static void gemm_ctn(size_t m, size_t n, size_t k, cx alpha, const cx* a, size_t lda, const cx* b,
                     size_t ldb, cx beta, cx* c, size_t ldc) {
  for (size_t j = 0; j < n; ++j)
    for (size_t i = 0; i < m; ++i) c[i + j * ldc] = combine(alpha, dotc(k, a + i * lda, b + j * ldb), beta, &c[i + j * ldc]);
}

/* kernels.cpp:152-167 + hemm (:285-308): C = alpha H B + beta C, H lower-read. */
static void hemm_left_lower(size_t n, size_t m, cx alpha, const cx* h, size_t ldh, const cx* b,
                            size_t ldb, cx beta, cx* c, size_t ldc) {
  for (size_t j = 0; j < m; ++j) {
    const cx* bj = b + j * ldb;
    cx* cj = c + j * ldc;
    for (size_t i = 0; i < n; ++i) {
      cx s = cx_make(0.0, 0.0);
      for (size_t l = 0; l <= i; ++l) s = cx_add(s, cx_mul(h[l * ldh + i], bj[l]));
      for (size_t l = i + 1; l < n; ++l) s = cx_add(s, cx_mul(cx_conj(h[i * ldh + l]), bj[l]));
      cj[i] = combine(alpha, s, beta, &cj[i]);
    }
  }
}

/* kernels.cpp:104-117 + herk (:310-329). */
static void herk_lower(size_t n, size_t k, double alpha, const cx* a, size_t lda, double beta, cx* c,
                       size_t ldc) {
  for (size_t j = 0; j < n; ++j)
    for (size_t i = j; i < n; ++i) {
      cx v = cx_scale(alpha, dotc(k, a + i * lda, a + j * lda));
      if (i == j) v = cx_make(v.re, 0.0);
      if (beta != 0.0) v = cx_add(v, cx_scale(beta, c[i + j * ldc]));
      c[i + j * ldc] = v;
    }
}

/* kernels.cpp:119-135 + her2k (:331-353). */
static void her2k_lower(size_t n, size_t k, cx alpha, const cx* a, size_t lda, const cx* b, size_t ldb,
                        double beta, cx* c, size_t ldc) {
  const cx alphac = cx_conj(alpha);
  for (size_t j = 0; j < n; ++j)
    for (size_t i = j; i < n; ++i) {
      cx v = cx_add(cx_mul(alpha, dotc(k, a + i * lda, b + j * ldb)),
                    cx_mul(alphac, dotc(k, b + i * ldb, a + j * lda)));
      if (i == j) v = cx_make(v.re, 0.0);
      if (beta != 0.0) v = cx_add(v, cx_scale(beta, c[i + j * ldc]));
      c[i + j * ldc] = v;
    }
}

/* kernels.cpp:137-150 + herkx (:355-377). */
static void herkx_lower(size_t n, size_t k, cx alpha, const cx* a, size_t lda, const cx* b, size_t ldb,
                        double beta, cx* c, size_t ldc) {
  for (size_t j = 0; j < n; ++j)
    for (size_t i = j; i < n; ++i) {
      cx v = cx_mul(alpha, dotc(k, a + i * lda, b + j * ldb));
      if (i == j) v = cx_make(v.re, 0.0);
      if (beta != 0.0) v = cx_add(v, cx_scale(beta, c[i + j * ldc]));
      c[i + j * ldc] = v;
    }
}

/* pipeline.cpp:149-157 load_block: dst (nl x ng) := rows [idx*nl, ...) of src (ld K). */
static void load_block(cx* dst, const cx* src, size_t K, size_t nl, size_t ng, size_t idx) {
  for (size_t j = 0; j < ng; ++j) memcpy(dst + j * nl, src + j * K + idx * nl, nl * sizeof(cx));
}
/* complex_matrix.cpp:65-75 stack_block_into. */
static void stack_block(cx* dst, const cx* blk, size_t K, size_t nl, size_t ng, size_t idx) {
  for (size_t j = 0; j < ng; ++j) memcpy(dst + j * K + idx * nl, blk + j * nl, nl * sizeof(cx));
}

void orc_flop_model(int variant, uint64_t na, uint64_t nl, uint64_t ng, uint64_t n_hpd, uint64_t* l) {
  /* pipeline.cpp:336-364; key order gemm, hemm, her2k, herk, scaling, herkx, potrf, trmm, total */
  const uint64_t n_fail = na - n_hpd;
  memset(l, 0, 9 * sizeof(uint64_t));
  l[0] = 8 * na * nl * nl * ng;
  l[1] = 8 * na * nl * nl * ng;
  l[2] = 8 * na * nl * ng * ng;
  l[3] = 8 * na * nl * ng * ng;
  l[4] = 2 * na * nl * ng;
  if (variant == 0) {
    l[6] = na * (4 * nl * nl * nl / 3);
    if (n_hpd > 0) {
      l[7] = 4 * n_hpd * nl * nl * ng;
      l[3] += 4 * n_hpd * nl * ng * ng;
    }
    if (n_fail > 0) {
      l[1] += 8 * n_fail * nl * nl * ng;
      l[0] += 8 * n_fail * nl * ng * ng;
    }
  } else {
    l[1] += 8 * na * nl * nl * ng;
    l[5] = 4 * na * nl * ng * ng;
  }
  for (int i = 0; i < 8; ++i) l[8] += l[i];
}

int orc_build_hs_refined(uint64_t na, uint64_t nl, uint64_t ng, const double* A_, const double* B_,
                         const double* T_AA, const double* T_AB, const double* T_BB,
                         const double* U, double* H_, double* S_, uint64_t* ledger) {
  const size_t K = na * nl;
  const cx* A = (const cx*)A_;
  const cx* B = (const cx*)B_;
  cx* H = (cx*)H_;
  cx* S = (cx*)S_;
  const size_t blk = nl * nl;
  cx* x = calloc(K * ng, sizeof(cx)); /* pipeline.cpp:291 */
  cx* a_slice = malloc(nl * ng * sizeof(cx));
  cx* b_slice = malloc(nl * ng * sizeof(cx));
  cx* z = malloc(nl * ng * sizeof(cx));
  if (!x || !a_slice || !b_slice || !z) return 2;
  const cx one = cx_make(1.0, 0.0), zero = cx_make(0.0, 0.0), half = cx_make(0.5, 0.0);

  /* phase s (pipeline.cpp:296-301) */
  herk_lower(ng, K, 1.0, A, K, 0.0, S, ng);
  for (size_t j = 0; j < ng; ++j) /* diag_scale, kernels.cpp:438-450 */
    for (size_t i = 0; i < K; ++i) x[i + j * K] = cx_scale(U[i], B[i + j * K]);
  herk_lower(ng, K, 1.0, x, K, 1.0, S, ng);

  /* phase z_loop (pipeline.cpp:302-307, compute_z :176-185) */
  for (size_t a = 0; a < na; ++a) {
    load_block(a_slice, A, K, nl, ng, a);
    load_block(b_slice, B, K, nl, ng, a);
    gemm_ctn(nl, ng, nl, one, (const cx*)T_AB + a * blk, nl, a_slice, nl, zero, z, nl);
    hemm_left_lower(nl, ng, half, (const cx*)T_BB + a * blk, nl, b_slice, nl, one, z, nl);
    stack_block(x, z, K, nl, ng, a);
  }
  /* phase her2k (pipeline.cpp:308-312) */
  her2k_lower(ng, K, one, x, K, B, K, 0.0, H, ng);
  /* phase hemm_loop (pipeline.cpp:313-321) */
  for (size_t a = 0; a < na; ++a) {
    load_block(a_slice, A, K, nl, ng, a);
    hemm_left_lower(nl, ng, one, (const cx*)T_AA + a * blk, nl, a_slice, nl, zero, z, nl);
    stack_block(x, z, K, nl, ng, a);
  }
  /* phase herkx (pipeline.cpp:322-325) */
  herkx_lower(ng, K, one, A, K, x, K, 1.0, H, ng);

  free(x);
  free(a_slice);
  free(b_slice);
  free(z);
  if (ledger) orc_flop_model(1, na, nl, ng, na, ledger);
  return 0;
}

/* kernels.cpp:417-436 potrf: left-looking Cholesky of the LOWER triangle of a
 * (n x n, column-major).  l receives the full n x n factor (upper exactly 0).
 * Returns -1 on success, else the failing pivot j (PotrfResult::pivot).
 * std::norm(z) is x*x + y*y in libstdc++ (<complex> _Norm_helper<true>). */
int64_t orc_potrf(uint64_t n, const double* a_, double* l_) {
  const cx* a = (const cx*)a_;
  cx* l = (cx*)l_;
  memset(l, 0, n * n * sizeof(cx));
  for (size_t j = 0; j < n; ++j) {
    double d = a[j + j * n].re;
    for (size_t p = 0; p < j; ++p) {
      const cx v = l[j + p * n];
      d -= v.re * v.re + v.im * v.im;
    }
    if (!(d > 0.0) || !isfinite(d)) return (int64_t)j;
    const double ljj = sqrt(d);
    l[j + j * n] = cx_make(ljj, 0.0);
    for (size_t i = j + 1; i < n; ++i) {
      cx s = a[i + j * n];
      for (size_t p = 0; p < j; ++p) {
        const cx t = cx_mul(l[i + p * n], cx_conj(l[j + p * n]));
        s = cx_make(s.re - t.re, s.im - t.im);
      }
      l[i + j * n] = cx_make(s.re / ljj, s.im / ljj);
    }
  }
  return -1;
}

/* kernels.cpp:385-415 trmm(Left, ConjTrans, alpha = 1): b := T^H b in place,
 * T lower triangular (nl x nl), b nl x ng. */
static void trmm_left_ctn(size_t n, size_t m, const cx* t, cx* b) {
  const cx one = cx_make(1.0, 0.0);
  for (size_t j = 0; j < m; ++j) {
    cx* bj = b + j * n;
    for (size_t i = 0; i < n; ++i) {
      cx s = cx_make(0.0, 0.0);
      const cx* ti = t + i * n;
      for (size_t l = i; l < n; ++l) s = cx_add(s, cx_mul(cx_conj(ti[l]), bj[l]));
      bj[i] = cx_mul(one, s);
    }
  }
}

/* pipeline.cpp:189-279 build_hs_original (Strategy::Cpu, Variant::Reference):
 * Z loop into work_a (B copy into work_b), her2k, restore + S with in-place U
 * scaling, per-atom potrf deciding trmm -> B_T (top of work_b) or hemm -> B_B
 * (below B_T) with A_a compressed into work_a, then H += B_T^H B_T (herk) and the
 * full gemm A_f^H B_B folded into the lower triangle.  n_hpd_out: atoms whose
 * T_AA factorised. */
int orc_build_hs_original(uint64_t na, uint64_t nl, uint64_t ng, const double* A_, const double* B_,
                          const double* T_AA, const double* T_AB, const double* T_BB,
                          const double* U, double* H_, double* S_, uint64_t* ledger, uint64_t* n_hpd_out) {
  const size_t K = na * nl, blk = nl * nl;
  const cx* A = (const cx*)A_;
  const cx* B = (const cx*)B_;
  cx* H = (cx*)H_;
  cx* S = (cx*)S_;
  cx* work_a = calloc(K * ng, sizeof(cx));
  cx* work_b = calloc(K * ng, sizeof(cx));
  cx* a_slice = malloc(nl * ng * sizeof(cx));
  cx* b_slice = malloc(nl * ng * sizeof(cx));
  cx* z = malloc(nl * ng * sizeof(cx));
  cx* fac = malloc(na * blk * sizeof(cx));
  int64_t* piv = malloc(na * sizeof(int64_t));
  if (!work_a || !work_b || !a_slice || !b_slice || !z || !fac || !piv) return 2;
  const cx one = cx_make(1.0, 0.0), zero = cx_make(0.0, 0.0), half = cx_make(0.5, 0.0);

  /* z_loop (pipeline.cpp:207-214) */
  for (size_t a = 0; a < na; ++a) {
    load_block(a_slice, A, K, nl, ng, a);
    load_block(b_slice, B, K, nl, ng, a);
    gemm_ctn(nl, ng, nl, one, (const cx*)T_AB + a * blk, nl, a_slice, nl, zero, z, nl);
    hemm_left_lower(nl, ng, half, (const cx*)T_BB + a * blk, nl, b_slice, nl, one, z, nl);
    stack_block(work_a, z, K, nl, ng, a);
    stack_block(work_b, b_slice, K, nl, ng, a);
  }
  /* her2k (:215-218) */
  her2k_lower(ng, K, one, work_a, K, work_b, K, 0.0, H, ng);
  /* s (:219-226): restore, S = A^H A, B := U B in place, S += B^H B */
  memcpy(work_a, A, K * ng * sizeof(cx));
  memcpy(work_b, B, K * ng * sizeof(cx));
  herk_lower(ng, K, 1.0, work_a, K, 0.0, S, ng);
  for (size_t j = 0; j < ng; ++j)
    for (size_t i = 0; i < K; ++i) work_b[i + j * K] = cx_scale(U[i], work_b[i + j * K]);
  herk_lower(ng, K, 1.0, work_b, K, 1.0, S, ng);
  /* chol_loop (:229-251) */
  size_t n_hpd = 0;
  for (size_t a = 0; a < na; ++a) {
    piv[a] = orc_potrf(nl, T_AA + 2 * a * blk, (double*)(fac + a * blk));
    if (piv[a] < 0) ++n_hpd;
  }
  size_t s = 0, f = 0;
  for (size_t a = 0; a < na; ++a) {
    load_block(a_slice, A, K, nl, ng, a);
    if (piv[a] < 0) {
      memcpy(z, a_slice, nl * ng * sizeof(cx));
      trmm_left_ctn(nl, ng, fac + a * blk, z);
      stack_block(work_b, z, K, nl, ng, s++);
    } else {
      hemm_left_lower(nl, ng, one, (const cx*)T_AA + a * blk, nl, a_slice, nl, zero, z, nl);
      stack_block(work_b, z, K, nl, ng, n_hpd + f);
      stack_block(work_a, a_slice, K, nl, ng, f++);
    }
  }
  /* h_aa_update (:253-276); the row blocks are used in place with ld = K (the
   * reference copies them out first: same values, same operation order). */
  const size_t n_fail = na - n_hpd;
  if (n_hpd > 0) herk_lower(ng, n_hpd * nl, 1.0, work_b, K, 1.0, H, ng);
  if (n_fail > 0) {
    cx* full = malloc(ng * ng * sizeof(cx));
    if (!full) return 2;
    gemm_ctn(ng, ng, n_fail * nl, one, work_a, K, work_b + n_hpd * nl, K, zero, full, ng);
    for (size_t j = 0; j < ng; ++j)
      for (size_t i = j; i < ng; ++i) H[i + j * ng] = cx_add(H[i + j * ng], full[i + j * ng]);
    free(full);
  }
  free(work_a);
  free(work_b);
  free(a_slice);
  free(b_slice);
  free(z);
  free(fac);
  free(piv);
  if (ledger) orc_flop_model(0, na, nl, ng, n_hpd, ledger);
  if (n_hpd_out) *n_hpd_out = n_hpd;
  return 0;
}

int orc_build_hs_sampled(uint64_t na, uint64_t nl, uint64_t ng, const double* A_, const double* B_,
                         const double* T_AA, const double* T_AB, const double* T_BB,
                         const double* U, const uint64_t* J, uint64_t nj, double* Hs, double* Ss) {
  const size_t K = na * nl;
  cx* As = malloc(K * nj * sizeof(cx));
  cx* Bs = malloc(K * nj * sizeof(cx));
  if (!As || !Bs) return 2;
  for (size_t c = 0; c < nj; ++c) {
    if (J[c] >= ng) return 1;
    memcpy(As + c * K, (const cx*)A_ + J[c] * K, K * sizeof(cx));
    memcpy(Bs + c * K, (const cx*)B_ + J[c] * K, K * sizeof(cx));
  }
  memset(Hs, 0, nj * nj * sizeof(cx));
  memset(Ss, 0, nj * nj * sizeof(cx));
  const int rc = orc_build_hs_refined(na, nl, nj, (double*)As, (double*)Bs, T_AA, T_AB, T_BB, U, Hs, Ss, NULL);
  free(As);
  free(Bs);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Naive direct oracle (proj/src/oracle.cpp:72-126).                        */
/* ------------------------------------------------------------------------ */

/* oracle.cpp:11-22 */
static void full_from_lower(const cx* h, size_t n, cx* f) {
  memset(f, 0, n * n * sizeof(cx));
  for (size_t j = 0; j < n; ++j) {
    f[j + j * n] = cx_make(h[j + j * n].re, 0.0);
    for (size_t i = j + 1; i < n; ++i) {
      f[i + j * n] = h[i + j * n];
      f[j + i * n] = cx_conj(h[i + j * n]);
    }
  }
}
/* oracle.cpp:24-34: c = x y */
static void mul(const cx* x, size_t xr, size_t xc, const cx* y, size_t yc, cx* c) {
  for (size_t j = 0; j < yc; ++j)
    for (size_t i = 0; i < xr; ++i) {
      cx s = cx_make(0.0, 0.0);
      for (size_t l = 0; l < xc; ++l) s = cx_add(s, cx_mul(x[i + l * xr], y[l + j * xc]));
      c[i + j * xr] = s;
    }
}
/* oracle.cpp:36-48: acc += x^H y (x: xr x xc, y: xr x yc) — accumulate() fused. */
static void acc_mul_ch(const cx* x, size_t xr, size_t xc, const cx* y, size_t yc, cx* acc) {
  for (size_t j = 0; j < yc; ++j)
    for (size_t i = 0; i < xc; ++i) {
      cx s = cx_make(0.0, 0.0);
      for (size_t l = 0; l < xr; ++l) s = cx_add(s, cx_mul(cx_conj(x[l + i * xr]), y[l + j * xr]));
      acc[i + j * xc] = cx_add(acc[i + j * xc], s);
    }
}

int orc_direct(int which, uint64_t na, uint64_t nl, uint64_t ng, const double* A_, const double* B_,
               const double* T_AA, const double* T_AB, const double* T_BB, const double* U,
               double* out_) {
  if (ng > 512) return 3; /* oracle.cpp:63-68 ConfigError */
  const size_t K = na * nl, blk = nl * nl;
  const cx* A = (const cx*)A_;
  const cx* B = (const cx*)B_;
  cx* out = (cx*)out_;
  memset(out, 0, ng * ng * sizeof(cx));
  cx* aa = malloc(nl * ng * sizeof(cx));
  cx* ba = malloc(nl * ng * sizeof(cx));
  cx* t1 = malloc(nl * ng * sizeof(cx));
  cx* t2 = malloc(nl * ng * sizeof(cx));
  cx* taa = malloc(blk * sizeof(cx));
  cx* tbb = malloc(blk * sizeof(cx));
  cx* tba = malloc(blk * sizeof(cx));
  for (size_t a = 0; a < na; ++a) {
    load_block(aa, A, K, nl, ng, a);
    load_block(ba, B, K, nl, ng, a);
    if (which == 1) { /* direct_S, oracle.cpp:72-86 */
      acc_mul_ch(aa, nl, ng, aa, ng, out);
      for (size_t j = 0; j < ng; ++j)
        for (size_t i = 0; i < nl; ++i) t1[i + j * nl] = cx_scale(U[a * nl + i], ba[i + j * nl]);
      acc_mul_ch(t1, nl, ng, t1, ng, out);
      continue;
    }
    const cx* tab = (const cx*)T_AB + a * blk;
    full_from_lower((const cx*)T_AA + a * blk, nl, taa);
    full_from_lower((const cx*)T_BB + a * blk, nl, tbb);
    for (size_t j = 0; j < nl; ++j) /* conj_t, oracle.cpp:50-56 */
      for (size_t i = 0; i < nl; ++i) tba[j + i * nl] = cx_conj(tab[i + j * nl]);
    if (which == 0) { /* direct_H, oracle.cpp:88-103 */
      mul(taa, nl, nl, aa, ng, t1);
      acc_mul_ch(aa, nl, ng, t1, ng, out);
      mul(tab, nl, nl, ba, ng, t1);
      acc_mul_ch(aa, nl, ng, t1, ng, out);
      mul(tba, nl, nl, aa, ng, t1);
      acc_mul_ch(ba, nl, ng, t1, ng, out);
      mul(tbb, nl, nl, ba, ng, t1);
      acc_mul_ch(ba, nl, ng, t1, ng, out);
    } else { /* direct_H_grouped, oracle.cpp:105-126 */
      mul(tba, nl, nl, aa, ng, t1);
      mul(tbb, nl, nl, ba, ng, t2);
      for (size_t i = 0; i < nl * ng; ++i) t1[i] = cx_add(t1[i], cx_scale(0.5, t2[i]));
      acc_mul_ch(ba, nl, ng, t1, ng, out);
      acc_mul_ch(t1, nl, ng, ba, ng, out);
      mul(taa, nl, nl, aa, ng, t2);
      acc_mul_ch(aa, nl, ng, t2, ng, out);
    }
  }
  free(aa);
  free(ba);
  free(t1);
  free(t2);
  free(taa);
  free(tbb);
  free(tba);
  return 0;
}

double orc_rel_frobenius_error_lower(uint64_t n, const double* x_, const double* y_) {
  const cx* x = (const cx*)x_;
  const cx* y = (const cx*)y_;
  double diff = 0.0, ref = 0.0;
  for (size_t j = 0; j < n; ++j)
    for (size_t i = j; i < n; ++i) {
      const double dr = x[i + j * n].re - y[i + j * n].re, di = x[i + j * n].im - y[i + j * n].im;
      diff += dr * dr + di * di;
      ref += y[i + j * n].re * y[i + j * n].re + y[i + j * n].im * y[i + j * n].im;
    }
  const double den = sqrt(ref);
  return sqrt(diff) / (den > 1e-300 ? den : 1e-300);
}

/* ------------------------------------------------------------------------ */
/* LAPW matching coefficients (self-authored; see hsdla_oracle.h).          */
/* ------------------------------------------------------------------------ */

/* Y_lm(K^) with the Condon-Shortley phase, lm = l(l+1)+m: unnormalised
 * P_l^m by the three-term recurrence in l, normalisation by lgamma. */
void orc_ylm(int lmax, double kx, double ky, double kz, double* Yd) {
  cx* Y = (cx*)Yd;
  const double rho = sqrt(kx * kx + ky * ky), kn = sqrt(kx * kx + ky * ky + kz * kz);
  const double x = kn > 0 ? kz / kn : 1.0, s = kn > 0 ? rho / kn : 0.0;
  const double phi = (rho > 0) ? atan2(ky, kx) : 0.0;
  for (int m = 0; m <= lmax; ++m) {
    /* P_m^m = (-1)^m (2m-1)!! s^m */
    double pmm = 1.0;
    for (int k = 1; k <= m; ++k) pmm *= -(2.0 * k - 1.0) * s;
    double pl2 = 0.0, pl1 = 0.0;
    for (int l = m; l <= lmax; ++l) {
      double p;
      if (l == m) p = pmm;
      else if (l == m + 1) p = x * (2.0 * m + 1.0) * pmm;
      else p = ((2.0 * l - 1.0) * x * pl1 - (l + m - 1.0) * pl2) / (l - m);
      pl2 = pl1;
      pl1 = p;
      const double norm = sqrt((2.0 * l + 1.0) / (4.0 * M_PI) * exp(lgamma(l - m + 1.0) - lgamma(l + m + 1.0)));
      const double v = norm * p;
      const int lm = l * (l + 1);
      Y[lm + m] = cx_make(v * cos(m * phi), v * sin(m * phi));
      if (m > 0) {
        const double sg = (m & 1) ? -1.0 : 1.0;
        Y[lm - m] = cx_make(sg * Y[lm + m].re, -sg * Y[lm + m].im);
      }
    }
  }
}

/* j_l(x), l = 0..lmax: series below 1e-3, Miller downward recurrence otherwise. */
void orc_sph_bessel(int lmax, double x, double* j) {
  if (x < 1e-3) {
    double xl = 1.0, df = 1.0;
    for (int l = 0; l <= lmax; ++l) {
      if (l) { xl *= x; df *= 2.0 * l + 1.0; }
      j[l] = xl / df * (1.0 - x * x / (2.0 * (2 * l + 3)) + x * x * x * x / (8.0 * (2 * l + 3) * (2 * l + 5)));
    }
    return;
  }
  const int top = lmax + 40 + (int)(2.0 * x);
  double jp1 = 0.0, jl = 1e-280, m1 = 0.0; /* m1: the unnormalised j_1 */
  double* tmp = calloc((size_t)lmax + 1, sizeof(double));
  for (int l = top; l >= 1; --l) {
    const double jm1 = (2.0 * l + 1.0) / x * jl - jp1;
    jp1 = jl;
    jl = jm1;
    if (l - 1 <= lmax) tmp[l - 1] = jl;
    if (l - 1 == 1) m1 = jl;
    if (fabs(jl) > 1e200) {
      jl *= 1e-200;
      jp1 *= 1e-200;
      m1 *= 1e-200;
      for (int m = l - 1; m <= lmax; ++m) tmp[m] *= 1e-200;
    }
  }
  /* normalise by the larger of j_0 and j_1 (they never vanish together: exact next to
     the zeros x = n pi of j_0) */
  const double j0 = sin(x) / x, j1 = (sin(x) / x - cos(x)) / x;
  const double norm = fabs(j1) > fabs(j0) ? j1 / m1 : j0 / jl;
  for (int l = 0; l <= lmax; ++l) j[l] = tmp[l] * norm;
  free(tmp);
}

int orc_lapw_coefficients(uint64_t n_atoms, uint64_t n_types, int lmax, uint64_t n_g, const double* kpt,
                          const double* gvec, const double* tau, const int32_t* type, const double* rmt,
                          const double* u, const double* du, const double* udot, const double* dudot,
                          const double* udot_norm, double omega, double* Ad, double* Bd, double* U) {
  const int nl = (lmax + 1) * (lmax + 1), nlv = lmax + 1;
  const size_t K = n_atoms * (size_t)nl;
  cx* A = (cx*)Ad;
  cx* B = (cx*)Bd;
  cx* Y = malloc(sizeof(cx) * nl);
  double* jl = malloc(sizeof(double) * (nlv + 1));
  const double pref = 4.0 * M_PI / sqrt(omega);
  for (uint64_t a = 0; a < n_atoms; ++a) {
    if (type[a] < 0 || (uint64_t)type[a] >= n_types) return 1;
    for (int l = 0; l <= lmax; ++l)
      for (int m = -l; m <= l; ++m) U[a * nl + l * (l + 1) + m] = udot_norm[type[a] * nlv + l];
  }
  for (uint64_t g = 0; g < n_g; ++g) {
    const double kx = kpt[0] + gvec[3 * g], ky = kpt[1] + gvec[3 * g + 1], kz = kpt[2] + gvec[3 * g + 2];
    const double kn = sqrt(kx * kx + ky * ky + kz * kz);
    orc_ylm(lmax, kx, ky, kz, (double*)Y);
    for (uint64_t a = 0; a < n_atoms; ++a) {
      const int t = type[a];
      const double R = rmt[t];
      orc_sph_bessel(lmax + 1, kn * R, jl);
      const double ph = kx * tau[3 * a] + ky * tau[3 * a + 1] + kz * tau[3 * a + 2];
      const cx sf = cx_make(pref * cos(ph), pref * sin(ph));
      for (int l = 0; l <= lmax; ++l) {
        /* K j_l'(KR) from j_l' = j_{l-1} - (l+1)/x j_l (a different identity than the GPU's) */
        double kjd;
        const double xr = kn * R;
        if (xr == 0.0) kjd = 0.0;
        else if (l == 0) kjd = -kn * jl[1];
        else kjd = kn * (jl[l - 1] - (l + 1.0) / xr * jl[l]);
        const int ti = t * nlv + l;
        const double det = u[ti] * dudot[ti] - udot[ti] * du[ti];
        if (det == 0.0) return 2;
        const double fa = (jl[l] * dudot[ti] - kjd * udot[ti]) / det;
        const double fb = (kjd * u[ti] - jl[l] * du[ti]) / det;
        const cx il = (l % 4 == 0) ? cx_make(1, 0) : (l % 4 == 1) ? cx_make(0, 1) : (l % 4 == 2) ? cx_make(-1, 0) : cx_make(0, -1);
        for (int m = -l; m <= l; ++m) {
          const int lm = l * (l + 1) + m;
          const cx c = cx_mul(cx_mul(sf, il), cx_conj(Y[lm]));
          A[a * nl + lm + g * K] = cx_scale(fa, c);
          B[a * nl + lm + g * K] = cx_scale(fb, c);
        }
      }
    }
  }
  free(Y);
  free(jl);
  return 0;
}
