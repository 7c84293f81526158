// C++ drop-in for the reference's kernel layer (hsdla::kernels, proj/include/hsdla/kernels.hpp:24-75)
// on the GPU: same signatures over the reference's own types (ComplexMatrix, HermitianView,
// FlopLedger), calling the hsdla_b200 C-ABI.  Header-only; compiled against the reference's
// public headers and linked with libhsdla_b200.so.  The KernelConfig argument of the
// reference selects CPU threading; here the device is chosen by `device` instead.
#pragma once

#include <complex>

#include "hsdla/complex_matrix.hpp"
#include "hsdla/errors.hpp"
#include "hsdla/flop_ledger.hpp"
#include "hsdla/kernels.hpp"
#include "hsdla_b200.h"
#include "hsdla_b200/pipeline.hpp"

namespace hsdla_b200::kernels {

using hsdla::ComplexMatrix;
using hsdla::cplx;
using hsdla::FlopLedger;
using hsdla::HermitianView;
using hsdla::kernels::Side;
using hsdla::kernels::Trans;

namespace detail {
inline const double* d(const ComplexMatrix& m) { return reinterpret_cast<const double*>(m.data()); }
inline double* d(ComplexMatrix& m) { return reinterpret_cast<double*>(m.data()); }
inline uint64_t ld(const ComplexMatrix& m) { return m.rows() > 0 ? m.rows() : 1; }
inline void charge(FlopLedger* l, const char* k, uint64_t f) {
  if (l) l->add(k, f);
}
}  // namespace detail

/// C := alpha op(A) op(B) + beta C (kernels.cpp:245-283).
inline void gemm(cplx alpha, const ComplexMatrix& a, Trans ta, const ComplexMatrix& b, Trans tb, cplx beta,
                 ComplexMatrix& c, FlopLedger* ledger = nullptr, int device = 0) {
  const std::size_t m = ta == Trans::None ? a.rows() : a.cols();
  const std::size_t k = ta == Trans::None ? a.cols() : a.rows();
  const std::size_t kb = tb == Trans::None ? b.rows() : b.cols();
  const std::size_t n = tb == Trans::None ? b.cols() : b.rows();
  if (k != kb || c.rows() != m || c.cols() != n) throw hsdla::DimensionError("gemm: nonconforming dimensions");
  const double al[2] = {alpha.real(), alpha.imag()}, be[2] = {beta.real(), beta.imag()};
  uint64_t f = 0;
  throw_status(hsdla_b200_gemm(device, ta == Trans::ConjTrans, tb == Trans::ConjTrans, m, n, k, al, detail::d(a),
                               detail::ld(a), detail::d(b), detail::ld(b), be, detail::d(c), detail::ld(c), &f),
               "hsdla_b200_gemm");
  detail::charge(ledger, "gemm", f);
}

/// Left side: C := alpha A B + beta C, A read from its lower triangle (kernels.cpp:285-308).
inline void hemm(Side side, cplx alpha, const HermitianView& a, const ComplexMatrix& b, cplx beta, ComplexMatrix& c,
                 FlopLedger* ledger = nullptr, int device = 0) {
  if (side != Side::Left) throw hsdla::DimensionError("hemm: only Side::Left supported");
  const std::size_t n = a.order(), m = b.cols();
  if (b.rows() != n || c.rows() != n || c.cols() != m) throw hsdla::DimensionError("hemm: nonconforming dimensions");
  const double al[2] = {alpha.real(), alpha.imag()}, be[2] = {beta.real(), beta.imag()};
  uint64_t f = 0;
  throw_status(hsdla_b200_hemm(device, n, m, al, detail::d(a.matrix()), detail::ld(a.matrix()), detail::d(b),
                               detail::ld(b), be, detail::d(c), detail::ld(c), &f),
               "hsdla_b200_hemm");
  detail::charge(ledger, "hemm", f);
}

/// C := alpha A^H A + beta C, lower triangle only (kernels.cpp:310-329).
inline void herk(double alpha, const ComplexMatrix& a, double beta, HermitianView& c, FlopLedger* ledger = nullptr,
                 int device = 0) {
  if (c.order() != a.cols()) throw hsdla::DimensionError("herk: nonconforming dimensions");
  uint64_t f = 0;
  throw_status(hsdla_b200_herk(device, a.cols(), a.rows(), alpha, detail::d(a), detail::ld(a), beta,
                               detail::d(c.matrix()), detail::ld(c.matrix()), &f),
               "hsdla_b200_herk");
  detail::charge(ledger, "herk", f);
}

/// C := alpha A^H B + conj(alpha) B^H A + beta C, lower triangle only (kernels.cpp:331-353).
inline void her2k(cplx alpha, const ComplexMatrix& a, const ComplexMatrix& b, double beta, HermitianView& c,
                  FlopLedger* ledger = nullptr, int device = 0) {
  if (!a.same_shape(b) || c.order() != a.cols()) throw hsdla::DimensionError("her2k: nonconforming dimensions");
  const double al[2] = {alpha.real(), alpha.imag()};
  uint64_t f = 0;
  throw_status(hsdla_b200_her2k(device, a.cols(), a.rows(), al, detail::d(a), detail::ld(a), detail::d(b),
                                detail::ld(b), beta, detail::d(c.matrix()), detail::ld(c.matrix()), &f),
               "hsdla_b200_her2k");
  detail::charge(ledger, "her2k", f);
}

/// C := alpha A^H B + beta C, lower triangle only (kernels.cpp:355-377).
inline void herkx(cplx alpha, const ComplexMatrix& a, const ComplexMatrix& b, double beta, HermitianView& c,
                  FlopLedger* ledger = nullptr, int device = 0) {
  if (!a.same_shape(b) || c.order() != a.cols()) throw hsdla::DimensionError("herkx: nonconforming dimensions");
  const double al[2] = {alpha.real(), alpha.imag()};
  uint64_t f = 0;
  throw_status(hsdla_b200_herkx(device, a.cols(), a.rows(), al, detail::d(a), detail::ld(a), detail::d(b),
                                detail::ld(b), beta, detail::d(c.matrix()), detail::ld(c.matrix()), &f),
               "hsdla_b200_herkx");
  detail::charge(ledger, "herkx", f);
}

/// In place B := alpha op(T) B, T lower triangular, left side (kernels.cpp:379-415).
inline void trmm(Side side, Trans trans, cplx alpha, const ComplexMatrix& t, ComplexMatrix& b,
                 FlopLedger* ledger = nullptr, int device = 0) {
  if (side != Side::Left) throw hsdla::DimensionError("trmm: only Side::Left supported");
  const std::size_t n = t.rows();
  if (t.cols() != n || b.rows() != n) throw hsdla::DimensionError("trmm: nonconforming dimensions");
  const double al[2] = {alpha.real(), alpha.imag()};
  uint64_t f = 0;
  throw_status(hsdla_b200_trmm(device, trans == Trans::ConjTrans, n, b.cols(), al, detail::d(t), detail::ld(t),
                               detail::d(b), detail::ld(b), &f),
               "hsdla_b200_trmm");
  detail::charge(ledger, "trmm", f);
}

/// Cholesky of the lower triangle (kernels.cpp:417-436); factor bit-identical to the reference.
inline hsdla::kernels::PotrfResult potrf(const HermitianView& a, FlopLedger* ledger = nullptr, int device = 0) {
  const std::size_t n = a.order();
  if (ledger) ledger->add("potrf", 4ull * n * n * n / 3);
  ComplexMatrix l(n, n);
  int64_t pivot = -1;
  throw_status(hsdla_b200_potrf(device, 1, n, detail::d(a.matrix()), detail::d(l), &pivot), "hsdla_b200_potrf");
  hsdla::kernels::PotrfResult r;
  if (pivot < 0)
    r.factor = std::move(l);
  else
    r.pivot = static_cast<std::size_t>(pivot);
  return r;
}

/// X[r][c] = u[r] B[r][c]; x may alias b (kernels.cpp:438-450).
inline void diag_scale(std::span<const double> u, const ComplexMatrix& b, ComplexMatrix& x,
                       FlopLedger* ledger = nullptr, int device = 0) {
  if (u.size() != b.rows()) throw hsdla::DimensionError("diag_scale: scale length does not match row count");
  if (!x.same_shape(b)) x = ComplexMatrix(b.rows(), b.cols());
  uint64_t f = 0;
  throw_status(hsdla_b200_diag_scale(device, b.rows(), b.cols(), u.data(), detail::d(b), detail::ld(b), detail::d(x),
                                     detail::ld(x), &f),
               "hsdla_b200_diag_scale");
  detail::charge(ledger, "scaling", f);
}

}  // namespace hsdla_b200::kernels
