"""The reference's kernel layer (``hsdla::kernels``, proj/include/hsdla/kernels.hpp:24-75)
on the GPU, through the C-ABI (hsdla_b200_herk / her2k / herkx / gemm / hemm / trmm /
potrf / diag_scale).  Same names, argument order and meaning as the reference:

  gemm(alpha, a, ta, b, tb, beta, c, ledger=None)       kernels.cpp:245-283
  hemm(side, alpha, a, b, beta, c, ledger=None)         kernels.cpp:285-308 (a read lower)
  herk(alpha, a, beta, c, ledger=None)                  kernels.cpp:310-329 (c lower)
  her2k(alpha, a, b, beta, c, ledger=None)              kernels.cpp:331-353
  herkx(alpha, a, b, beta, c, ledger=None)              kernels.cpp:355-377
  trmm(side, trans, alpha, t, b, ledger=None)           kernels.cpp:379-415 (b in place)
  potrf(a, ledger=None) -> PotrfResult                  kernels.cpp:417-436
  diag_scale(u, b, x=None, ledger=None) -> x            kernels.cpp:438-450

Matrices are complex128 numpy arrays in Fortran (column-major) order, updated in
place like the reference's ``ComplexMatrix&`` outputs; ``ledger`` is a FlopLedger
charged the reference's closed form.  All arithmetic runs on the GPU.
"""
import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .errors import DimensionError, check

NONE, CONJ_TRANS = "none", "conj_trans"
LEFT, RIGHT = "left", "right"
_TRANS = {NONE: 0, CONJ_TRANS: 1, "N": 0, "C": 1}


def _mat(x, name, writable=False):
    if not isinstance(x, np.ndarray) or x.dtype != np.complex128 or x.ndim != 2:
        raise DimensionError(f"{name} must be a 2-D complex128 array")
    if not x.flags.f_contiguous:
        if writable:
            raise DimensionError(f"{name} must be Fortran-contiguous (it is updated in place)")
        x = np.asfortranarray(x)
    return x


def _ld(x):
    return C.c_uint64(max(x.shape[0], 1))


def _ptr(x):
    return x.ctypes.data_as(C.c_void_p)


def _cplx(z):
    z = complex(z)
    return (C.c_double * 2)(z.real, z.imag)


def _charge(ledger, kernel, counter):
    if ledger is not None:
        ledger.add(kernel, int(counter.value))


def _trans(t):
    if t not in _TRANS:
        raise DimensionError(f"unknown trans {t!r}")
    return _TRANS[t]


def gemm(alpha, a, ta, b, tb, beta, c, ledger=None, device=0):
    """C := alpha op(A) op(B) + beta C (kernels.cpp:245-283)."""
    a, b, c = _mat(a, "a"), _mat(b, "b"), _mat(c, "c", True)
    ia, ib = _trans(ta), _trans(tb)
    m, k = (a.shape[1], a.shape[0]) if ia else a.shape
    kb, n = (b.shape[1], b.shape[0]) if ib else b.shape
    if k != kb or c.shape != (m, n):
        raise DimensionError("gemm: nonconforming dimensions")
    fl = C.c_uint64(0)
    check(_lib.lib().hsdla_b200_gemm(C.c_int(device), C.c_int(ia), C.c_int(ib), C.c_uint64(m), C.c_uint64(n),
                                     C.c_uint64(k), _cplx(alpha), _ptr(a), _ld(a), _ptr(b), _ld(b), _cplx(beta),
                                     _ptr(c), _ld(c), C.byref(fl)), "gemm")
    _charge(ledger, "gemm", fl)
    return c


def hemm(side, alpha, a, b, beta, c, ledger=None, device=0):
    """Left side: C := alpha A B + beta C, A Hermitian read from its lower triangle."""
    if side != LEFT:
        raise DimensionError("hemm: only Side::Left supported")
    a, b, c = _mat(a, "a"), _mat(b, "b"), _mat(c, "c", True)
    n, m = a.shape[0], b.shape[1]
    if a.shape != (n, n) or b.shape[0] != n or c.shape != (n, m):
        raise DimensionError("hemm: nonconforming dimensions")
    fl = C.c_uint64(0)
    check(_lib.lib().hsdla_b200_hemm(C.c_int(device), C.c_uint64(n), C.c_uint64(m), _cplx(alpha), _ptr(a), _ld(a),
                                     _ptr(b), _ld(b), _cplx(beta), _ptr(c), _ld(c), C.byref(fl)), "hemm")
    _charge(ledger, "hemm", fl)
    return c


def _tri(fn, kernel, alpha, a, b, beta, c, ledger, device):
    a, c = _mat(a, "a"), _mat(c, "c", True)
    k, n = a.shape
    if b is not None:
        b = _mat(b, "b")
        if b.shape != a.shape:
            raise DimensionError(f"{kernel}: nonconforming dimensions")
    if c.shape != (n, n):
        raise DimensionError(f"{kernel}: nonconforming dimensions")
    fl = C.c_uint64(0)
    if b is None:
        rc = fn(C.c_int(device), C.c_uint64(n), C.c_uint64(k), C.c_double(float(alpha)), _ptr(a), _ld(a),
                C.c_double(float(beta)), _ptr(c), _ld(c), C.byref(fl))
    else:
        rc = fn(C.c_int(device), C.c_uint64(n), C.c_uint64(k), _cplx(alpha), _ptr(a), _ld(a), _ptr(b), _ld(b),
                C.c_double(float(beta)), _ptr(c), _ld(c), C.byref(fl))
    check(rc, kernel)
    _charge(ledger, kernel, fl)
    return c


def herk(alpha, a, beta, c, ledger=None, device=0):
    """C := alpha A^H A + beta C, lower triangle only (A is k x n)."""
    return _tri(_lib.lib().hsdla_b200_herk, "herk", alpha, a, None, beta, c, ledger, device)


def her2k(alpha, a, b, beta, c, ledger=None, device=0):
    """C := alpha A^H B + conj(alpha) B^H A + beta C, lower triangle only."""
    return _tri(_lib.lib().hsdla_b200_her2k, "her2k", alpha, a, b, beta, c, ledger, device)


def herkx(alpha, a, b, beta, c, ledger=None, device=0):
    """C := alpha A^H B + beta C, lower triangle only (the caller guarantees Hermitian)."""
    return _tri(_lib.lib().hsdla_b200_herkx, "herkx", alpha, a, b, beta, c, ledger, device)


def trmm(side, trans, alpha, t, b, ledger=None, device=0):
    """In place B := alpha op(T) B with lower-triangular T (left side)."""
    if side != LEFT:
        raise DimensionError("trmm: only Side::Left supported")
    t, b = _mat(t, "t"), _mat(b, "b", True)
    n, m = t.shape[0], b.shape[1]
    if t.shape != (n, n) or b.shape[0] != n:
        raise DimensionError("trmm: nonconforming dimensions")
    fl = C.c_uint64(0)
    check(_lib.lib().hsdla_b200_trmm(C.c_int(device), C.c_int(_trans(trans)), C.c_uint64(n), C.c_uint64(m),
                                     _cplx(alpha), _ptr(t), _ld(t), _ptr(b), _ld(b), C.byref(fl)), "trmm")
    _charge(ledger, "trmm", fl)
    return b


@dataclass
class PotrfResult:
    factor: Optional[np.ndarray]  # lower triangular, C C^H = A; None when not HPD
    pivot: int = 0                # failing pivot index when not ok()

    def ok(self):
        return self.factor is not None


def potrf(a, ledger=None, device=0):
    """Cholesky of the lower triangle of A (bit-identical to the reference's factor)."""
    from .pipeline import potrf as batched
    a = _mat(a, "a")
    n = a.shape[0]
    if a.shape != (n, n):
        raise DimensionError("potrf: square matrix required")
    if ledger is not None:
        ledger.add("potrf", 4 * n * n * n // 3)
    L, piv = batched(a[:, :, None], device)
    return PotrfResult(np.asfortranarray(L[:, :, 0]), 0) if piv[0] < 0 else PotrfResult(None, int(piv[0]))


def diag_scale(u, b, x=None, ledger=None, device=0):
    """X[r][c] = u[r] B[r][c]; x may be b (in place)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    b = _mat(b, "b")
    if u.ndim != 1 or u.size != b.shape[0]:
        raise DimensionError("diag_scale: scale length does not match row count")
    if x is None or x.shape != b.shape:
        x = np.zeros(b.shape, np.complex128, order="F")
    x = _mat(x, "x", True)
    fl = C.c_uint64(0)
    check(_lib.lib().hsdla_b200_diag_scale(C.c_int(device), C.c_uint64(b.shape[0]), C.c_uint64(b.shape[1]), _ptr(u),
                                           _ptr(b), _ld(b), _ptr(x), _ld(x), C.byref(fl)), "diag_scale")
    _charge(ledger, "scaling", fl)
    return x
