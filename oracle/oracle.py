"""TEST INFRASTRUCTURE ONLY — ctypes front-ends for the two CPU oracles.

* ``Restatement`` wraps ``oracle/liboracle.so`` (``hsdla_oracle.c``), the plain-C
  restatement of the reference algorithm; it builds everywhere from repo sources.
* ``Reference`` wraps ``oracle/_ref/libhsdla_ref.so``: the UNMODIFIED reference
  library compiled from /root/reference/proj/src by ``oracle/Makefile`` (it
  travels to the GPU box as a prebuilt file).

Both expose the same methods.  Arrays follow the reference storage:
A, B: complex128 (K, N_G) Fortran order; T_*: complex128 (N_L, N_L, N_A)
Fortran order (block a = T[:, :, a], column-major); U: float64 (N_L, N_A)
Fortran order (U[:, a] = atom a's diagonal).  Ledger key order:
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LEDGER_KEYS = ("gemm", "hemm", "her2k", "herk", "scaling", "herkx", "potrf", "trmm")

_u64 = C.c_uint64
_dp = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _ledger(arr):
    d = {k: int(v) for k, v in zip(LEDGER_KEYS, arr[:8]) if int(v) != 0}
    d["total"] = int(arr[8])
    return d


class _Problem:
    """Plain container matching hsdla::ProblemInstance (problem.hpp:16-27)."""

    def __init__(self, n_atoms, n_l, n_g, A, B, T_AA, T_AB, T_BB, U, hpd_flags):
        self.n_atoms, self.n_l, self.n_g = int(n_atoms), int(n_l), int(n_g)
        self.A, self.B, self.T_AA, self.T_AB, self.T_BB, self.U = A, B, T_AA, T_AB, T_BB, U
        self.hpd_flags = hpd_flags


def alloc_problem(na, nl, ng):
    K = na * nl
    return _Problem(
        na, nl, ng,
        np.zeros((K, ng), np.complex128, order="F"),
        np.zeros((K, ng), np.complex128, order="F"),
        np.zeros((nl, nl, na), np.complex128, order="F"),
        np.zeros((nl, nl, na), np.complex128, order="F"),
        np.zeros((nl, nl, na), np.complex128, order="F"),
        np.zeros((nl, na), np.float64, order="F"),
        np.zeros(na, np.uint8),
    )


def _args(p):
    f = lambda a: np.asfortranarray(a)
    return (f(p.A), f(p.B), f(p.T_AA), f(p.T_AB), f(p.T_BB), f(p.U))


class _Base:
    lib = None

    def generate_problem(self, na, nl, ng, seed, n_not_hpd=0):
        p = alloc_problem(na, nl, ng)
        rc = self._gen(_u64(na), _u64(nl), _u64(ng), _u64(seed), _u64(n_not_hpd), _ptr(p.A), _ptr(p.B),
                       _ptr(p.T_AA), _ptr(p.T_AB), _ptr(p.T_BB), _ptr(p.U), _ptr(p.hpd_flags))
        if rc:
            raise ValueError(f"generate_problem failed rc={rc}")
        return p

    def direct(self, which, p):
        out = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
        A, B, taa, tab, tbb, U = _args(p)
        rc = self._direct(C.c_int(which), _u64(p.n_atoms), _u64(p.n_l), _u64(p.n_g), _ptr(A), _ptr(B),
                          _ptr(taa), _ptr(tab), _ptr(tbb), _ptr(U), _ptr(out))
        if rc:
            raise ValueError(f"direct oracle refused rc={rc}")
        return out

    def direct_H(self, p):
        return self.direct(0, p)

    def direct_S(self, p):
        return self.direct(1, p)

    def direct_H_grouped(self, p):
        return self.direct(2, p)

    def potrf(self, T):
        """kernels::potrf (kernels.cpp:417-436) of every block of T ((n, n, N_A) complex128
        Fortran): returns (L (n, n, N_A) with zeros where it failed, pivot (N_A,) int64,
        -1 = success)."""
        T = np.asfortranarray(T, dtype=np.complex128)
        n, na = T.shape[0], T.shape[2]
        L = np.zeros_like(T, order="F")
        piv = np.zeros(na, np.int64)
        for a in range(na):
            blk = np.asfortranarray(T[:, :, a])
            out = np.zeros((n, n), np.complex128, order="F")
            piv[a] = self._potrf(_u64(n), _ptr(blk), _ptr(out))
            L[:, :, a] = out
        return L, piv

    def flop_model(self, na, nl, ng, variant="refined", n_hpd=None):
        out = np.zeros(9, np.uint64)
        self._flops(C.c_int(0 if variant == "original" else 1), _u64(na), _u64(nl), _u64(ng),
                    _u64(na if n_hpd is None else n_hpd), _ptr(out))
        return _ledger(out)


class Restatement(_Base):
    """The plain-C restatement (hsdla_oracle.c)."""

    def __init__(self, path=None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        lib = C.CDLL(path)
        self.lib = lib
        lib.orc_generate_problem.restype = C.c_int
        self._gen = lib.orc_generate_problem
        lib.orc_direct.restype = C.c_int
        self._direct = lib.orc_direct
        lib.orc_flop_model.restype = None
        self._flops = lambda v, na, nl, ng, nh, out: lib.orc_flop_model(v, na, nl, ng, nh, out)
        self._potrf = lambda n, a, l: lib.orc_potrf(n, a, l)
        lib.orc_rel_frobenius_error_lower.restype = C.c_double
        lib.orc_potrf.restype = C.c_int64

    def build_hs_refined(self, p):
        H = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
        S = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
        led = np.zeros(9, np.uint64)
        A, B, taa, tab, tbb, U = _args(p)
        rc = self.lib.orc_build_hs_refined(_u64(p.n_atoms), _u64(p.n_l), _u64(p.n_g), _ptr(A), _ptr(B), _ptr(taa),
                                           _ptr(tab), _ptr(tbb), _ptr(U), _ptr(H), _ptr(S), _ptr(led))
        if rc:
            raise MemoryError(f"orc_build_hs_refined rc={rc}")
        return H, S, _ledger(led)

    def build_hs_original(self, p):
        """Algorithm 1 (pipeline.cpp:189-279).  Returns H, S, ledger, n_hpd."""
        H = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
        S = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
        led = np.zeros(9, np.uint64)
        nh = C.c_uint64(0)
        A, B, taa, tab, tbb, U = _args(p)
        rc = self.lib.orc_build_hs_original(_u64(p.n_atoms), _u64(p.n_l), _u64(p.n_g), _ptr(A), _ptr(B), _ptr(taa),
                                            _ptr(tab), _ptr(tbb), _ptr(U), _ptr(H), _ptr(S), _ptr(led),
                                            C.byref(nh))
        if rc:
            raise MemoryError(f"orc_build_hs_original rc={rc}")
        return H, S, _ledger(led), int(nh.value)

    def build_hs_sampled(self, p, J):
        J = np.ascontiguousarray(J, dtype=np.uint64)
        nj = J.size
        Hs = np.zeros((nj, nj), np.complex128, order="F")
        Ss = np.zeros((nj, nj), np.complex128, order="F")
        A, B, taa, tab, tbb, U = _args(p)
        rc = self.lib.orc_build_hs_sampled(_u64(p.n_atoms), _u64(p.n_l), _u64(p.n_g), _ptr(A), _ptr(B), _ptr(taa),
                                           _ptr(tab), _ptr(tbb), _ptr(U), _ptr(J), _u64(nj), _ptr(Hs), _ptr(Ss))
        if rc:
            raise ValueError(f"orc_build_hs_sampled rc={rc}")
        return Hs, Ss

    def ylm(self, lmax, K):
        Y = np.zeros((lmax + 1) ** 2, np.complex128)
        self.lib.orc_ylm(C.c_int(lmax), *[C.c_double(float(v)) for v in K], _ptr(Y))
        return Y

    def sph_bessel(self, lmax, x):
        j = np.zeros(lmax + 1)
        self.lib.orc_sph_bessel(C.c_int(lmax), C.c_double(float(x)), _ptr(j))
        return j

    def lapw_coefficients(self, s):
        """Self-authored LAPW matching coefficients (no reference implementation exists)."""
        nl = (s.lmax + 1) ** 2
        K = s.n_atoms * nl
        A = np.zeros((K, s.n_g), np.complex128, order="F")
        B = np.zeros((K, s.n_g), np.complex128, order="F")
        U = np.zeros((nl, s.n_atoms), np.float64, order="F")
        f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        args = [f(s.kpt), f(s.gvec), f(s.tau), np.ascontiguousarray(s.atom_type, dtype=np.int32), f(s.rmt), f(s.u),
                f(s.du), f(s.udot), f(s.dudot), f(s.udot_norm)]
        rc = self.lib.orc_lapw_coefficients(_u64(s.n_atoms), _u64(s.n_types), C.c_int(s.lmax), _u64(s.n_g),
                                            *[_ptr(a) for a in args], C.c_double(s.omega), _ptr(A), _ptr(B), _ptr(U))
        if rc:
            raise ValueError(f"orc_lapw_coefficients rc={rc}")
        return A, B, U

    def rel_frobenius_error_lower(self, x, y):
        x = np.asfortranarray(x, dtype=np.complex128)
        y = np.asfortranarray(y, dtype=np.complex128)
        return float(self.lib.orc_rel_frobenius_error_lower(_u64(x.shape[0]), _ptr(x), _ptr(y)))


class Reference(_Base):
    """The unmodified reference library (oracle/_ref/libhsdla_ref.so)."""

    PATH = os.path.join(HERE, "_ref", "libhsdla_ref.so")

    @classmethod
    def available(cls):
        return os.path.exists(cls.PATH)

    def __init__(self, path=None):
        path = path or self.PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(path)
        self.lib = lib
        lib.ref_last_error.restype = C.c_char_p
        self._gen = lib.ref_generate
        self._direct = lib.ref_direct
        self._flops = lambda v, na, nl, ng, nh, out: lib.ref_flop_model(v, na, nl, ng, nh, out)

        def _potrf(n, a, l):
            piv = C.c_int64(0)
            if lib.ref_potrf(n, a, l, C.byref(piv)):
                raise RuntimeError(lib.ref_last_error().decode())
            return piv.value
        self._potrf = _potrf

    def build_hs(self, p, variant="refined", threads=1, blocked=True, block=128, want_hs=True):
        H = S = None
        if want_hs:
            H = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
            S = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
        phases = np.zeros(8)
        nph = C.c_int(0)
        led = np.zeros(9, np.uint64)
        wall = C.c_double(0)
        peak = C.c_uint64(0)
        A, B, taa, tab, tbb, U = _args(p)
        hpd = np.ascontiguousarray(p.hpd_flags, dtype=np.uint8)
        rc = self.lib.ref_build_hs(C.c_int(0 if variant == "original" else 1), _u64(p.n_atoms), _u64(p.n_l),
                                   _u64(p.n_g), _ptr(A), _ptr(B), _ptr(taa), _ptr(tab), _ptr(tbb), _ptr(U),
                                   _ptr(hpd), C.c_int(1 if blocked else 0), _u64(block), C.c_int(threads),
                                   _ptr(H), _ptr(S), _ptr(phases), C.byref(nph), _ptr(led), C.byref(wall),
                                   C.byref(peak))
        if rc:
            raise RuntimeError(f"reference build_hs failed ({rc}): {self.lib.ref_last_error().decode()}")
        names = (["s", "z_loop", "her2k", "hemm_loop", "herkx"] if variant != "original"
                 else ["z_loop", "her2k", "s", "chol_loop", "h_aa_update"])
        return {"H": H, "S": S, "ledger": _ledger(led), "wall_seconds": wall.value,
                "phases": list(zip(names or [str(i) for i in range(nph.value)], phases[: nph.value].tolist())),
                "peak_temp_bytes": peak.value}

    def build_hs_refined(self, p, threads=1):
        r = self.build_hs(p, "refined", threads=threads, blocked=False)
        return r["H"], r["S"], r["ledger"]

    def save_problem(self, p, path):
        A, B, taa, tab, tbb, U = _args(p)
        rc = self.lib.ref_save_problem(path.encode(), _u64(p.n_atoms), _u64(p.n_l), _u64(p.n_g), _ptr(A), _ptr(B),
                                       _ptr(taa), _ptr(tab), _ptr(tbb), _ptr(U),
                                       _ptr(np.ascontiguousarray(p.hpd_flags, dtype=np.uint8)))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
