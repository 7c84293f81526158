"""LAPW matching-coefficient setup (north_star subsystem 1) — host-side API.

The reference takes A, B as synthetic inputs and has no code for
this step; the math (paper Eq. basis) and its conventions are
documented in csrc/lapw_setup.cuh.  The computation runs on the GPU
(hsdla_b200_lapw_coefficients / hsdla_b200_engine_setup_lapw); this module holds
the system description, a synthetic-system generator and the GPU-side build
`build_hs_lapw` that never moves A, B over PCIe.
"""
import ctypes as C
import math
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

from . import _lib
from .errors import ConfigError, DimensionError, check
from .pipeline import ALGOS, Engine, HSResult, PhaseTime, flop_model


class _Lapw(C.Structure):
    _fields_ = [("n_atoms", C.c_uint64), ("n_types", C.c_uint64), ("n_g", C.c_uint64), ("lmax", C.c_int),
                ("kpt", C.c_double * 3), ("omega", C.c_double), ("gvec", C.c_void_p), ("tau", C.c_void_p),
                ("atom_type", C.c_void_p), ("rmt", C.c_void_p), ("u", C.c_void_p), ("du", C.c_void_p),
                ("udot", C.c_void_p), ("dudot", C.c_void_p), ("udot_norm", C.c_void_p)]


@dataclass
class LapwSystem:
    """One k-point of an LAPW calculation: G vectors, atoms, radial boundary values.

    gvec (n_g, 3), tau (n_atoms, 3) Cartesian; atom_type (n_atoms,) int32; rmt (n_types,);
    u, du, udot, dudot, udot_norm (n_types, lmax+1): u_l(R), u_l'(R), udot_l(R), udot_l'(R), ||udot_l||."""
    lmax: int
    kpt: np.ndarray
    omega: float
    gvec: np.ndarray
    tau: np.ndarray
    atom_type: np.ndarray
    rmt: np.ndarray
    u: np.ndarray
    du: np.ndarray
    udot: np.ndarray
    dudot: np.ndarray
    udot_norm: np.ndarray

    @property
    def n_atoms(self):
        return self.tau.shape[0]

    @property
    def n_types(self):
        return self.rmt.shape[0]

    @property
    def n_g(self):
        return self.gvec.shape[0]

    @property
    def n_l(self):
        return (self.lmax + 1) ** 2

    def c_struct(self):
        f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        self._keep = [f64(self.gvec), f64(self.tau), np.ascontiguousarray(self.atom_type, dtype=np.int32),
                      f64(self.rmt), f64(self.u), f64(self.du), f64(self.udot), f64(self.dudot),
                      f64(self.udot_norm)]
        nlv = self.lmax + 1
        for name, a in zip(("u", "du", "udot", "dudot", "udot_norm"), self._keep[4:]):
            if a.shape != (self.n_types, nlv):
                raise DimensionError(f"{name}: expected shape {(self.n_types, nlv)}")
        if self.gvec.shape[1:] != (3,) or self.tau.shape[1:] != (3,) or self.atom_type.shape != (self.n_atoms,):
            raise DimensionError("gvec/tau must be (n, 3) and atom_type (n_atoms,)")
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)
        return _Lapw(self.n_atoms, self.n_types, self.n_g, int(self.lmax), (C.c_double * 3)(*map(float, self.kpt)),
                     float(self.omega), *[ptr(a) for a in self._keep])


def make_lapw_system(n_atoms, lmax, n_g, n_types=2, seed=1, volume_per_atom=120.0):
    """Deterministic synthetic system: cubic cell (Omega = n_atoms * volume_per_atom bohr^3),
    atoms on a jittered simple-cubic sub-grid, the n_g shortest k+G of the cubic reciprocal
    lattice, radial boundary values with the LAPW Wronskian normalisation
    R^2 (u udot' - udot u') = -1 (so the matching system is never singular)."""
    if n_atoms < 1 or lmax < 0 or n_g < 1 or n_types < 1:
        raise DimensionError("make_lapw_system: bad dims")
    rng = np.random.default_rng(seed)
    omega = n_atoms * volume_per_atom
    a = omega ** (1.0 / 3.0)
    m = int(math.ceil(n_atoms ** (1.0 / 3.0) - 1e-9))
    idx = np.array([(i, j, k) for i in range(m) for j in range(m) for k in range(m)][:n_atoms], dtype=np.float64)
    tau = (idx + 0.5 + 0.05 * rng.uniform(-1, 1, size=idx.shape)) * (a / m)
    atom_type = (np.arange(n_atoms) % n_types).astype(np.int32)
    b = 2.0 * math.pi / a
    kpt = np.array([0.1, 0.2, 0.3]) * b
    r = int(math.ceil((3.0 * n_g / (4.0 * math.pi)) ** (1.0 / 3.0))) + 2
    while True:
        n = np.arange(-r, r + 1)
        g = np.stack(np.meshgrid(n, n, n, indexing="ij"), -1).reshape(-1, 3).astype(np.float64) * b
        kg = np.linalg.norm(g + kpt, axis=1)
        if np.sum(kg <= (r - 0.5) * b) >= n_g:
            break
        r += 2
    order = np.lexsort((g[:, 2], g[:, 1], g[:, 0], np.round(kg, 12)))
    gvec = np.ascontiguousarray(g[order[:n_g]])
    rmt = 2.0 + 0.2 * np.arange(n_types)
    nlv = lmax + 1
    u = rng.uniform(0.5, 1.5, size=(n_types, nlv))
    du = rng.uniform(-1.0, 1.0, size=(n_types, nlv))
    udot = rng.uniform(-1.0, 1.0, size=(n_types, nlv))
    dudot = (udot * du - 1.0 / rmt[:, None] ** 2) / u  # u udot' - udot u' = -1/R^2
    udot_norm = rng.uniform(0.5, 1.5, size=(n_types, nlv))
    return LapwSystem(lmax, kpt, omega, gvec, tau, atom_type, rmt, u, du, udot, dudot, udot_norm)


def lapw_coefficients(sys_: LapwSystem, device=0):
    """A, B ((n_atoms N_L) x n_g complex128, Fortran order) and U (N_L, n_atoms) on the GPU."""
    K = sys_.n_atoms * sys_.n_l
    A = np.empty((K, sys_.n_g), np.complex128, order="F")
    B = np.empty((K, sys_.n_g), np.complex128, order="F")
    U = np.empty((sys_.n_l, sys_.n_atoms), np.float64, order="F")
    cs = sys_.c_struct()
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    check(_lib.lib().hsdla_b200_lapw_coefficients(C.c_int(device), C.byref(cs), ptr(A), ptr(B), ptr(U)),
          "lapw_coefficients")
    return A, B, U


def _engine_setup_lapw(eng, sys_, atom_begin=0):
    cs = sys_.c_struct()
    check(_lib.lib().hsdla_b200_engine_setup_lapw(eng.h, C.byref(cs), C.c_uint64(atom_begin)), "engine_setup_lapw")


def _engine_upload_operators(eng, T_AA, T_AB, T_BB, atom_begin=0):
    f = [np.asfortranarray(T, dtype=np.complex128) for T in (T_AA, T_AB, T_BB)]
    eng._ops_keep = f
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    check(_lib.lib().hsdla_b200_engine_upload_operators(eng.h, *[ptr(a) for a in f], C.c_uint64(atom_begin)),
          "engine_upload_operators")


def _engine_setup_time(eng):
    """CUDA-event times of the last setup: ms (tables + stream kernels), stream_ms (the
    HBM-write stream kernel alone) and the bytes written."""
    ms, nb, ms_s = C.c_double(), C.c_uint64(), C.c_double()
    check(_lib.lib().hsdla_b200_engine_setup_time(eng.h, C.byref(ms), C.byref(nb), C.byref(ms_s)),
          "engine_setup_time")
    return {"ms": ms.value, "bytes": nb.value, "stream_ms": ms_s.value}


Engine.setup_lapw = _engine_setup_lapw
Engine.upload_operators = _engine_upload_operators
Engine.setup_time = _engine_setup_time


def build_hs_lapw(sys_: LapwSystem, T_AA, T_AB, T_BB, algo="merged", device=0) -> HSResult:
    """H and S of one k-point straight from the LAPW description: A, B, U are built in
    HBM by the setup kernel (never cross PCIe), T operators are uploaded, then the
    refined H/S build runs.  T_*: complex128 (N_L, N_L, n_atoms) Fortran order."""
    if algo not in ALGOS:
        raise ConfigError(f"unknown algo: {algo}")
    nl = sys_.n_l
    for T in (T_AA, T_AB, T_BB):
        if T.shape != (nl, nl, sys_.n_atoms):
            raise DimensionError(f"T operators must be ({nl}, {nl}, {sys_.n_atoms})")
    eng = Engine(device, sys_.n_atoms, nl, sys_.n_g)
    try:
        eng.set_download_overlap(True)
        eng.setup_lapw(sys_)
        eng.upload_operators(T_AA, T_AB, T_BB)
        eng.build(algo)
        st = eng.sync()
        H, S = eng.download()
        led = flop_model(SimpleNamespace(n_atoms=sys_.n_atoms, n_l=nl, n_g=sys_.n_g, hpd_flags=None))
    finally:
        eng.close()
    phases = [PhaseTime(k, v) for k, v in st["phase_seconds"].items()]
    return HSResult(H, S, led, st["peak_temp_bytes"], phases, [], st)
