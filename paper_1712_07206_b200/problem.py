"""ProblemInstance, the synthetic generator, presets and the HSDL v1 file format.

Mirrors hsdla::ProblemInstance (proj/include/hsdla/problem.hpp:16-27) with numpy
storage that is byte-identical to the reference's column-major
std::complex<double> layout:

* ``A``, ``B``: complex128 (n_atoms*n_l, n_g), Fortran order (ld = n_atoms*n_l),
  atom a = rows [a*n_l, (a+1)*n_l).
* ``T_AA``, ``T_AB``, ``T_BB``: complex128 (n_l, n_l, n_atoms), Fortran order, so
  ``T[:, :, a]`` is atom a's column-major block and blocks are contiguous.
  T_AA / T_BB are Hermitian with the LOWER triangle authoritative.
* ``U``: float64 (n_l, n_atoms), Fortran order (``U[:, a]`` = atom a's diagonal).
"""
import ctypes as C
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DimensionError, IoError, SizingError, check


@dataclass
class ProblemInstance:
    n_atoms: int
    n_l: int
    n_g: int
    A: np.ndarray
    B: np.ndarray
    T_AA: np.ndarray
    T_AB: np.ndarray
    T_BB: np.ndarray
    U: np.ndarray
    hpd_flags: np.ndarray = field(default=None)

    def validate(self):
        na, nl, ng = self.n_atoms, self.n_l, self.n_g
        if na < 1 or nl < 1 or ng < 1:
            raise DimensionError("all dims must be >= 1")
        K = na * nl
        for name, arr, shape, dt in (("A", self.A, (K, ng), np.complex128), ("B", self.B, (K, ng), np.complex128),
                                     ("T_AA", self.T_AA, (nl, nl, na), np.complex128),
                                     ("T_AB", self.T_AB, (nl, nl, na), np.complex128),
                                     ("T_BB", self.T_BB, (nl, nl, na), np.complex128),
                                     ("U", self.U, (nl, na), np.float64)):
            if arr is None or tuple(arr.shape) != shape:
                raise DimensionError(f"{name}: expected shape {shape}, got {None if arr is None else arr.shape}")
            if arr.dtype != dt:
                raise DimensionError(f"{name}: expected dtype {np.dtype(dt)}, got {arr.dtype}")
            if not arr.flags.f_contiguous:
                raise DimensionError(f"{name}: must be Fortran-contiguous (column-major)")
        return self

    def c_struct(self):
        self.validate()
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)
        return _lib.Problem(self.n_atoms, self.n_l, self.n_g, ptr(self.A), ptr(self.B), ptr(self.T_AA),
                            ptr(self.T_AB), ptr(self.T_BB), ptr(self.U))


def empty_problem(n_atoms, n_l, n_g):
    K = n_atoms * n_l
    if K * n_g > (1 << 62) // 16:
        raise SizingError("problem allocation overflows")
    return ProblemInstance(
        n_atoms, n_l, n_g,
        np.empty((K, n_g), np.complex128, order="F"), np.empty((K, n_g), np.complex128, order="F"),
        np.empty((n_l, n_l, n_atoms), np.complex128, order="F"),
        np.empty((n_l, n_l, n_atoms), np.complex128, order="F"),
        np.empty((n_l, n_l, n_atoms), np.complex128, order="F"),
        np.empty((n_l, n_atoms), np.float64, order="F"), np.zeros(n_atoms, np.bool_))


def generate_problem(n_atoms, n_l, n_g, seed=1, n_not_hpd=0):
    """hsdla::generate_problem (problem.cpp:79-142), bit-identical (C++ in libhsdla_b200)."""
    if n_atoms < 1 or n_l < 1 or n_g < 1:
        raise DimensionError("generate_problem: all dims must be >= 1")
    if n_not_hpd > n_atoms:
        raise DimensionError("generate_problem: n_not_hpd > n_atoms")
    p = empty_problem(n_atoms, n_l, n_g)
    hpd = np.zeros(n_atoms, np.uint8)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    check(_lib.lib().hsdla_b200_generate_problem(
        C.c_uint64(n_atoms), C.c_uint64(n_l), C.c_uint64(n_g), C.c_uint64(seed), C.c_uint64(n_not_hpd),
        ptr(p.A), ptr(p.B), ptr(p.T_AA), ptr(p.T_AB), ptr(p.T_BB), ptr(p.U), ptr(hpd)), "generate_problem")
    p.hpd_flags = hpd.astype(np.bool_)
    return p


def generate_problem_shard(n_atoms, n_l, n_g, atom_begin, atom_end, seed=1, n_not_hpd=0):
    """Atoms [atom_begin, atom_end) of generate_problem(n_atoms, n_l, n_g, seed, n_not_hpd), bit-identical
    to the same rows / blocks of the full instance, generated without the other atoms' storage (each
    rank of a multi-GPU run builds only its own shard).  Returns a ProblemInstance of atom_end -
    atom_begin atoms; its `atom_begin` / `n_atoms_total` attributes record where it sits."""
    if n_atoms < 1 or n_l < 1 or n_g < 1:
        raise DimensionError("generate_problem_shard: all dims must be >= 1")
    if n_not_hpd > n_atoms or not 0 <= atom_begin < atom_end <= n_atoms:
        raise DimensionError("generate_problem_shard: need n_not_hpd <= n_atoms, 0 <= atom_begin < atom_end <= n_atoms")
    na = atom_end - atom_begin
    p = empty_problem(na, n_l, n_g)
    hpd = np.zeros(na, np.uint8)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    check(_lib.lib().hsdla_b200_generate_problem_shard(
        C.c_uint64(n_atoms), C.c_uint64(n_l), C.c_uint64(n_g), C.c_uint64(seed), C.c_uint64(n_not_hpd),
        C.c_uint64(atom_begin), C.c_uint64(atom_end), ptr(p.A), ptr(p.B), ptr(p.T_AA), ptr(p.T_AB), ptr(p.T_BB),
        ptr(p.U), ptr(hpd)), "generate_problem_shard")
    p.hpd_flags = hpd.astype(np.bool_)
    p.atom_begin, p.n_atoms_total = atom_begin, n_atoms
    return p


# ---- presets (problem.cpp:247-270) -----------------------------------------
@dataclass
class Preset:
    name: str
    n_atoms: int
    n_l: int
    n_g: int


_PRESETS = [
    Preset("nacl-2.5", 512, 49, 2256), Preset("nacl-3.0", 512, 49, 3893),
    Preset("nacl-3.5", 512, 49, 6217), Preset("nacl-4.0", 512, 49, 9273),
    Preset("auag-2.5", 108, 121, 3275), Preset("auag-3.0", 108, 121, 5638),
    Preset("auag-3.5", 108, 121, 8970), Preset("auag-4.0", 108, 121, 13379),
    Preset("tio2-2.5", 384, 81, 7094), Preset("tio2-3.0", 384, 81, 12293),
    Preset("tio2-3.5", 384, 81, 19553), Preset("tio2-4.0", 384, 81, 29144),
]


def presets():
    return list(_PRESETS)


def find_preset(name, scale=1.0):
    for p in _PRESETS:
        if p.name == name:
            sc = lambda d: int(math.ceil(d * scale))
            return Preset(p.name, sc(p.n_atoms), sc(p.n_l), sc(p.n_g))
    return None


# ---- HSDL v1 binary file (problem.cpp:144-243) -------------------------------
_MAGIC = b"HSDL"
_VERSION = 1


def save_problem(p, path):
    """Write the reference's "HSDL" v1 format (save_problem, problem.cpp:172-195)."""
    p.validate()
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC)
            f.write(struct.pack("<I", _VERSION))
            f.write(struct.pack("<3Q", p.n_atoms, p.n_l, p.n_g))
            flags = np.zeros((p.n_atoms + 7) // 8, np.uint8)
            hpd = np.ones(p.n_atoms, bool) if p.hpd_flags is None else np.asarray(p.hpd_flags, bool)
            for a in range(p.n_atoms):
                if hpd[a]:
                    flags[a // 8] |= 1 << (a % 8)
            f.write(flags.tobytes())
            f.write(p.A.tobytes(order="F"))
            f.write(p.B.tobytes(order="F"))
            for a in range(p.n_atoms):
                f.write(p.T_AA[:, :, a].tobytes(order="F"))
                f.write(p.T_AB[:, :, a].tobytes(order="F"))
                f.write(p.T_BB[:, :, a].tobytes(order="F"))
            f.write(p.U.tobytes(order="F"))
    except OSError as e:
        raise IoError(f"write failed: {path}: {e}") from e


def load_problem(path):
    """Read the "HSDL" v1 format (load_problem, problem.cpp:197-243); IoError on
    bad magic, unsupported version or truncation."""
    try:
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"cannot open: {path}") from e
    with f:
        def read(n):
            b = f.read(n)
            if len(b) != n:
                raise IoError("problem file truncated")
            return b

        if read(4) != _MAGIC:
            raise IoError(f"bad magic: {path}")
        (version,) = struct.unpack("<I", read(4))
        if version != _VERSION:
            raise IoError(f"unsupported format version {version}")
        na, nl, ng = struct.unpack("<3Q", read(24))
        if na * nl * ng * 16 > (1 << 62):
            raise SizingError("problem allocation overflows")
        flags = np.frombuffer(read((na + 7) // 8), np.uint8)
        p = empty_problem(na, nl, ng)
        p.hpd_flags = np.array([(flags[a // 8] >> (a % 8)) & 1 for a in range(na)], dtype=bool)
        K = na * nl
        p.A[...] = np.frombuffer(read(K * ng * 16), np.complex128).reshape((K, ng), order="F")
        p.B[...] = np.frombuffer(read(K * ng * 16), np.complex128).reshape((K, ng), order="F")
        blk = nl * nl * 16
        for a in range(na):
            p.T_AA[:, :, a] = np.frombuffer(read(blk), np.complex128).reshape((nl, nl), order="F")
            p.T_AB[:, :, a] = np.frombuffer(read(blk), np.complex128).reshape((nl, nl), order="F")
            p.T_BB[:, :, a] = np.frombuffer(read(blk), np.complex128).reshape((nl, nl), order="F")
        p.U[...] = np.frombuffer(read(na * nl * 8), np.float64).reshape((nl, na), order="F")
        return p
