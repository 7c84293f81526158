"""Host-side mirror of the reference pipeline API for the B200 strategy.

Reference interface mirrored (names, argument meaning, error behaviour):
  hsdla::pipeline::build_hs_original / build_hs_refined / build_hs / flop_model   pipeline.hpp:47-62
  hsdla::kernels::potrf (batched over atom blocks)                 kernels.hpp:63-71
  PipelineConfig / HSResult / PhaseTime / FlopLedger              pipeline.hpp:22-44, flop_ledger.hpp
  HermitianView::mirror, rel_frobenius_error_lower               complex_matrix.hpp:62-94
All arithmetic runs in libhsdla_b200.so on the GPU; nothing here computes H or S.
"""
import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import ConfigError, DimensionError, check

VARIANTS = ("original", "refined")
STRATEGIES = ("b200",)
ALGOS = {"merged": _lib.ALGO_REFINED_MERGED, "fused": _lib.ALGO_REFINED_FUSED, "refined": _lib.ALGO_REFINED,
         "original": _lib.ALGO_ORIGINAL}
REFINED_ALGOS = ("merged", "fused", "refined")


def _algo_warnings(algo):
    if algo == "fused":
        return ["herkx fused into the her2k contraction (phase time 0)"]
    if algo == "merged":
        return ["her2k, hemm_loop and herkx merged: z_loop builds W = M Y per atom, her2k is the one H "
                "contraction [A;B]^H W (hemm_loop, herkx 0 s)"]
    return []


def parse_variant(s):
    if s not in VARIANTS:
        raise ConfigError(f"unknown variant: {s}")
    return s


def parse_strategy(s):
    """The B200 build provides one strategy.  The reference's cpu/static/dynamic
    strategies (pipeline.hpp:15) are host-CPU paths and are not part of it."""
    if s not in STRATEGIES:
        raise ConfigError(f"unknown strategy: {s} (the B200 build implements: {', '.join(STRATEGIES)})")
    return s


@dataclass
class PipelineConfig:
    variant: str = "refined"
    strategy: str = "b200"
    n_gpus: int = 1
    device_ids: Optional[Sequence[int]] = None
    # refined variant only: "merged" (default: H = [A;B]^H [W_A;W_B], 16 K N_G^2 contraction flops) |
    # "fused" (her2k+herkx in one contraction over [Z;B;A], 20 K N_G^2) | "refined" (reference phase order)
    algo: str = "merged"
    # complex arithmetic of the contractions: "3m" (Gauss, 6 executed flops per complex MAC,
    # the default) | "4m" (four real multiplications, plain FP64 rounding per product)
    arith: str = "3m"
    # multi-GPU: "scatter" (default: every GPU receives and downloads its own slices of H, S) |
    # "root" (ncclReduce onto the first GPU, which downloads everything)
    reduce: str = "scatter"
    # 2-D tiling of H, S into column windows (0: automatic, by the per-GPU memory budget)
    col_groups: int = 0
    mem_budget_gb: float = 0.0


@dataclass
class PhaseTime:
    name: str
    seconds: float


class FlopLedger:
    """Per-kernel integer real-flop counts, complex MAC = 8 (flop_ledger.hpp:9-35)."""

    def __init__(self, counts=None):
        self._counts = {k: int(v) for k, v in (counts or {}).items() if int(v) != 0}

    @classmethod
    def from_array(cls, arr):
        return cls({k: int(v) for k, v in zip(_lib.LEDGER_KEYS, list(arr)[:8])})

    def add(self, kernel, flops):
        self._counts[kernel] = self._counts.get(kernel, 0) + int(flops)

    def total(self):
        return sum(self._counts.values())

    def count(self, kernel):
        return self._counts.get(kernel, 0)

    def counts(self):
        return dict(sorted(self._counts.items()))

    def __eq__(self, other):
        return isinstance(other, FlopLedger) and self.counts() == other.counts()

    def __repr__(self):
        return f"FlopLedger({self.counts()}, total={self.total()})"


@dataclass
class HSResult:
    H: np.ndarray  # (n_g, n_g) complex128, Fortran order; lower triangle authoritative, upper exactly 0
    S: np.ndarray
    ledger: FlopLedger
    peak_temp_bytes: int = 0
    phases: List[PhaseTime] = field(default_factory=list)
    warnings: List[str] = field(default_factory=list)
    stats: dict = field(default_factory=dict)


def _options(cfg, algo):
    ids = None
    if cfg.device_ids is not None:
        if len(cfg.device_ids) < cfg.n_gpus:
            raise ConfigError("device_ids shorter than n_gpus")
        ids = (C.c_int * len(cfg.device_ids))(*cfg.device_ids)
    if cfg.n_gpus < 1:
        raise ConfigError("n_gpus must be >= 1")
    if cfg.arith not in _lib.ARITH:
        raise ConfigError(f"unknown arith: {cfg.arith} (3m | 4m)")
    if cfg.reduce not in _lib.REDUCE:
        raise ConfigError(f"unknown reduce: {cfg.reduce} (scatter | root)")
    flags = (_lib.FLAG_ARITH_4M if cfg.arith == "4m" else 0) | (_lib.FLAG_REDUCE_ROOT if cfg.reduce == "root" else 0)
    return _lib.Options(int(cfg.n_gpus), ids, ALGOS[algo], flags, int(cfg.col_groups), float(cfg.mem_budget_gb)), ids


def _phase_names(algo):
    return _lib.PHASE_NAMES_ORIGINAL if algo == "original" else _lib.PHASE_NAMES


def _phases(st, algo):
    slot = {n: i for i, n in enumerate(_lib.PHASE_SLOTS)}
    return [PhaseTime(nm, float(st.phase_seconds[slot[nm]])) for nm in _phase_names(algo)]


def stats_dict(st, algo="merged"):
    return {
        "phase_seconds": {ph.name: ph.seconds for ph in _phases(st, algo)}, "n_hpd": int(st.n_hpd),
        "h2d_seconds": st.h2d_seconds, "device_seconds": st.device_seconds, "reduce_seconds": st.reduce_seconds,
        "d2h_seconds": st.d2h_seconds, "total_seconds": st.total_seconds,
        "ledger_total": int(st.ledger[8]), "executed_flops": int(st.executed_flops),
        "peak_device_bytes": int(st.peak_device_bytes), "peak_temp_bytes": int(st.peak_temp_bytes),
        "n_gpus": st.n_gpus, "kernel_launches": st.kernel_launches, "col_groups": st.col_groups,
        "reduce": {v: k for k, v in _lib.REDUCE.items()}.get(st.reduce_mode, "root"),
    }


def _run(p, cfg, algo, H, S, what):
    parse_strategy(cfg.strategy)
    prob = p.c_struct()
    n = p.n_g
    if H is None:
        H = np.zeros((n, n), np.complex128, order="F")
    if S is None:
        S = np.zeros((n, n), np.complex128, order="F")
    for name, M in (("H", H), ("S", S)):
        if M.shape != (n, n) or M.dtype != np.complex128 or not M.flags.f_contiguous:
            raise DimensionError(f"{name} must be a ({n}, {n}) complex128 Fortran array")
    opts, _keep = _options(cfg, algo)
    st = _lib.Stats()
    check(_lib.lib().hsdla_b200_build_hs(C.byref(prob), C.byref(opts), H.ctypes.data_as(C.c_void_p),
                                         S.ctypes.data_as(C.c_void_p), C.byref(st)), what)
    warnings = _algo_warnings(algo)
    return HSResult(H, S, FlopLedger.from_array(st.ledger), int(st.peak_temp_bytes), _phases(st, algo), warnings,
                    stats_dict(st, algo))


def build_hs_refined(p, cfg: Optional[PipelineConfig] = None, H=None, S=None) -> HSResult:
    """build_hs_refined (pipeline.cpp:281-329) on B200.  ``H``/``S`` may be passed
    preallocated (n_g x n_g complex128, Fortran order); only their lower triangles
    are written.  Fresh outputs have exactly-zero upper triangles."""
    cfg = cfg or PipelineConfig()
    if parse_variant(cfg.variant) != "refined":
        raise ConfigError("build_hs_refined needs variant 'refined' (use build_hs / build_hs_original)")
    if cfg.algo not in REFINED_ALGOS:
        raise ConfigError(f"unknown algo: {cfg.algo}")
    return _run(p, cfg, cfg.algo, H, S, "build_hs_refined")


def build_hs_kpoints(p, As, Bs, cfg: Optional[PipelineConfig] = None, Hs=None, Ss=None):
    """n k-points of one cell in one call (hsdla_b200_build_hs_kpoints): p's operators and U are
    shared, As[k] / Bs[k] are each k-point's coefficients ((n_atoms n_l) x N_G(k), p.A's layout;
    N_G(k) may differ per k-point).  Uploads of k+1 and downloads of k-1 overlap the build of k.
    Returns (list of (H, S) pairs, stats of the last k-point with total_seconds for the batch)."""
    cfg = cfg or PipelineConfig()
    parse_strategy(cfg.strategy)
    algo = "original" if parse_variant(cfg.variant) == "original" else cfg.algo
    if algo not in ALGOS:
        raise ConfigError(f"unknown algo: {algo}")
    nk = len(As)
    if len(Bs) != nk:
        raise DimensionError("As and Bs differ in length")
    K = p.n_atoms * p.n_l
    ngk = []
    for A_, B_ in zip(As, Bs):
        for M in (A_, B_):
            if M.ndim != 2 or M.shape[0] != K or M.dtype != np.complex128 or not M.flags.f_contiguous:
                raise DimensionError(f"A/B must be ({K}, N_G(k)) complex128 Fortran arrays")
        if A_.shape != B_.shape:
            raise DimensionError("A[k] and B[k] differ in shape")
        ngk.append(A_.shape[1])
    Hs = Hs or [np.zeros((n, n), np.complex128, order="F") for n in ngk]
    Ss = Ss or [np.zeros((n, n), np.complex128, order="F") for n in ngk]
    for n, H_, S_ in zip(ngk, Hs, Ss):
        for M in (H_, S_):
            if M.shape != (n, n) or M.dtype != np.complex128 or not M.flags.f_contiguous:
                raise DimensionError(f"H/S must be ({n}, {n}) complex128 Fortran arrays")
    prob = p.c_struct()
    opts, _keep = _options(cfg, algo)
    ptrs = lambda L: (C.c_void_p * nk)(*[M.ctypes.data for M in L])  # noqa: E731
    ng_arr = (C.c_uint64 * max(nk, 1))(*ngk)
    st = _lib.Stats()
    check(_lib.lib().hsdla_b200_build_hs_kpoints(C.byref(prob), C.c_uint64(nk), ng_arr, ptrs(As), ptrs(Bs),
                                                 C.byref(opts), ptrs(Hs), ptrs(Ss), C.byref(st)), "build_hs_kpoints")
    return list(zip(Hs, Ss)), stats_dict(st, algo)


def build_hs_original(p, cfg: Optional[PipelineConfig] = None, H=None, S=None) -> HSResult:
    """build_hs_original (pipeline.cpp:189-279, paper Algorithm 1) on B200: Cholesky
    try/fail of every T_AA on the GPU, trmm / hemm per atom, H += herk(B_T) +
    lower(A_f^H B_B).  Phases z_loop, her2k, s, chol_loop, h_aa_update; ledger ==
    flop_model(p, "original") with the observed potrf outcomes."""
    cfg = cfg or PipelineConfig(variant="original")
    return _run(p, cfg, "original", H, S, "build_hs_original")


def problem_file_info(path):
    """Header of an HSDL v1 file (problem.cpp:197-225) read natively: (n_atoms, n_l,
    n_g, hpd_flags).  IoError on a missing / malformed / truncated file."""
    na, nl, ng = C.c_uint64(), C.c_uint64(), C.c_uint64()
    bpath = os.fsencode(path)
    check(_lib.lib().hsdla_b200_problem_file_info(bpath, C.byref(na), C.byref(nl), C.byref(ng), None),
          "problem_file_info")
    hpd = np.zeros(na.value, np.uint8)
    check(_lib.lib().hsdla_b200_problem_file_info(bpath, None, None, None, hpd.ctypes.data_as(C.c_void_p)),
          "problem_file_info")
    return na.value, nl.value, ng.value, hpd.astype(bool)


def build_hs_file(path, cfg: Optional[PipelineConfig] = None, H=None, S=None) -> HSResult:
    """build_hs(load_problem(path), cfg) with the file streamed shard by shard
    straight into HBM (no host ProblemInstance)."""
    cfg = cfg or PipelineConfig()
    parse_strategy(cfg.strategy)
    algo = "original" if parse_variant(cfg.variant) == "original" else cfg.algo
    if algo not in ALGOS:
        raise ConfigError(f"unknown algo: {algo}")
    _na, _nl, n, _hpd = problem_file_info(path)
    if H is None:
        H = np.zeros((n, n), np.complex128, order="F")
    if S is None:
        S = np.zeros((n, n), np.complex128, order="F")
    for name, M in (("H", H), ("S", S)):
        if M.shape != (n, n) or M.dtype != np.complex128 or not M.flags.f_contiguous:
            raise DimensionError(f"{name} must be a ({n}, {n}) complex128 Fortran array")
    opts, _keep = _options(cfg, algo)
    st = _lib.Stats()
    check(_lib.lib().hsdla_b200_build_hs_file(os.fsencode(path), C.byref(opts), H.ctypes.data_as(C.c_void_p),
                                              S.ctypes.data_as(C.c_void_p), C.byref(st)), "build_hs_file")
    warnings = _algo_warnings(algo)
    return HSResult(H, S, FlopLedger.from_array(st.ledger), int(st.peak_temp_bytes), _phases(st, algo), warnings,
                    stats_dict(st, algo))


def build_hs(p, cfg: PipelineConfig) -> HSResult:
    """build_hs (pipeline.cpp:331-334): dispatch on the variant."""
    if parse_variant(cfg.variant) == "original":
        return build_hs_original(p, cfg)
    return build_hs_refined(p, cfg)


def potrf(T, device=0):
    """kernels::potrf (kernels.cpp:417-436) on the GPU for every atom block of T
    ((n_l, n_l, n_blocks) complex128, Fortran order, lower triangles read).
    Returns (L, pivot): L[:, :, b] the factor (upper 0) where pivot[b] == -1, else the
    hemm fallback operand Q with Q^H = T[:, :, b] read from its lower triangle (full(T)
    with the diagonal conjugated); factors bit-identical to the reference's."""
    T = np.asfortranarray(T, dtype=np.complex128)
    if T.ndim == 2:
        T = T[:, :, None]
    if T.ndim != 3 or T.shape[0] != T.shape[1]:
        raise DimensionError("potrf: T must be (n_l, n_l, n_blocks)")
    n, nb = T.shape[0], T.shape[2]
    L = np.zeros_like(T, order="F")
    piv = np.zeros(nb, np.int64)
    check(_lib.lib().hsdla_b200_potrf(C.c_int(device), C.c_uint64(nb), C.c_uint64(n), T.ctypes.data_as(C.c_void_p),
                                      L.ctypes.data_as(C.c_void_p), piv.ctypes.data_as(C.c_void_p)), "potrf")
    return L, piv


def flop_model(p, variant="refined") -> FlopLedger:
    """Closed-form ledger (pipeline.cpp:336-364)."""
    parse_variant(variant)
    n_hpd = p.n_atoms if getattr(p, "hpd_flags", None) is None else int(np.sum(np.asarray(p.hpd_flags, bool)))
    out = (C.c_uint64 * 9)()
    check(_lib.lib().hsdla_b200_flop_model(C.c_int(0 if variant == "original" else 1), C.c_uint64(p.n_atoms),
                                           C.c_uint64(p.n_l), C.c_uint64(p.n_g), C.c_uint64(n_hpd), out),
          "flop_model")
    return FlopLedger.from_array(out)


def mirror(M):
    """HermitianView::mirror (complex_matrix.cpp:39-45), in place."""
    n = M.shape[0]
    iu = np.triu_indices(n, 1)
    M[iu] = np.conj(M.T[iu])
    M[np.diag_indices(n)] = M.diagonal().real
    return M


def rel_frobenius_error_lower(x, y):
    """complex_matrix.cpp:106-118."""
    if x.shape != y.shape or x.shape[0] != x.shape[1]:
        raise DimensionError("rel_frobenius_error_lower: shape mismatch")
    il = np.tril_indices(x.shape[0])
    d = np.linalg.norm((x - y)[il])
    r = np.linalg.norm(y[il])
    return float(d / max(r, 1e-300))


class Engine:
    """Device-resident engine for one shard on one GPU (C-ABI hsdla_b200_engine_*): n_atoms_local
    atoms (an atom shard) and the column window [col_begin, col_end) of H and S (col_end 0: n_g;
    2-D tiling: engines of different windows compute disjoint tile-column bands).  n_g_capacity
    sizes a whole-window engine for reshape() to larger N_G without reallocation.  [row_begin,
    row_end) restricts the H/S contractions to those rows of the shard's K (a row-balanced
    shard from shard_rows; row_end 0: all rows)."""

    def __init__(self, device, n_atoms_local, n_l, n_g, col_begin=0, col_end=0, n_g_capacity=0,
                 row_begin=0, row_end=0):
        h = C.c_void_p()
        sh = _lib.Shard(n_atoms_local, n_l, n_g, col_begin, col_end, n_g_capacity, row_begin, row_end)
        check(_lib.lib().hsdla_b200_engine_create_shard(C.c_int(device), C.byref(sh), C.byref(h)), "engine_create")
        self.h = h
        self.n_g = n_g
        self.device = device

    def reshape(self, n_g):
        """Re-target a whole-window engine at N_G = n_g within its capacity (inputs must be re-uploaded)."""
        check(_lib.lib().hsdla_b200_engine_reshape(self.h, C.c_uint64(n_g)), "engine_reshape")
        self.n_g = n_g

    def set_reduce_mode(self, mode):
        """"root" (ncclReduce onto the reduce root; the default) or "scatter" (every rank owns slices)."""
        if mode not in _lib.REDUCE:
            raise ConfigError(f"unknown reduce mode: {mode} (root | scatter)")
        check(_lib.lib().hsdla_b200_engine_set_reduce_mode(self.h, C.c_int(_lib.REDUCE[mode])), "set_reduce_mode")

    def owned(self):
        """Global packed-lower index ranges [(begin, end), ...] this engine holds final values for."""
        n = C.c_uint64()
        check(_lib.lib().hsdla_b200_engine_owned(self.h, None, C.c_uint64(0), C.byref(n)), "engine_owned")
        buf = (C.c_uint64 * max(1, 2 * n.value))()
        check(_lib.lib().hsdla_b200_engine_owned(self.h, buf, n, C.byref(n)), "engine_owned")
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)]

    def close(self):
        if self.h:
            _lib.lib().hsdla_b200_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, p, atom_begin=0):
        prob = p.c_struct()
        check(_lib.lib().hsdla_b200_engine_upload(self.h, C.byref(prob), C.c_uint64(atom_begin)), "engine_upload")

    def fill_synthetic(self, seed=1):
        """Device-side synthetic inputs (timing sweeps only; not the reference generator)."""
        check(_lib.lib().hsdla_b200_engine_fill_synthetic(self.h, C.c_uint64(seed)), "engine_fill_synthetic")

    def set_arith(self, arith):
        """Complex arithmetic of this engine's contractions: "3m" (default) or "4m"."""
        if arith not in _lib.ARITH:
            raise ConfigError(f"unknown arith: {arith} (3m | 4m)")
        check(_lib.lib().hsdla_b200_engine_set_arith(self.h, C.c_int(_lib.ARITH[arith])), "engine_set_arith")

    def set_download_overlap(self, on=True):
        """Band the final H contraction of this engine's builds so that a download issued right
        after build() overlaps it (hsdla_b200_engine_set_download_overlap)."""
        check(_lib.lib().hsdla_b200_engine_set_download_overlap(self.h, C.c_int(1 if on else 0)),
              "engine_set_download_overlap")

    def load(self, path, atom_begin=0):
        """Stream this shard of an HSDL v1 file into the engine (hsdla_b200_engine_load)."""
        check(_lib.lib().hsdla_b200_engine_load(self.h, os.fsencode(path), C.c_uint64(atom_begin)), "engine_load")

    def build(self, algo="merged"):
        self._algo = algo
        check(_lib.lib().hsdla_b200_engine_build(self.h, C.c_int(ALGOS[algo])), "engine_build")

    def build_streamed(self, p, atom_begin=0, algo="merged"):
        """Upload shard `atom_begin` of host problem p in atom chunks overlapped with the build."""
        self._prob = p.c_struct()  # keep the struct alive while the copies are in flight
        self._algo = algo
        check(_lib.lib().hsdla_b200_engine_build_streamed(self.h, C.byref(self._prob), C.c_uint64(atom_begin),
                                                          C.c_int(ALGOS[algo])), "engine_build_streamed")

    def reduce(self, root=0):
        check(_lib.lib().hsdla_b200_engine_reduce(self.h, C.c_int(root)), "engine_reduce")

    def sync(self):
        st = _lib.Stats()
        check(_lib.lib().hsdla_b200_engine_sync(self.h, C.byref(st)), "engine_sync")
        return stats_dict(st, getattr(self, "_algo", "merged"))

    def download(self, H=None, S=None):
        n = self.n_g
        if H is None:
            H = np.zeros((n, n), np.complex128, order="F")
        if S is None:
            S = np.zeros((n, n), np.complex128, order="F")
        check(_lib.lib().hsdla_b200_engine_download(self.h, H.ctypes.data_as(C.c_void_p),
                                                    S.ctypes.data_as(C.c_void_p)), "engine_download")
        return H, S

    def set_comm(self, uid: Optional[bytes], nranks, rank):
        buf = None if uid is None else C.create_string_buffer(uid, 128)
        check(_lib.lib().hsdla_b200_engine_set_comm(self.h, buf, C.c_int(nranks), C.c_int(rank)), "set_comm")

    def device_results(self):
        """Device pointers (ints) of the packed-lower H and S (LAPACK 'L' packed, column-major)."""
        h, s_ = C.c_void_p(), C.c_void_p()
        check(_lib.lib().hsdla_b200_engine_device_results(self.h, C.byref(h), C.byref(s_)), "engine_device_results")
        return h.value, s_.value

    def stream(self):
        s = C.c_void_p()
        check(_lib.lib().hsdla_b200_engine_stream(self.h, C.byref(s)), "engine_stream")
        return s.value

    def kernel_times(self, reset=False):
        """Mean CUDA-event duration of the S and H contraction launches over all
        builds since the last reset (recorded on the engine stream)."""
        ms_s, ms_h = C.c_double(), C.c_double()
        fs, fh, nb = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(_lib.lib().hsdla_b200_engine_kernel_times(self.h, C.c_int(1 if reset else 0), C.byref(ms_s),
                                                        C.byref(ms_h), C.byref(fs), C.byref(fh), C.byref(nb)),
              "kernel_times")
        return {"s_ms": ms_s.value, "h_ms": ms_h.value, "s_flops": fs.value, "h_flops": fh.value,
                "builds": nb.value}


def group_reduce(engines, mode="scatter", root=0):
    """hsdla_b200_group_reduce: sum the partial H, S of engines of this process that share a
    column window (disjoint atom shards; engines[r] is rank r): grouped NCCL calls when each has
    a communicator, else (one shared device) a deterministic sum kernel."""
    if mode not in _lib.REDUCE:
        raise ConfigError(f"unknown reduce mode: {mode} (root | scatter)")
    arr = (C.c_void_p * len(engines))(*[e.h.value for e in engines])
    check(_lib.lib().hsdla_b200_group_reduce(arr, C.c_int(len(engines)), C.c_int(_lib.REDUCE[mode]), C.c_int(root)),
          "group_reduce")


def set_default_arith(arith):
    """Process default complex arithmetic for new engines and the kernel layer ("3m" | "4m")."""
    if arith not in _lib.ARITH:
        raise ConfigError(f"unknown arith: {arith} (3m | 4m)")
    check(_lib.lib().hsdla_b200_set_default_arith(C.c_int(_lib.ARITH[arith])), "set_default_arith")


def fp64_peak(device=0, seconds=0.5):
    """Measured FP64 DMMA throughput (TFLOP/s) — the roofline denominator."""
    tf = C.c_double()
    check(_lib.lib().hsdla_b200_fp64_peak(C.c_int(device), C.c_double(seconds), C.byref(tf)), "fp64_peak")
    return tf.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_lib.lib().hsdla_b200_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


def shard_atoms(n_atoms, parts):
    """Contiguous count-balanced atom ranges (the engine's multi-GPU partition)."""
    out = (C.c_uint64 * (parts + 1))()
    check(_lib.lib().hsdla_b200_shard_atoms(C.c_uint64(n_atoms), C.c_int(parts), out), "shard_atoms")
    return [int(x) for x in out]


def shard_rows(n_atoms, n_l, parts):
    """Row-balanced shards (the multi-GPU drop-in's partition): the K = n_atoms n_l rows split
    evenly; a list of (atom_begin, n_atoms_local, row_begin, row_end) per part, rows local to the
    shard (Engine(..., row_begin=, row_end=))."""
    out = (C.c_uint64 * (4 * parts))()
    check(_lib.lib().hsdla_b200_shard_rows(C.c_uint64(n_atoms), C.c_uint64(n_l), C.c_int(parts), out), "shard_rows")
    return [tuple(int(x) for x in out[4 * r:4 * r + 4]) for r in range(parts)]


def device_count():
    n = C.c_int(0)
    check(_lib.lib().hsdla_b200_device_count(C.byref(n)), "device_count")
    return n.value


def host_register(arr):
    check(_lib.lib().hsdla_b200_host_register(arr.ctypes.data_as(C.c_void_p), C.c_size_t(arr.nbytes)),
          "host_register")


def host_unregister(arr):
    check(_lib.lib().hsdla_b200_host_unregister(arr.ctypes.data_as(C.c_void_p)), "host_unregister")


def release_cache():
    check(_lib.lib().hsdla_b200_release_cache(), "release_cache")
