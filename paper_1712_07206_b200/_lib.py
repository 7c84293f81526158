"""ctypes binding of the C-ABI in include/hsdla_b200.h (libhsdla_b200.so, built in-tree).

The product path is this shared library only: there is no CPU fallback.  If the
library is missing the import of anything that computes raises loudly.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhsdla_b200.so")

OK, DIMENSION_ERROR, SIZING_ERROR, CONFIG_ERROR, IO_ERROR, CUDA_ERROR, NCCL_ERROR = range(7)
ALGO_REFINED_MERGED, ALGO_REFINED, ALGO_ORIGINAL, ALGO_REFINED_FUSED = 0, 1, 2, 3
ARITH = {"3m": 0, "4m": 1}  # HSDLA_B200_ARITH_*: Gauss 3-multiplication / plain 4-multiplication complex
FLAG_ARITH_4M = 1
FLAG_REDUCE_ROOT = 2
REDUCE = {"root": 0, "scatter": 1}  # HSDLA_B200_REDUCE_*
LEDGER_KEYS = ("gemm", "hemm", "her2k", "herk", "scaling", "herkx", "potrf", "trmm")
N_PHASES = 8
# phase slot names (include/hsdla_b200.h HSDLA_B200_PHASE_*)
PHASE_SLOTS = ("s", "z_loop", "her2k", "hemm_loop", "herkx", "chol_loop", "h_aa_update", "")
# reported phases per variant, in the reference's order (test_pipeline.cpp:167-176)
PHASE_NAMES = ("s", "z_loop", "her2k", "hemm_loop", "herkx")
PHASE_NAMES_ORIGINAL = ("z_loop", "her2k", "s", "chol_loop", "h_aa_update")

# Every symbol include/hsdla_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "hsdla_b200_build_hs", "hsdla_b200_flop_model", "hsdla_b200_potrf", "hsdla_b200_generate_problem", "hsdla_b200_last_error",
    "hsdla_b200_device_count", "hsdla_b200_host_register", "hsdla_b200_host_unregister",
    "hsdla_b200_release_cache", "hsdla_b200_engine_create", "hsdla_b200_engine_destroy",
    "hsdla_b200_engine_upload", "hsdla_b200_engine_build", "hsdla_b200_engine_build_streamed", "hsdla_b200_engine_reduce",
    "hsdla_b200_engine_sync", "hsdla_b200_engine_download", "hsdla_b200_engine_device_results",
    "hsdla_b200_engine_stream", "hsdla_b200_nccl_unique_id", "hsdla_b200_engine_set_comm",
    "hsdla_b200_engine_kernel_times", "hsdla_b200_fp64_peak", "hsdla_b200_shard_atoms",
    "hsdla_b200_lapw_coefficients", "hsdla_b200_engine_setup_lapw", "hsdla_b200_engine_upload_operators",
    "hsdla_b200_engine_setup_time", "hsdla_b200_problem_file_info", "hsdla_b200_build_hs_file",
    "hsdla_b200_engine_load", "hsdla_b200_engine_fill_synthetic",
    "hsdla_b200_herk", "hsdla_b200_her2k", "hsdla_b200_herkx", "hsdla_b200_gemm", "hsdla_b200_hemm",
    "hsdla_b200_trmm", "hsdla_b200_diag_scale", "hsdla_b200_engine_set_arith", "hsdla_b200_set_default_arith",
    "hsdla_b200_engine_set_download_overlap", "hsdla_b200_build_hs_kpoints",
    "hsdla_b200_engine_create_shard", "hsdla_b200_engine_reshape", "hsdla_b200_engine_set_reduce_mode",
    "hsdla_b200_group_reduce", "hsdla_b200_engine_owned", "hsdla_b200_generate_problem_shard",
    "hsdla_b200_shard_rows",
)


class Problem(C.Structure):
    _fields_ = [("n_atoms", C.c_uint64), ("n_l", C.c_uint64), ("n_g", C.c_uint64),
                ("A", C.c_void_p), ("B", C.c_void_p), ("T_AA", C.c_void_p), ("T_AB", C.c_void_p),
                ("T_BB", C.c_void_p), ("U", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("n_gpus", C.c_int), ("device_ids", C.POINTER(C.c_int)), ("algo", C.c_int), ("flags", C.c_int),
                ("col_groups", C.c_int), ("mem_budget_gb", C.c_double)]


class Shard(C.Structure):
    _fields_ = [("n_atoms_local", C.c_uint64), ("n_l", C.c_uint64), ("n_g", C.c_uint64),
                ("col_begin", C.c_uint64), ("col_end", C.c_uint64), ("n_g_capacity", C.c_uint64),
                ("row_begin", C.c_uint64), ("row_end", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("phase_seconds", C.c_double * N_PHASES), ("h2d_seconds", C.c_double), ("device_seconds", C.c_double),
                ("reduce_seconds", C.c_double), ("d2h_seconds", C.c_double), ("total_seconds", C.c_double),
                ("ledger", C.c_uint64 * 9), ("executed_flops", C.c_uint64), ("peak_device_bytes", C.c_uint64),
                ("peak_temp_bytes", C.c_uint64), ("n_gpus", C.c_int), ("kernel_launches", C.c_int),
                ("n_hpd", C.c_uint64), ("col_groups", C.c_int), ("reduce_mode", C.c_int)]


_lib = None


def lib():
    """Load libhsdla_b200.so (fails loudly: the product has no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (no CPU fallback exists for the B200 path)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name in EXPORTS:
            getattr(L, name).restype = C.c_int
        L.hsdla_b200_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def last_error():
    return lib().hsdla_b200_last_error().decode(errors="replace")
