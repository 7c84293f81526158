"""The C-ABI library loads and exports every symbol include/hsdla_b200.h declares
(no compute calls: this runs without a GPU)."""
import ctypes as C
import os
import re

import paper_1712_07206_b200 as hb
from paper_1712_07206_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hsdla_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hsdla_b200_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_library_is_sm100a_only():
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_status_codes_and_last_error():
    L = _lib.lib()
    rc = L.hsdla_b200_flop_model(C.c_int(1), C.c_uint64(1), C.c_uint64(1), C.c_uint64(1), C.c_uint64(1), None)
    assert rc == _lib.DIMENSION_ERROR
    assert "null" in _lib.last_error()
    n = C.c_int(-1)
    assert L.hsdla_b200_device_count(C.byref(n)) == 0 and n.value >= 0
    h = C.c_void_p()
    assert L.hsdla_b200_engine_create(C.c_int(0), C.c_uint64(0), C.c_uint64(1), C.c_uint64(1), C.byref(h)) == \
        _lib.DIMENSION_ERROR
    assert hb.flop_model(hb.empty_problem(2, 3, 4)).total() > 0


def test_library_then_torch_share_one_nccl():
    """Loading libhsdla_b200.so before torch must not break torch: both resolve the same
    libnccl.so.2 (the library links torch's bundled NCCL and records it as its RUNPATH)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import paper_1712_07206_b200 as hb; hb._lib.lib(); "
            "import torch, torch.distributed; print('ok', torch.__version__)" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_python_constants_match_the_header():
    """The ctypes mirror's algorithm / arithmetic numbering equals include/hsdla_b200.h."""
    from paper_1712_07206_b200.pipeline import ALGOS
    src = open(os.path.join(ROOT, "include", "hsdla_b200.h")).read()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define (HSDLA_B200_\w+)\s+(\d+)u?\b", src)}
    assert ALGOS == {"merged": defs["HSDLA_B200_ALGO_REFINED_MERGED"], "refined": defs["HSDLA_B200_ALGO_REFINED"],
                     "original": defs["HSDLA_B200_ALGO_ORIGINAL"], "fused": defs["HSDLA_B200_ALGO_REFINED_FUSED"]}
    assert _lib.ARITH == {"3m": defs["HSDLA_B200_ARITH_3M"], "4m": defs["HSDLA_B200_ARITH_4M"]}
    assert _lib.FLAG_ARITH_4M == defs["HSDLA_B200_FLAG_ARITH_4M"]
    assert _lib.FLAG_REDUCE_ROOT == defs["HSDLA_B200_FLAG_REDUCE_ROOT"]
    assert _lib.REDUCE == {"root": defs["HSDLA_B200_REDUCE_ROOT"], "scatter": defs["HSDLA_B200_REDUCE_SCATTER"]}


def test_ctypes_structs_match_the_header_layout():
    """Options / Shard field order and sizes as declared in include/hsdla_b200.h (the ctypes
    mirror must not drift from the C structs the library reads)."""
    import ctypes as C
    assert [f for f, _ in _lib.Options._fields_] == ["n_gpus", "device_ids", "algo", "flags", "col_groups",
                                                      "mem_budget_gb"]
    assert C.sizeof(_lib.Options) == 40  # int, pad, ptr, 3 x int, pad, double
    assert [f for f, _ in _lib.Shard._fields_] == ["n_atoms_local", "n_l", "n_g", "col_begin", "col_end",
                                                    "n_g_capacity", "row_begin", "row_end"]
    assert C.sizeof(_lib.Shard) == 64

