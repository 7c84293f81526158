"""HSDL v1 problem files streamed straight into HBM (hsdla_b200_build_hs_file /
hsdla_b200_engine_load; reference problem.cpp:144-243 format): the result equals
the host-buffer drop-in on the same instance, shards read only their rows."""
import os

import numpy as np
import pytest

import paper_1712_07206_b200 as hb
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    assert hb.device_count() > 0, "GPU tests need a CUDA device"
    yield
    hb.release_cache()


def rel(x, y):
    return hb.rel_frobenius_error_lower(x, y)


def test_reference_written_file(restatement):
    path = os.path.join(GOLDEN, "small_2_3_16_s1_nh1.hsdl")
    p = hb.generate_problem(2, 3, 16, 1, 1)
    H, S, led = restatement.build_hs_refined(p)
    for cfg in (hb.PipelineConfig(), hb.PipelineConfig(algo="refined"), hb.PipelineConfig(variant="original")):
        r = hb.build_hs_file(path, cfg)
        assert rel(r.H, H) <= TOL and rel(r.S, S) <= TOL
        iu = np.triu_indices(16, 1)
        assert np.all(r.H[iu] == 0) and np.all(r.S[iu] == 0)
        assert r.ledger == hb.flop_model(p, cfg.variant)


def test_file_equals_host_dropin_and_shards(tmp_path):
    """A multi-slab file (A, B > one 64 MB staging slab): build_hs_file == build_hs on
    the host problem, and two engines loading disjoint atom ranges of the same file
    (strided per-column reads) sum to the full result."""
    p = hb.generate_problem(24, 81, 2200, 9, 7)
    path = str(tmp_path / "p.hsdl")
    hb.save_problem(p, path)
    want = hb.build_hs_refined(p)
    got = hb.build_hs_file(path)
    assert rel(got.H, want.H) <= TOL and rel(got.S, want.S) <= TOL
    assert got.stats["h2d_seconds"] > 0
    o = hb.build_hs_file(path, hb.PipelineConfig(variant="original"))
    assert rel(o.H, want.H) <= TOL and o.stats["n_hpd"] == 24 - 7
    hb.release_cache()
    parts = []
    for a0, a1 in ((0, 11), (11, 24)):
        e = hb.Engine(0, a1 - a0, p.n_l, p.n_g)
        e.load(path, a0)
        e.build("fused")
        e.sync()
        parts.append(e.download())
        e.close()
    H = parts[0][0] + parts[1][0]
    S = parts[0][1] + parts[1][1]
    assert rel(H, want.H) <= TOL and rel(S, want.S) <= TOL


def test_engine_load_shape_mismatch(tmp_path):
    p = hb.generate_problem(4, 5, 30, 2, 0)
    path = str(tmp_path / "q.hsdl")
    hb.save_problem(p, path)
    e = hb.Engine(0, 3, 5, 31)
    with pytest.raises(hb.DimensionError):
        e.load(path, 0)
    e.close()
    e = hb.Engine(0, 3, 5, 30)
    with pytest.raises(hb.DimensionError):
        e.load(path, 2)  # atoms 2..4 exceed the file's 4 atoms
    e.close()


def test_file_view_follows_a_rewritten_file(tmp_path):
    """The engine keeps a read-only mapping of the last file it loaded; rewriting the file
    (same shape, other values) between calls must remap it, so the second build sees the
    new contents, and the same file again reproduces the first result bit for bit."""
    path = str(tmp_path / "p.hsdl")
    p1 = hb.generate_problem(6, 25, 400, 1, 0)
    p2 = hb.generate_problem(6, 25, 400, 2, 0)
    hb.save_problem(p1, path)
    r1 = hb.build_hs_file(path)
    hb.save_problem(p2, path)
    os.utime(path, ns=(0, os.stat(path).st_mtime_ns + 1_000_000))  # a distinct mtime even on coarse clocks
    r2 = hb.build_hs_file(path)
    w2 = hb.build_hs_refined(p2)
    assert rel(r2.H, w2.H) <= TOL and rel(r2.S, w2.S) <= TOL
    assert rel(r2.H, r1.H) > 1e-3
    hb.save_problem(p1, path)
    r3 = hb.build_hs_file(path)
    assert np.array_equal(r3.H, r1.H) and np.array_equal(r3.S, r1.S)


def test_truncated_file_is_an_io_error(tmp_path):
    """A file cut short after its header: IoError from the loader, never a crash."""
    p = hb.generate_problem(4, 9, 300, 3, 0)
    path = str(tmp_path / "t.hsdl")
    hb.save_problem(p, path)
    size = os.path.getsize(path)
    with open(path, "r+b") as f:
        f.truncate(size // 2)
    with pytest.raises(hb.IoError):
        hb.build_hs_file(path)
