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
