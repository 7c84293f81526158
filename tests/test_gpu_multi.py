"""Multi-GPU data plane: atom shards x column windows (2-D tiling of H and S), the reduce in
ROOT and SCATTER modes, ownership of the reduced ranges and the per-GPU downloads.

On one GPU the grid is EMULATED: several engines share device 0 and the engines of a window
are summed by a deterministic kernel instead of NCCL, with the same segments, ownership and
download code as the NCCL path (one GPU cannot host NCCL ranks that wait on each other).
Tests marked `multigpu` need >= 2 GPUs and run the real NCCL grid (single-process
ncclCommInitAll drop-in and the torchrun engine path); they skip on a 1-GPU box.

Bar (north_star): rel. Frobenius error of the lower triangle <= 1e-11 against the oracle /
the unmodified reference (oracle/_ref).  The sum over atoms the reduce relies on is
pipeline.cpp:296-324.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1712_07206_b200 as hb

pytestmark = pytest.mark.gpu
TOL = 1e-11
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(x, y):
    return hb.rel_frobenius_error_lower(x, y)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    assert hb.device_count() > 0, "GPU tests need a CUDA device"
    yield
    hb.release_cache()


def _shard(p, a0, a1):
    K0, K1 = a0 * p.n_l, a1 * p.n_l
    f = np.asfortranarray
    return hb.ProblemInstance(a1 - a0, p.n_l, p.n_g, f(p.A[K0:K1]), f(p.B[K0:K1]), f(p.T_AA[:, :, a0:a1]),
                              f(p.T_AB[:, :, a0:a1]), f(p.T_BB[:, :, a0:a1]), f(p.U[:, a0:a1]))


def _packed_cover(ranges_per_engine, n):
    """The owned ranges of the engines of one window tile its packed range exactly once."""
    allr = sorted(r for rs in ranges_per_engine for r in rs)
    for (a0, a1), (b0, b1) in zip(allr, allr[1:]):
        assert a1 == b0, (a0, a1, b0, b1)
    return allr[0][0], allr[-1][1]


@pytest.mark.parametrize("algo", ["merged", "fused", "refined", "original"])
def test_column_windows_assemble_to_the_full_result(restatement, algo):
    """2-D owner-computes tiling: three engines each hold every atom and one column window
    [c0, c1) of H, S (operand columns [c0, N_G)); their downloads fill disjoint columns of H, S
    and together equal the full build."""
    p = hb.generate_problem(6, 25, 333, 9, 2)
    if algo == "original":
        H0, S0, _, _ = restatement.build_hs_original(p)
    else:
        H0, S0, _ = restatement.build_hs_refined(p)
    H = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
    S = np.zeros_like(H)
    iu = np.triu_indices(p.n_g, 1)
    H[iu] = np.nan  # the upper triangle is never written
    S[iu] = np.nan
    n = p.n_g
    for c0, c1 in ((0, 128), (128, 192), (192, 0)):
        e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g, col_begin=c0, col_end=c1)
        e.upload(p)
        e.build(algo)
        e.sync()
        own = e.owned()
        end = c1 or n
        assert own == [(c0 * (2 * n - c0 + 1) // 2, end * (2 * n - end + 1) // 2)]
        e.download(H, S)
        e.close()
    assert np.all(np.isnan(H[iu])) and np.all(np.isnan(S[iu]))
    assert rel(H, H0) <= TOL and rel(S, S0) <= TOL


def test_column_window_errors():
    with pytest.raises(hb.ConfigError):
        hb.Engine(0, 2, 5, 300, col_begin=10, col_end=128)  # not a multiple of 64
    with pytest.raises(hb.ConfigError):
        hb.Engine(0, 2, 5, 300, col_begin=128, col_end=128)
    e = hb.Engine(0, 2, 5, 300, col_begin=64, col_end=256)
    with pytest.raises(hb.ConfigError):
        e.reshape(200)  # only whole-window engines are re-targeted
    e.close()


@pytest.mark.parametrize("mode", ["scatter", "root"])
@pytest.mark.parametrize("dims", [(7, 25, 333, 4, 1), (8, 49, 4000, 9, 3)], ids=["small", "banded"])
def test_emulated_grid_group_reduce(restatement, mode, dims):
    """A 2 x 3 grid (two column windows x three atom shards) on one device: each window's three
    engines are summed by group_reduce (the same-device sum kernel); in SCATTER mode every
    engine owns one slice of every reduce segment (8 bands for the banded final H at N_G 2200),
    in ROOT mode rank 0 owns the window.  The downloads assemble the full result."""
    p = hb.generate_problem(*dims)
    Hs, Ss, _ = restatement.build_hs_refined(p) if p.n_g < 1000 else (None, None, None)
    n = p.n_g
    bounds = hb.shard_atoms(p.n_atoms, 3)
    # banded: N_G 4000 = 63 tile columns, two windows of 1026 / 990 lower tiles (>= 4 waves of
    # 148 CTAs each, so each window's final H runs in 8 bands = 8 reduce segments)
    windows = ((0, 128), (128, 0)) if n < 1000 else ((0, 1216), (1216, 0))
    H = np.zeros((n, n), np.complex128, order="F")
    S = np.zeros_like(H)
    engines = []
    for c0, c1 in windows:
        grp = []
        for r in range(3):
            e = hb.Engine(0, bounds[r + 1] - bounds[r], p.n_l, n, col_begin=c0, col_end=c1)
            e.set_download_overlap(True)  # banded final H -> 8 reduce segments when large enough
            e.upload(p, bounds[r])
            e.build()
            grp.append(e)
        hb.group_reduce(grp, mode, 0)
        owned = [e.owned() for e in grp]
        if mode == "root":
            assert all(o == [] for o in owned[1:])
        else:
            assert all(len(o) == len(owned[0]) for o in owned)
        lo, hi = _packed_cover(owned, n)
        end = c1 or n
        assert (lo, hi) == (c0 * (2 * n - c0 + 1) // 2, end * (2 * n - end + 1) // 2)
        engines += grp
    for e in engines:
        e.download(H, S)
    st = engines[0].sync()
    for e in engines:
        e.close()
    if Hs is None:  # large case: against a whole single-engine build (itself oracle-pinned elsewhere)
        f = hb.Engine(0, p.n_atoms, p.n_l, n)
        f.upload(p)
        f.build()
        Hs, Ss = f.download()
        f.close()
        assert st["kernel_launches"] > 8  # banded
    assert rel(H, Hs) <= TOL and rel(S, Ss) <= TOL


@pytest.mark.parametrize("algo", ["merged", "fused", "refined", "original"])
def test_row_balanced_shards_sum_to_the_full_result(restatement, algo):
    """Row-balanced shards (shard_rows: K = 7 x 25 rows over 3 engines on one device, boundary
    atoms held by two engines, each engine contracting only its row range): the summed partials
    equal the full result, and the original algorithm's potrf outcomes (an HPD-failing atom
    among them) are counted once per atom."""
    p = hb.generate_problem(7, 25, 333, 4, 3)
    if algo == "original":
        Hs, Ss, _, want_hpd = restatement.build_hs_original(p)
    else:
        (Hs, Ss, _), want_hpd = restatement.build_hs_refined(p), p.n_atoms
    n = p.n_g
    H = np.zeros((n, n), np.complex128, order="F")
    S = np.zeros_like(H)
    shards = hb.shard_rows(p.n_atoms, p.n_l, 3)
    assert any(r0 > 0 for _, _, r0, _ in shards)  # genuinely mid-atom boundaries
    n_hpd = 0
    for a0, na, r0, r1 in shards:
        e = hb.Engine(0, na, p.n_l, n, row_begin=r0, row_end=r1)
        e.upload(p, a0)
        e.build(algo)
        Hp, Sp = e.download()
        H += Hp
        S += Sp
        n_hpd += e.sync()["n_hpd"]
        e.close()
    assert rel(H, Hs) <= TOL and rel(S, Ss) <= TOL
    assert n_hpd == want_hpd and (algo != "original" or want_hpd < p.n_atoms)


def test_row_range_errors():
    with pytest.raises(hb.ConfigError):
        hb.Engine(0, 3, 10, 100, row_begin=10, row_end=25)  # starts past the first atom
    with pytest.raises(hb.ConfigError):
        hb.Engine(0, 3, 10, 100, row_begin=0, row_end=20)  # ends before the last atom


@pytest.mark.parametrize("reduce", ["scatter", "root"])
@pytest.mark.parametrize("grid", [(3, 1), (4, 2), (2, 2)], ids=["3x1", "2x2", "1x2"])
def test_dropin_emulated_grid(restatement, grid, reduce):
    """build_hs_refined / build_hs_original / build_hs_file with n_gpus engines on device 0
    (device_ids repeated): atom shards x column windows, reduce, per-engine downloads."""
    P, pc = grid
    p = hb.generate_problem(9, 25, 400, 5, 2)
    H0, S0, _ = restatement.build_hs_refined(p)
    cfg = hb.PipelineConfig(n_gpus=P, device_ids=[0] * P, col_groups=pc, reduce=reduce)
    r = hb.build_hs_refined(p, cfg)
    assert r.stats["col_groups"] == pc and r.stats["n_gpus"] == P
    assert rel(r.H, H0) <= TOL and rel(r.S, S0) <= TOL
    iu = np.triu_indices(p.n_g, 1)
    assert np.all(r.H[iu] == 0) and np.all(r.S[iu] == 0)
    assert r.ledger == hb.flop_model(p)
    Ho, So, _, n_hpd = restatement.build_hs_original(p)
    ro = hb.build_hs_original(p, hb.PipelineConfig(variant="original", n_gpus=P, device_ids=[0] * P, col_groups=pc,
                                                   reduce=reduce))
    assert rel(ro.H, Ho) <= TOL and rel(ro.S, So) <= TOL
    assert ro.ledger == hb.flop_model(p, "original")
    hb.release_cache()


def test_dropin_emulated_grid_from_file(restatement, tmp_path):
    p = hb.generate_problem(8, 49, 300, 3, 1)
    path = str(tmp_path / "p.hsdl")
    hb.save_problem(p, path)
    H0, S0, _ = restatement.build_hs_refined(p)
    r = hb.build_hs_file(path, hb.PipelineConfig(n_gpus=4, device_ids=[0] * 4, col_groups=2))
    assert rel(r.H, H0) <= TOL and rel(r.S, S0) <= TOL
    hb.release_cache()


def test_auto_col_groups_follow_the_memory_budget(restatement):
    """col_groups = 0: 1 (replicated H, S) when the per-GPU estimate fits the budget; a budget
    below the replicated footprint selects 2-D tiling (the smallest divisor of n_gpus that fits)."""
    p = hb.generate_problem(4, 9, 1200, 2, 0)
    H0, S0, _ = restatement.build_hs_refined(p)
    big = hb.build_hs_refined(p, hb.PipelineConfig(n_gpus=4, device_ids=[0] * 4, mem_budget_gb=10.0))
    assert big.stats["col_groups"] == 1
    # replicated: 2 x 1200^2/2 x 16 B x 1.1 ~ 25 MB of H, S per GPU; 2 windows halve it
    small = hb.build_hs_refined(p, hb.PipelineConfig(n_gpus=4, device_ids=[0] * 4, mem_budget_gb=0.020))
    assert small.stats["col_groups"] > 1
    for r in (big, small):
        assert rel(r.H, H0) <= TOL and rel(r.S, S0) <= TOL
    with pytest.raises(hb.ConfigError):
        hb.build_hs_refined(p, hb.PipelineConfig(n_gpus=4, device_ids=[0] * 4, col_groups=3))
    if hb.device_count() > 1:  # a window's GPUs must be all distinct (NCCL) or all one device
        with pytest.raises(hb.ConfigError):
            hb.build_hs_refined(p, hb.PipelineConfig(n_gpus=3, device_ids=[0, 0, 1], col_groups=1))
    hb.release_cache()


def test_engine_cache_reshapes_within_capacity():
    """The drop-in keeps its engines across calls whose N_G varies by a few per cent (5 %
    headroom): same device allocation, results still exact."""
    hb.release_cache()
    sizes = [1000, 1030, 980, 1045, 1000]
    peaks = []
    for i, ng in enumerate(sizes):
        p = hb.generate_problem(6, 25, ng, 10 + i, 0)
        r = hb.build_hs_refined(p)
        peaks.append(r.stats["peak_device_bytes"])
        e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g)
        e.upload(p)
        e.build()
        H, S = e.download()
        e.close()
        assert rel(r.H, H) <= 1e-14 and rel(r.S, S) <= 1e-14, ng
    assert len(set(peaks)) == 1, peaks
    hb.release_cache()


def test_engine_reshape_api():
    p = hb.generate_problem(5, 9, 700, 3, 1)
    q = hb.generate_problem(5, 9, 640, 4, 1)
    e = hb.Engine(0, 5, 9, 700, n_g_capacity=720)
    for prob in (p, q, p):
        e.reshape(prob.n_g)
        e.upload(prob)
        e.build()
        H, S = e.download()
        w = hb.build_hs_refined(prob)
        assert rel(H, w.H) <= 1e-14 and rel(S, w.S) <= 1e-14
    with pytest.raises(hb.SizingError):
        e.reshape(721)
    e.close()
    hb.release_cache()


@pytest.mark.parametrize("algo", ["merged", "original"])
def test_kpoints_with_varying_basis_size(algo):
    """N_G(k) differs per k-point (a real k-point set): one engine sized for the largest,
    re-targeted per k-point; N_G >= 2200 runs the banded final H, whose download of k-1 overlaps
    build k (the H / S storage-reuse ordering).  Every k-point equals its own per-call build."""
    base = hb.generate_problem(12, 49, 2300, 3, 2)
    ngk = [2300, 2240, 2288, 2200, 2300]
    kps = [hb.generate_problem(12, 49, n, 20 + k, 2) for k, n in enumerate(ngk)]
    cfg = hb.PipelineConfig(variant="original") if algo == "original" else hb.PipelineConfig()
    got, st = hb.build_hs_kpoints(base, [q.A for q in kps], [q.B for q in kps], cfg)
    for k, (H, S) in enumerate(got):
        # the cell's operators and U with k-point k's coefficients
        pk = hb.ProblemInstance(12, 49, ngk[k], kps[k].A, kps[k].B, base.T_AA, base.T_AB, base.T_BB, base.U,
                                base.hpd_flags)
        want = hb.build_hs(pk, cfg)
        assert H.shape == (ngk[k], ngk[k])
        assert rel(H, want.H) <= 1e-13 and rel(S, want.S) <= 1e-13, k
    hb.release_cache()


# ---------------------------------------------------------------------------------------
# >= 2 GPUs: the real NCCL grid (skipped on a one-GPU box)
# ---------------------------------------------------------------------------------------
def _need_gpus(n):
    if hb.device_count() < n:
        pytest.skip(f"needs {n} GPUs (this box has {hb.device_count()})")


@pytest.mark.parametrize("reduce", ["scatter", "root"])
def test_multigpu_dropin_config1_full_vs_reference(reduce):
    """Single-process n_gpus = 2 (ncclCommInitAll, grouped NCCL calls, one host thread per GPU)
    on config 1 in full against the unmodified reference."""
    _need_gpus(2)
    from oracle.oracle import Reference, Restatement
    p = hb.generate_problem(16, 49, 1000, 1, 0)
    if Reference.available():
        ref = Reference().build_hs(p, "refined", threads=os.cpu_count() or 1, blocked=True)
        H0, S0 = ref["H"], ref["S"]
    else:
        H0, S0, _ = Restatement().build_hs_refined(p)
    for P, pc in ((2, 1), (min(4, hb.device_count()), 2)):
        if P % pc:
            continue
        r = hb.build_hs_refined(p, hb.PipelineConfig(n_gpus=P, col_groups=pc, reduce=reduce))
        assert r.stats["n_gpus"] == P
        assert rel(r.H, H0) <= TOL and rel(r.S, S0) <= TOL, (P, pc)
    hb.release_cache()


def test_multigpu_dropin_config3_sampled(restatement):
    """Config 3 (108 atoms, N_L 121, N_G 6000) K-row-sharded over every GPU: principal-submatrix
    sampling against the oracle on the J-sliced problem."""
    _need_gpus(2)
    P = hb.device_count()
    p = hb.generate_problem(108, 121, 6000, 1, 0)
    r = hb.build_hs_refined(p, hb.PipelineConfig(n_gpus=P))
    J = np.sort(np.random.default_rng(7).choice(p.n_g, size=96, replace=False))
    Hs, Ss = restatement.build_hs_sampled(p, J.astype(np.uint64))
    assert rel(np.asfortranarray(r.H[np.ix_(J, J)]), Hs) <= TOL
    assert rel(np.asfortranarray(r.S[np.ix_(J, J)]), Ss) <= TOL
    hb.release_cache()


@pytest.mark.parametrize("reduce", ["scatter", "root"])
def test_multigpu_torchrun_engine_path(tmp_path, reduce):
    """One process per GPU (torchrun, NCCL communicator per engine via hsdla_b200_engine_set_comm):
    each rank generates only its atom shard, builds, reduces and downloads what it owns; rank 0
    assembles (gloo) and compares with the reference run of the same problem."""
    _need_gpus(2)
    out = tmp_path / "result.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "tests", "dist_engine_worker.py"),
           "--reduce", reduce, "--out", str(out)]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    z = np.load(out)
    assert z["err_h"] <= TOL and z["err_s"] <= TOL


@pytest.mark.parametrize("split", ["always", "never"])
def test_split_triangle_launches_in_windows_bands_and_kpoints(restatement, monkeypatch, split):
    """The triangle as separate strictly-lower / diagonal / ragged-last-row launches (thresholds
    forced to 0) or as one launch (thresholds huge), in every place a triangle is enumerated: whole
    builds, column windows of an emulated 2 x 2 grid, the banded final H and k-point batches.
    N_G = 2200 (35 tile columns: 630 lower tiles, enough for the banded final H) leaves the last
    tile row with 24 of 64 rows (v = 3)."""
    big = "1e18" if split == "never" else "0"
    monkeypatch.setenv("HSDLA_B200_DIAG_SPLIT_MIN", big)
    monkeypatch.setenv("HSDLA_B200_ROW_SPLIT_MIN", big)
    p = hb.generate_problem(4, 16, 2200, 7, 1)
    Hs, Ss, _ = restatement.build_hs_refined(p)
    for algo in ("merged", "refined"):
        r = hb.build_hs_refined(p, hb.PipelineConfig(algo=algo))
        assert rel(r.H, Hs) <= TOL and rel(r.S, Ss) <= TOL, algo
    r = hb.build_hs_refined(p, hb.PipelineConfig(n_gpus=4, device_ids=[0, 0, 0, 0], col_groups=2))
    assert rel(r.H, Hs) <= TOL and rel(r.S, Ss) <= TOL
    e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g)
    e.set_download_overlap(True)  # banded final H: 8 tile-column bands, each split or not
    e.upload(p)
    e.build()
    H, S = e.download()
    st = e.sync()
    e.close()
    assert rel(H, Hs) <= TOL and rel(S, Ss) <= TOL
    assert st["kernel_launches"] == 12 if split == "never" else st["kernel_launches"] > 12  # 8 bands
    kps = [hb.generate_problem(4, 16, 2200, 20 + k, 1) for k in range(2)]
    got, _ = hb.build_hs_kpoints(p, [q.A for q in kps], [q.B for q in kps])
    for (Hk, Sk), q in zip(got, kps):
        pk = hb.generate_problem(4, 16, 2200, 7, 1)
        pk.A, pk.B = q.A, q.B
        Hq, Sq, _ = restatement.build_hs_refined(pk)
        assert rel(Hk, Hq) <= TOL and rel(Sk, Sq) <= TOL
    hb.release_cache()


@pytest.mark.parametrize("ng", [1, 63, 64, 65, 127, 130, 200, 257, 450])
def test_split_triangle_launches_edge_sizes(restatement, monkeypatch, ng):
    """Forced split launches at edge tile counts: one tile (no strictly-lower tiles), a last tile row
    with 1..8 valid fragment rows, and the kernel layer's herk on the same sizes."""
    from paper_1712_07206_b200 import kernels as K
    monkeypatch.setenv("HSDLA_B200_DIAG_SPLIT_MIN", "0")
    monkeypatch.setenv("HSDLA_B200_ROW_SPLIT_MIN", "0")
    p = hb.generate_problem(3, 9, ng, 11, 1)
    Hs, Ss, _ = restatement.build_hs_refined(p)
    r = hb.build_hs_refined(p)
    assert rel(r.H, Hs) <= TOL and rel(r.S, Ss) <= TOL
    C = np.zeros((ng, ng), np.complex128, order="F")
    K.herk(1.0, p.A, 0.0, C)
    il = np.tril_indices(ng)
    want = (p.A.conj().T @ p.A)[il]
    assert np.linalg.norm(C[il] - want) <= 1e-12 * max(np.linalg.norm(want), 1e-300)
    hb.release_cache()
