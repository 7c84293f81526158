"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Bar (north_star): relative Frobenius error of the lower triangle <= 1e-11 on H and S
(rel_frobenius_error_lower, complex_matrix.cpp:106-118).  Plus the reference's
behavioural contract: upper triangle never written, diagonal imag 0,
T_AA/T_BB read from the lower triangle only, ledger == flop_model, five phases.
"""
import os

import numpy as np
import pytest

import paper_1712_07206_b200 as hb
from conftest import as_problem, golden_cases, load_case

pytestmark = pytest.mark.gpu
TOL = 1e-11  # north_star FP64 tolerance, relative Frobenius, lower triangle


def rel(x, y):
    return hb.rel_frobenius_error_lower(x, y)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    assert hb.device_count() > 0, "GPU tests need a CUDA device"
    yield
    hb.release_cache()


@pytest.mark.parametrize("algo,arith", [("merged", "3m"), ("fused", "3m"), ("refined", "3m"), ("merged", "4m"),
                                       ("fused", "4m"), ("refined", "4m")])
@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1][:-4])
def test_golden_parity(path, algo, arith):
    dims, d = load_case(path)
    p = as_problem(d, dims)
    r = hb.build_hs_refined(p, hb.PipelineConfig(algo=algo, arith=arith))
    assert rel(r.H, d["H"]) <= TOL, rel(r.H, d["H"])
    assert rel(r.S, d["S"]) <= TOL, rel(r.S, d["S"])
    ng = dims[2]
    iu = np.triu_indices(ng, 1)
    assert np.all(r.H[iu] == 0) and np.all(r.S[iu] == 0)
    assert np.all(np.diag(r.H).imag == 0) and np.all(np.diag(r.S).imag == 0)
    assert [ph.name for ph in r.phases] == ["s", "z_loop", "her2k", "hemm_loop", "herkx"]
    assert r.ledger.total() == int(d["ledger"][8])


def test_unit_problem_hand_values():
    p = hb.empty_problem(1, 1, 1)
    p.A[0, 0] = 1.0
    p.B[0, 0] = 1j
    p.T_AA[0, 0, 0] = 2.0
    p.T_AB[0, 0, 0] = 1.0
    p.T_BB[0, 0, 0] = 4.0
    p.U[0, 0] = 1.0
    r = hb.build_hs_refined(p)
    assert r.H[0, 0] == 6.0 and r.S[0, 0] == 2.0


def test_upper_triangle_never_written():
    """NaN-poisoned caller buffers: the upper triangle survives untouched
    (test_kernels.cpp:76-109, complex_matrix.cpp:47-52)."""
    p = hb.generate_problem(3, 9, 70, 51, 1)
    n = p.n_g
    H = np.full((n, n), np.nan + 1j * np.nan, order="F")
    S = np.full((n, n), np.nan + 1j * np.nan, order="F")
    r = hb.build_hs_refined(p, H=H, S=S)
    iu = np.triu_indices(n, 1)
    assert np.all(np.isnan(r.H[iu])) and np.all(np.isnan(r.S[iu]))
    il = np.tril_indices(n)
    assert np.all(np.isfinite(r.H[il])) and np.all(np.isfinite(r.S[il]))


def test_hermitian_operators_read_lower_only(restatement):
    """T_AA and T_BB are read from their lower triangles only (test_kernels.cpp:173-187)."""
    p = hb.generate_problem(4, 11, 90, 3, 0)
    want = hb.build_hs_refined(p)
    iu = np.triu_indices(p.n_l, 1)
    for a in range(p.n_atoms):
        for T in (p.T_AA, p.T_BB):
            blk = T[:, :, a]
            blk[iu] = np.nan
    got = hb.build_hs_refined(p)
    assert np.array_equal(got.H, want.H) and np.array_equal(got.S, want.S)


def test_config1_full_vs_oracle():
    """Config 1 (16 atoms, lmax 6, N_G 1000), the reference's CPU-runnable case, in full."""
    from oracle.oracle import Reference, Restatement
    p = hb.generate_problem(16, 49, 1000, 1, 0)
    r = hb.build_hs_refined(p)
    if Reference.available():
        ref = Reference().build_hs(p, "refined", threads=16, blocked=True)
        Hr, Sr = ref["H"], ref["S"]
    else:
        Hr, Sr, _ = Restatement().build_hs_refined(p)
    assert rel(r.H, Hr) <= TOL and rel(r.S, Sr) <= TOL
    assert r.ledger == hb.flop_model(p)


def test_config2_full_vs_unmodified_reference():
    """Config 2 (64 atoms, lmax 8, N_G 3000), the bench workload, in full against the
    unmodified reference's own CPU run (oracle/_ref, BlockedParallel on every host core,
    ~20 s on the GPU box), for the default (merged) and the reference-order algorithms."""
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    p = hb.generate_problem(64, 81, 3000, 1, 0)
    ref = Reference().build_hs(p, "refined", threads=os.cpu_count() or 1, blocked=True)
    for algo in ("merged", "refined"):
        r = hb.build_hs_refined(p, hb.PipelineConfig(algo=algo))
        assert rel(r.H, ref["H"]) <= TOL and rel(r.S, ref["S"]) <= TOL, algo
        assert r.ledger == hb.flop_model(p)


@pytest.mark.parametrize("dims", [(64, 81, 3000)], ids=["config2"])
def test_sampled_parity_at_config_sizes(dims, restatement):
    """Config 2 (configs 3-5: tests/test_gpu_large.py against the unmodified reference):
    principal-submatrix sampling (SURVEY §7 hard part 3):
    H[J,J], S[J,J] depend only on columns J of A, B; the oracle runs the J-sliced problem."""
    na, nl, ng = dims
    p = hb.generate_problem(na, nl, ng, 1, 0)
    r = hb.build_hs_refined(p)
    rng = np.random.default_rng(7)
    J = np.sort(rng.choice(ng, size=96, replace=False))
    Hs, Ss = restatement.build_hs_sampled(p, J.astype(np.uint64))
    sub = np.ix_(J, J)
    assert rel(np.asfortranarray(r.H[sub]), Hs) <= TOL
    assert rel(np.asfortranarray(r.S[sub]), Ss) <= TOL


def test_properties_at_config2():
    """Size-independent properties: S Hermitian positive definite (test_pipeline.cpp:149-165);
    linearity in T (doubling every T doubles H, leaves S); atom additivity (the sum over
    atom shards that the multi-GPU NCCL reduce relies on); determinism run to run."""
    p = hb.generate_problem(64, 81, 3000, 1, 0)
    r1 = hb.build_hs_refined(p)  # streamed: 8 atom chunks, H2D overlapped, beta=1 accumulation
    r2 = hb.build_hs_refined(p)
    assert np.array_equal(r1.H, r2.H) and np.array_equal(r1.S, r2.S)
    e = hb.Engine(0, 64, 81, 3000)  # device-resident single-chunk build
    e.upload(p)
    e.build()
    e.sync()
    He, Se = e.download()
    e.close()
    assert rel(He, r1.H) <= 1e-13 and rel(Se, r1.S) <= 1e-13
    S = hb.mirror(r1.S.copy())
    S[np.diag_indices_from(S)] += 1e-8 * np.linalg.norm(S)
    np.linalg.cholesky(S)
    # linearity
    q = hb.generate_problem(64, 81, 3000, 1, 0)
    for T in (q.T_AA, q.T_AB, q.T_BB):
        T *= 2.0
    r3 = hb.build_hs_refined(q)
    assert rel(r3.H, 2.0 * r1.H) <= TOL and np.array_equal(r3.S, r1.S)
    # atom additivity: H(all atoms) = H(atoms 0..31) + H(atoms 32..63)
    parts = []
    for a0, a1 in ((0, 32), (32, 64)):
        K0, K1 = a0 * p.n_l, a1 * p.n_l
        s = hb.ProblemInstance(a1 - a0, p.n_l, p.n_g, np.asfortranarray(p.A[K0:K1]), np.asfortranarray(p.B[K0:K1]),
                               np.asfortranarray(p.T_AA[:, :, a0:a1]), np.asfortranarray(p.T_AB[:, :, a0:a1]),
                               np.asfortranarray(p.T_BB[:, :, a0:a1]), np.asfortranarray(p.U[:, a0:a1]))
        parts.append(hb.build_hs_refined(s))
    assert rel(parts[0].H + parts[1].H, r1.H) <= TOL
    assert rel(parts[0].S + parts[1].S, r1.S) <= TOL


def test_engine_sharded_reduce_emulation():
    """The per-rank engine API on shards [0,a) and [a,N): partial packed results summed
    on the host equal the single-engine result (what ncclReduce(sum) does on 2 GPUs)."""
    p = hb.generate_problem(6, 25, 333, 9, 0)
    full = hb.Engine(0, 6, 25, 333)
    full.upload(p, 0)
    full.build()
    full.sync()
    Hf, Sf = full.download()
    acc_h = np.zeros_like(Hf)
    acc_s = np.zeros_like(Sf)
    for a0, na in ((0, 4), (4, 2)):
        e = hb.Engine(0, na, 25, 333)
        e.upload(p, a0)
        e.build("refined")
        st = e.sync()
        assert st["kernel_launches"] >= 5
        h, s = e.download()
        acc_h += h
        acc_s += s
        e.close()
    full.close()
    assert rel(acc_h, Hf) <= TOL and rel(acc_s, Sf) <= TOL


def test_algos_agree():
    p = hb.generate_problem(7, 49, 515, 2, 0)
    a = hb.build_hs_refined(p, hb.PipelineConfig(algo="fused"))
    b = hb.build_hs_refined(p, hb.PipelineConfig(algo="refined"))
    m = hb.build_hs_refined(p, hb.PipelineConfig(algo="merged"))
    assert rel(a.H, b.H) <= 1e-13 and rel(a.S, b.S) == 0.0
    assert rel(m.H, b.H) <= 1e-13 and rel(m.S, b.S) == 0.0
    assert a.stats["kernel_launches"] >= 5
    # merged: 16 K N_G^2 + 32 N_A N_L^2 N_G complex-MAC flops (3M: 6 per MAC) + 2 K N_G
    K = p.n_atoms * p.n_l
    assert m.stats["executed_flops"] == (16 * K * p.n_g ** 2 + 32 * p.n_atoms * p.n_l ** 2 * p.n_g) // 8 * 6 + \
        2 * K * p.n_g
    assert m.ledger.total() == a.ledger.total()


@pytest.mark.parametrize("algo", ["merged", "fused", "refined", "original"])
def test_banded_final_h_matches_device_resident(algo):
    """The one-shot drop-in runs its final H contraction in tile-column bands (each band's
    download overlapping the next band); the device-resident engine runs it whole.
    Both agree to rounding, and the bands cover every lower tile exactly once."""
    for dims in ((24, 81, 2200, 9, 3), (3, 7, 70, 2, 1), (2, 5, 130, 4, 0)):
        p = hb.generate_problem(*dims)
        cfg = hb.PipelineConfig(variant="original") if algo == "original" else hb.PipelineConfig(algo=algo)
        r = hb.build_hs(p, cfg)
        e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g)
        e.upload(p)
        e.build(algo)
        e.sync()
        H, S = e.download()
        e.close()
        assert rel(r.H, H) <= 1e-14 and rel(r.S, S) <= 1e-14, dims


@pytest.mark.parametrize("algo", ["merged", "fused", "refined", "original"])
def test_operators_with_complex_diagonals_follow_reference_hemm(restatement, algo):
    """The reference's hemm uses T's diagonal as stored (kernels.cpp:152-167), also a
    non-real one; the device operand expansion reproduces that exactly."""
    p = hb.generate_problem(5, 9, 60, 8, 2)
    g = np.random.default_rng(3)
    for T in (p.T_AA, p.T_BB):
        for a in range(p.n_atoms):
            T[np.arange(p.n_l), np.arange(p.n_l), a] += 1j * g.uniform(-0.5, 0.5, p.n_l)
    if algo == "original":
        H, S, _, _ = restatement.build_hs_original(p)
        r = hb.build_hs_original(p)
    else:
        H, S, _ = restatement.build_hs_refined(p)
        r = hb.build_hs_refined(p, hb.PipelineConfig(algo=algo))
    assert rel(r.H, H) <= TOL and rel(r.S, S) <= TOL


@pytest.mark.parametrize("algo", ["merged", "fused", "original"])
def test_nccl_reduce_path_single_rank(restatement, algo):
    """The multi-GPU reduce path (comm stream, S reduce overlapping H, ncclReduce of the
    packed triangles, download ordered after the reduce) through a real 1-rank NCCL
    communicator: same result as the communicator-free build."""
    p = hb.generate_problem(6, 25, 300, 4, 1)
    H0, S0 = (restatement.build_hs_original(p)[:2] if algo == "original" else restatement.build_hs_refined(p)[:2])
    e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g)
    e.set_comm(hb.nccl_unique_id(), 1, 0)
    for streamed in (False, True):
        if streamed:
            e.build_streamed(p, 0, algo)
        else:
            e.upload(p)
            e.build(algo)
        e.reduce(0)
        st = e.sync()
        H, S = e.download()
        assert rel(H, H0) <= TOL and rel(S, S0) <= TOL
        assert st["reduce_seconds"] >= 0.0
    e.set_comm(None, 1, 0)
    e.close()


EDGE_DIMS = [(1, 1, 1, 1, 0), (1, 2, 2, 2, 0), (3, 3, 63, 3, 1), (2, 5, 65, 4, 1), (1, 7, 129, 5, 0),
             (7, 1, 200, 6, 3), (9, 4, 1, 7, 2), (2, 9, 64, 8, 0), (5, 2, 257, 9, 5), (3, 17, 3, 10, 1)]


@pytest.mark.parametrize("dims", EDGE_DIMS, ids=lambda d: "x".join(map(str, d[:3])))
def test_edge_shapes_all_algorithms(restatement, dims):
    """Ragged / degenerate shapes: N_G and K = N_A N_L not multiples of the 8-complex k-slab or
    the 64-wide tiles, N_L = 1, N_G = 1..3, one atom, all-failed potrf mixes."""
    p = hb.generate_problem(*dims)
    H, S, _ = restatement.build_hs_refined(p)
    Ho, So, _, n_hpd = restatement.build_hs_original(p)
    n = p.n_g
    iu = np.triu_indices(n, 1)
    for cfg in (hb.PipelineConfig(), hb.PipelineConfig(algo="refined"), hb.PipelineConfig(variant="original")):
        r = hb.build_hs(p, cfg)
        Hw, Sw = (Ho, So) if cfg.variant == "original" else (H, S)
        assert rel(r.H, Hw) <= TOL and rel(r.S, Sw) <= TOL, (dims, cfg)
        assert np.all(r.H[iu] == 0) and np.all(r.S[iu] == 0)
        assert r.ledger == hb.flop_model(p, cfg.variant)


def test_bitwise_determinism_stress():
    """Stream-K partial-tile fixups are ordered, so repeated device-resident builds are
    bitwise identical: 40 builds per algorithm, compared on the device (torch views of the
    engine's packed H, S)."""
    import torch
    p = hb.generate_problem(24, 81, 1500, 5, 3)
    e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g)
    e.upload(p)
    npk = p.n_g * (p.n_g + 1) // 2
    Hp, Sp = e.device_results()

    def as_tensor(ptr):
        # wrap the engine's device buffer without copying
        class _A:
            __cuda_array_interface__ = {"shape": (2 * npk,), "typestr": "<f8", "data": (ptr, False), "version": 3}
        return torch.as_tensor(_A(), device="cuda")

    th, ts = as_tensor(Hp), as_tensor(Sp)
    for algo in ("merged", "fused", "refined", "original"):
        e.build(algo)
        e.sync()
        h0, s0 = th.clone(), ts.clone()
        for _ in range(40):
            e.build(algo)
            e.sync()
            assert torch.equal(th, h0) and torch.equal(ts, s0), algo
    e.close()


def test_concurrent_host_threads(restatement):
    """The drop-in and the kernel layer called from several host threads at once (ctypes
    releases the GIL): engine-cache, staging-ring and host-pool locking keep every result
    exact."""
    import threading
    from paper_1712_07206_b200 import kernels as K
    p = hb.generate_problem(6, 25, 400, 3, 1)
    H0, S0, _ = restatement.build_hs_refined(p)
    A = p.A
    C0 = np.zeros((p.n_g, p.n_g), np.complex128, order="F")
    K.herk(1.0, A, 0.0, C0)
    errs = []

    def worker(i):
        try:
            for _ in range(3):
                r = hb.build_hs_refined(p)
                assert rel(r.H, H0) <= TOL and rel(r.S, S0) <= TOL
                C = np.zeros_like(C0, order="F")
                K.herk(1.0, A, 0.0, C)
                assert np.array_equal(C, C0)
        except Exception as ex:  # noqa: BLE001 - reported below
            errs.append(f"{i}: {ex!r}")

    th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


def test_arith_modes_agree_and_account(restatement):
    """3M and 4M complex arithmetic: both within the bar of the reference-pinned oracle,
    each bitwise deterministic, 3M executes 3/4 of the contraction flops; the ledger is
    identical (the reference's flop model counts 8 real flops per complex MAC)."""
    p = hb.generate_problem(16, 49, 600, 2, 3)
    H, S, _ = restatement.build_hs_refined(p)
    K, ng = p.n_atoms * p.n_l, p.n_g
    for algo in ("merged", "fused"):
        res = {}
        for arith in ("3m", "4m"):
            a = hb.build_hs_refined(p, hb.PipelineConfig(algo=algo, arith=arith))
            b = hb.build_hs_refined(p, hb.PipelineConfig(algo=algo, arith=arith))
            assert np.array_equal(a.H, b.H) and np.array_equal(a.S, b.S)
            assert rel(a.H, H) <= 1e-13 and rel(a.S, S) <= 1e-13, (algo, arith, rel(a.H, H), rel(a.S, S))
            res[arith] = a
        assert res["3m"].ledger == res["4m"].ledger == hb.flop_model(p)
        if algo == "merged":
            cmac = 16 * K * ng * ng + 32 * p.n_atoms * p.n_l ** 2 * ng
        else:
            cmac = 20 * K * ng * ng + 24 * p.n_atoms * p.n_l ** 2 * ng
        assert res["4m"].stats["executed_flops"] == cmac + 2 * K * ng
        assert res["3m"].stats["executed_flops"] == cmac // 8 * 6 + 2 * K * ng
    with pytest.raises(hb.ConfigError):
        hb.build_hs_refined(p, hb.PipelineConfig(arith="2m"))


def test_pageable_and_pinned_inputs_agree_bitwise_with_multi_slab_operator_chunks(restatement, monkeypatch):
    """The host-buffer drop-in with pageable inputs (rows and operator blocks packed into
    pinned slabs with streaming stores) and with registered inputs runs the same chunk plan,
    so H and S are bitwise identical.  A forced 100-atom chunk at N_L 121 carries
    3 x 100 x 121^2 x 16 B = 70 MB of operator blocks, more than one 64 MB staging slab."""
    monkeypatch.setenv("HSDLA_B200_STREAM_PLAN", "100,20")
    hb.release_cache()
    try:
        p = hb.generate_problem(120, 121, 300, 5, 0)
        a = hb.build_hs_refined(p)
        bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U]
        for b in bufs:
            hb.host_register(b)
        try:
            b_ = hb.build_hs_refined(p)
        finally:
            for b in bufs:
                hb.host_unregister(b)
    finally:
        hb.release_cache()
    assert np.array_equal(a.H, b_.H) and np.array_equal(a.S, b_.S)
    J = np.sort(np.random.default_rng(4).choice(p.n_g, size=32, replace=False))
    Hs, Ss = restatement.build_hs_sampled(p, J)
    assert rel(np.asfortranarray(a.H[np.ix_(J, J)]), Hs) <= TOL
    assert rel(np.asfortranarray(a.S[np.ix_(J, J)]), Ss) <= TOL


@pytest.mark.parametrize("algo", ["merged", "refined", "original"])
def test_registered_rows_with_pageable_operators(algo, monkeypatch):
    """A caller who page-locks A and B but not the operator blocks: the rows are copied straight
    from the caller's buffers in the chunk plan, and every atom's T_AA, T_AB, T_BB and U go up
    once, staged after the first chunk's rows (here 70 MB, two 64 MB slabs), with each
    expansion waiting for them.  Bitwise equal to the build with everything registered."""
    monkeypatch.setenv("HSDLA_B200_STREAM_PLAN", "20,100")
    hb.release_cache()
    p = hb.generate_problem(120, 121, 300, 6, 7)
    run = (lambda: hb.build_hs_original(p)) if algo == "original" else \
        (lambda: hb.build_hs_refined(p, hb.PipelineConfig(algo=algo)))
    out = []
    try:
        for bufs in ([p.A, p.B], [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U]):
            for b in bufs:
                hb.host_register(b)
            try:
                out.append(run())
            finally:
                for b in bufs:
                    hb.host_unregister(b)
    finally:
        hb.release_cache()
    assert np.array_equal(out[0].H, out[1].H) and np.array_equal(out[0].S, out[1].S)
    assert out[0].ledger.total() == out[1].ledger.total()


def test_engine_download_overlap_matches_whole_build():
    """hsdla_b200_engine_set_download_overlap: the device-resident build bands its final H
    contraction (band downloads overlap the remaining bands); same H, S to rounding."""
    p = hb.generate_problem(24, 81, 2200, 9, 3)
    out = []
    for on in (False, True):
        e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g)
        e.set_download_overlap(on)
        e.upload(p)
        e.build()
        out.append(e.download())
        e.sync()
        e.close()
    assert rel(out[1][0], out[0][0]) <= 1e-14 and rel(out[1][1], out[0][1]) <= 1e-14


def test_no_device_or_host_leaks_across_many_calls(tmp_path):
    """Many drop-in calls over varying shapes, algorithms, pinned / pageable inputs and a file,
    then release_cache(): device memory returns to its starting level (engines, staging slabs,
    the kernel layer's pooled temporaries and the file view are all released)."""
    import torch
    from paper_1712_07206_b200 import kernels as K
    hb.release_cache()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    rng = np.random.default_rng(5)
    path = str(tmp_path / "p.hsdl")
    for it in range(12):
        na, nl, ng = int(rng.integers(1, 9)), int(rng.choice([5, 9, 25, 49])), int(rng.integers(40, 400))
        p = hb.generate_problem(na, nl, ng, it + 1, int(rng.integers(0, na + 1)))
        algo = ("merged", "fused", "refined")[it % 3]
        if it % 4 == 3:
            bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U]
            for b in bufs:
                hb.host_register(b)
            try:
                hb.build_hs_refined(p, hb.PipelineConfig(algo=algo))
            finally:
                for b in bufs:
                    hb.host_unregister(b)
        else:
            hb.build_hs_refined(p, hb.PipelineConfig(algo=algo))
        if it % 5 == 0:
            hb.build_hs_original(p)
            hb.save_problem(p, path)
            hb.build_hs_file(path)
            C = np.zeros((ng, ng), np.complex128, order="F")
            K.herk(1.0, p.A, 0.0, C)
    hb.release_cache()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free1 >= free0 - (64 << 20), (free0, free1)


def test_first_chunk_split_s_matches_unsplit(monkeypatch):
    """The streamed drop-in starts the first chunk's S with its A^H A half on A's rows alone
    (HSDLA_B200_SPLIT_S=0 turns it off): both orders agree to FP64 rounding."""
    p = hb.generate_problem(24, 81, 1200, 6, 0)
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("HSDLA_B200_SPLIT_S", flag)
        monkeypatch.setenv("HSDLA_B200_STREAM_PLAN", "3,7,14")
        hb.release_cache()
        out.append(hb.build_hs_refined(p))
    hb.release_cache()
    assert rel(out[0].S, out[1].S) <= 1e-14 and rel(out[0].H, out[1].H) <= 1e-14
    assert out[0].stats["kernel_launches"] == out[1].stats["kernel_launches"] + 1


@pytest.mark.parametrize("algo", ["merged", "fused", "refined", "original"])
def test_operators_uploaded_on_the_copy_stream(algo):
    """engine_upload_operators copies T on the copy stream (the build's S runs meanwhile and
    waits for them only before the operator expansion): re-uploading new operators between
    two builds of one engine gives each build its own operators' result."""
    p = hb.generate_problem(6, 25, 300, 4, 2)
    q = hb.generate_problem(6, 25, 300, 5, 2)  # other operators, same shape
    want_p = hb.build_hs(p, hb.PipelineConfig(variant="original") if algo == "original" else
                         hb.PipelineConfig(algo=algo))
    q.A, q.B, q.U = p.A, p.B, p.U              # same coefficients, q's operators
    want_q = hb.build_hs(q, hb.PipelineConfig(variant="original") if algo == "original" else
                         hb.PipelineConfig(algo=algo))
    e = hb.Engine(0, p.n_atoms, p.n_l, p.n_g)
    e.upload(p)
    got = []
    for prob in (q, p, q):
        e.upload_operators(prob.T_AA, prob.T_AB, prob.T_BB)
        e.build(algo)
        got.append(e.download())
    e.sync()
    e.close()
    for (H, S), want in zip(got, (want_q, want_p, want_q)):
        assert rel(H, want.H) <= 1e-13 and rel(S, want.S) <= 1e-13


@pytest.mark.parametrize("pinned", [False, True])
def test_kpoint_batch_matches_per_call_builds(pinned):
    """hsdla_b200_build_hs_kpoints: n k-points sharing the operators and U, their A, B
    alternating between two device sets with uploads / downloads overlapping the builds:
    every k-point equals its own per-call build (to FP64 rounding), for pinned and pageable
    coefficients, in the default and the original algorithm."""
    base = hb.generate_problem(12, 49, 700, 3, 2)
    kps = [hb.generate_problem(12, 49, 700, 10 + k, 2) for k in range(5)]
    As = [q.A for q in kps]
    Bs = [q.B for q in kps]
    if pinned:
        for M in As + Bs:
            hb.host_register(M)
    try:
        for cfg in (hb.PipelineConfig(), hb.PipelineConfig(variant="original")):
            got, st = hb.build_hs_kpoints(base, As, Bs, cfg)
            assert len(got) == 5 and st["total_seconds"] > 0
            for k, (H, S) in enumerate(got):
                pk = hb.generate_problem(12, 49, 700, 3, 2)
                pk.A, pk.B = As[k], Bs[k]
                want = hb.build_hs(pk, cfg)
                assert rel(H, want.H) <= 1e-13 and rel(S, want.S) <= 1e-13, k
                iu = np.triu_indices(700, 1)
                assert np.all(H[iu] == 0) and np.all(S[iu] == 0)
    finally:
        if pinned:
            for M in As + Bs:
                hb.host_unregister(M)
        hb.release_cache()


@pytest.mark.parametrize("every_k,slots", [(False, 3), (True, 3), (False, 2), (True, 2)])
def test_kpoint_batch_banded_final_h_storage_reuse(every_k, slots, monkeypatch):
    """N_G = 2240 (35 tile columns, 630 lower tiles >= 4 x 148): the last k-point's final H runs
    band by band (HSDLA_B200_KPOINT_BANDS=1: every k-point's), and build k reuses the H, S storage
    while the D2H of k-1 is still in flight (build k waits on k-1's last H piece download and on
    its S download).  The downloads rotate over 3 host slots (the host unpacks k-2 while build k
    runs) or, for stages above HSDLA_B200_KPOINT_SLOT_MB, 2.  Every k-point equals its own
    per-call build."""
    if every_k:
        monkeypatch.setenv("HSDLA_B200_KPOINT_BANDS", "1")
    if slots == 2:
        monkeypatch.setenv("HSDLA_B200_KPOINT_SLOT_MB", "0")
    ng = 2240
    base = hb.generate_problem(6, 16, ng, 3, 1)
    kps = [hb.generate_problem(6, 16, ng, 20 + k, 1) for k in range(5)]
    As = [q.A for q in kps]
    Bs = [q.B for q in kps]
    try:
        got, _ = hb.build_hs_kpoints(base, As, Bs, hb.PipelineConfig())
        for k, (H, S) in enumerate(got):
            pk = hb.generate_problem(6, 16, ng, 3, 1)
            pk.A, pk.B = As[k], Bs[k]
            want = hb.build_hs_refined(pk)
            assert rel(H, want.H) <= 1e-13 and rel(S, want.S) <= 1e-13, k
    finally:
        hb.release_cache()


@pytest.mark.parametrize("algo", ["merged", "refined", "original"])
def test_phase_times_from_launch_stamps(algo):
    """Phase and device times come from the kernels' own %globaltimer stamps (stamp.cuh), not
    from CUDA timing events on the compute stream: every phase the algorithm runs is timed,
    phases are disjoint (their sum stays within the device time) and the device time of a
    device-resident build agrees with the host's wall clock around it."""
    import time
    p = hb.generate_problem(16, 49, 1000, 1, 0)
    # streamed drop-in: copies overlap the kernels
    r = hb.build_hs_original(p) if algo == "original" else hb.build_hs_refined(p, hb.PipelineConfig(algo=algo))
    ph = r.stats["phase_seconds"]
    ran = {"merged": ["s", "z_loop", "her2k"], "refined": ["s", "z_loop", "her2k", "hemm_loop", "herkx"],
           "original": ["z_loop", "her2k", "s", "chol_loop", "h_aa_update"]}[algo]
    for k in ran:
        assert ph[k] > 0, (k, ph)
    dev = r.stats["device_seconds"]
    assert 0 < sum(ph.values()) <= dev * 1.001 + 1e-6, (ph, dev)
    e = hb.Engine(0, 16, 49, 1000)
    e.upload(p)
    for _ in range(3):  # warm up
        e.build(algo)
        e.sync()
    t = time.perf_counter()
    e.build(algo)
    st = e.sync()
    wall = time.perf_counter() - t
    e.close()
    assert 0 < st["device_seconds"] <= wall, (st["device_seconds"], wall)
    assert sum(st["phase_seconds"].values()) <= st["device_seconds"] * 1.001 + 1e-6
