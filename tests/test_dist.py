"""Multi-rank host logic on CPU (gloo, world_size 2): the atom partition the engine
uses, and the sum-reduce of per-shard partial H, S that NCCL performs on GPUs.
Partials are computed by the CPU oracle (test infrastructure) on each rank's shard."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1712_07206_b200 as hb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard(p, a0, a1):
    from oracle.oracle import _Problem
    K0, K1 = a0 * p.n_l, a1 * p.n_l
    f = np.asfortranarray
    return _Problem(a1 - a0, p.n_l, p.n_g, f(p.A[K0:K1]), f(p.B[K0:K1]), f(p.T_AA[:, :, a0:a1]),
                    f(p.T_AB[:, :, a0:a1]), f(p.T_BB[:, :, a0:a1]), f(p.U[:, a0:a1]), None)


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    from oracle.oracle import Restatement
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Restatement()
        p = orc.generate_problem(7, 6, 48, 3, 2)
        b = hb.shard_atoms(p.n_atoms, world)
        H, S, _ = orc.build_hs_refined(_shard(p, b[rank], b[rank + 1]))
        # packed-lower partials, summed like ncclReduce(sum, root 0)
        il = np.tril_indices(p.n_g)
        hp = torch.from_numpy(np.ascontiguousarray(H.T[il[1], il[0]]).view(np.float64).copy())
        sp = torch.from_numpy(np.ascontiguousarray(S.T[il[1], il[0]]).view(np.float64).copy())
        dist.reduce(hp, dst=0, op=dist.ReduceOp.SUM)
        dist.reduce(sp, dst=0, op=dist.ReduceOp.SUM)
        # bench.py's Dist helpers: max over ranks, byte broadcast of the NCCL id
        sys.argv = ["bench.py"]
        import bench
        d = bench.Dist.__new__(bench.Dist)
        d.world, d.rank, d.dist = world, rank, dist
        mx = d.max(float(rank) + 0.5)
        uid = d.bcast_bytes(b"x" * 128 if rank == 0 else None)
        if rank == 0:
            Hf, Sf, _ = orc.build_hs_refined(p)
            Hr = np.zeros_like(Hf)
            Sr = np.zeros_like(Sf)
            Hr[il] = hp.numpy().view(np.complex128)
            Sr[il] = sp.numpy().view(np.complex128)
            q.put((b, hb.rel_frobenius_error_lower(Hr, Hf), hb.rel_frobenius_error_lower(Sr, Sf), mx, uid))
    finally:
        dist.destroy_process_group()


def test_sharded_partials_reduce_to_full_result():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    bounds, eh, es, mx, uid = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert bounds == [0, 3, 7]
    assert eh <= 1e-14 and es <= 1e-14
    assert mx == 1.5 and uid == b"x" * 128


def test_shard_atoms_partition():
    for na in (1, 7, 64, 108, 512):
        for parts in (1, 2, 3, 8):
            if parts > na:
                with pytest.raises(hb.ConfigError):
                    hb.shard_atoms(na, parts)
                continue
            b = hb.shard_atoms(na, parts)
            sizes = np.diff(b)
            assert b[0] == 0 and b[-1] == na and sizes.min() >= 1 and sizes.max() - sizes.min() <= 1


def test_shard_rows_partition():
    """Row-balanced shards: the K = n_atoms n_l rows split evenly (sizes differ by <= 1), each
    shard's row range lies in its atoms and touches the first and the last one, and the global
    rows are covered exactly once."""
    for na, nl in ((1, 7), (7, 25), (16, 49), (108, 121), (512, 121)):
        K = na * nl
        for parts in (1, 2, 3, 8):
            if parts > na:
                with pytest.raises(hb.ConfigError):
                    hb.shard_rows(na, nl, parts)
                continue
            sh = hb.shard_rows(na, nl, parts)
            covered, sizes = 0, []
            for a0, n_loc, r0, r1 in sh:
                assert 0 <= r0 < nl and n_loc * nl - nl < r1 <= n_loc * nl
                assert a0 * nl + r0 == covered  # contiguous, no gap, no overlap
                covered = a0 * nl + r1
                sizes.append(r1 - r0)
            assert covered == K and max(sizes) - min(sizes) <= 1
