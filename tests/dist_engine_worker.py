"""Worker of tests/test_gpu_multi.py::test_multigpu_torchrun_engine_path (launched by torchrun,
one process per GPU): the multi-process engine path of the drop-in.

Each rank generates only its atom shard of config 1 (generate_problem_shard), builds it on its
GPU, joins the NCCL communicator (hsdla_b200_engine_set_comm, id from rank 0), reduces
(ROOT or SCATTER) and downloads the packed ranges it owns.  The owned ranges are disjoint, so
a gloo sum assembles the full H, S on rank 0, which compares them with the unmodified
reference (oracle/_ref; the C restatement when it is not built) on the full problem."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reduce", default="scatter", choices=["scatter", "root"])
    ap.add_argument("--out", required=True)
    ap.add_argument("--dims", default="16,49,1000")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1712_07206_b200 as hb
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dist.init_process_group("gloo")
    na, nl, ng = (int(x) for x in args.dims.split(","))
    a0, na_sh, r0, r1 = hb.shard_rows(na, nl, world)[rank]
    p = hb.generate_problem_shard(na, nl, ng, a0, a0 + na_sh, 1, 0)
    e = hb.Engine(local, p.n_atoms, nl, ng, row_begin=r0, row_end=r1)
    obj = [hb.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    e.set_comm(obj[0], world, rank)
    e.set_reduce_mode(args.reduce)
    e.set_download_overlap(True)
    e.upload(p, 0)
    e.build()
    e.reduce(0)
    H, S = e.download()
    own = e.owned()
    e.sync()
    e.set_comm(None, 1, 0)
    e.close()
    # disjoint owned ranges: the sum over ranks is the assembled result
    th = torch.from_numpy(np.ascontiguousarray(H).view(np.float64).copy())
    ts = torch.from_numpy(np.ascontiguousarray(S).view(np.float64).copy())
    dist.reduce(th, dst=0)
    dist.reduce(ts, dst=0)
    counts = torch.tensor([sum(b1 - b0 for b0, b1 in own)], dtype=torch.float64)
    dist.reduce(counts, dst=0)
    if rank == 0:
        from oracle.oracle import Reference, Restatement
        full = hb.generate_problem(na, nl, ng, 1, 0)
        if Reference.available():
            ref = Reference().build_hs(full, "refined", threads=os.cpu_count() or 1, blocked=True)
            H0, S0 = ref["H"], ref["S"]
        else:
            H0, S0, _ = Restatement().build_hs_refined(full)
        Hg = th.numpy().view(np.complex128).reshape(ng, ng)
        Sg = ts.numpy().view(np.complex128).reshape(ng, ng)
        Hg, Sg = np.asfortranarray(Hg), np.asfortranarray(Sg)
        assert int(counts.item()) == ng * (ng + 1) // 2, counts.item()
        np.savez(args.out, err_h=hb.rel_frobenius_error_lower(Hg, H0), err_s=hb.rel_frobenius_error_lower(Sg, S0))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
