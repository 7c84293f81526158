"""The reference CPU path (oracle/_ref: unmodified reference, Strategy::Cpu BlockedParallel,
block 128, all host threads) timed on a subsampled instance of each BASELINE config:
--mode atoms (same N_L, N_G; H and S are sums over atoms, so ledger flop/s is the
full-size rate) or --mode columns (all atoms, fewer G-vectors: SURVEY section 8d's recipe
for C4/C5, full-length dot products).

    python tools/cpu_ref_sweep.py [--mode columns] [--budget 10] [--out gpurun_out/cpu_ref_sweep.jsonl]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000), "c4": (512, 121, 13000)}

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=list(CFG))
ap.add_argument("--budget", type=float, default=10.0)
ap.add_argument("--mode", default="atoms", choices=["atoms", "columns"])
ap.add_argument("--out", default="gpurun_out/cpu_ref_sweep.jsonl")
a = ap.parse_args()
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "a") as f:
    for name in a.configs:
        na, nl, ng = CFG[name]
        r = bench.cpu_reference_sample(na, nl, ng, a.budget, mode=a.mode)
        r.update(config=name, n_atoms=na, n_l=nl, n_g=ng)
        print(json.dumps(r), flush=True)
        f.write(json.dumps(r) + "\n")
