"""End-to-end (host buffers) throughput of the public drop-in across the BASELINE configs.

    python tools/e2e_sweep.py [c2 c3 c4] [--out gpurun_out/e2e_sweep.jsonl]

For each config: the reference generator's problem in host memory, then
paper_1712_07206_b200.build_hs_refined -> hsdla_b200_build_hs (H2D of A, B, T, U and the
D2H of H, S inside every call), with the inputs pinned (hsdla_b200_host_register) and
pageable.  One JSON line per (config, memory kind): ledger TF/s per call.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000), "c4": (512, 121, 13000),
       "c5_na64_ng20000": (64, 81, 20000), "c5_na256_ng10000": (256, 81, 10000), "c5_na1024_ng5000": (1024, 81, 5000)}


def timed(p, H, S, n):
    hb.build_hs_refined(p, H=H, S=S)  # warm (engine cache)
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        r = hb.build_hs_refined(p, H=H, S=S)
        ts.append(time.perf_counter() - t)
    return float(np.median(ts)), r.stats


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c3", "c4"])
    ap.add_argument("--out", default="gpurun_out/e2e_sweep.jsonl")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "a") as f:
        for name in a.configs:
            na, nl, ng = CFG[name]
            p = hb.generate_problem(na, nl, ng, 1, 0)
            led = hb.flop_model(p).total()
            H = np.zeros((ng, ng), np.complex128, order="F")
            S = np.zeros((ng, ng), np.complex128, order="F")
            n = 5 if name in ("c1", "c2") else 3 if name == "c3" else 2
            dt_pg, st_pg = timed(p, H, S, n)
            bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U, H, S]
            for b in bufs:
                hb.host_register(b)
            try:
                dt_pin, st_pin = timed(p, H, S, n)
            finally:
                for b in bufs:
                    hb.host_unregister(b)
            hb.release_cache()
            h2d = sum(b.nbytes for b in (p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U))
            for kind, dt, st in (("pinned", dt_pin, st_pin), ("pageable", dt_pg, st_pg)):
                rec = {"config": name, "n_atoms": na, "n_l": nl, "n_g": ng, "inputs": kind, "ms_per_call": dt * 1e3,
                       "tflops": led / dt / 1e12, "device_ms": st["device_seconds"] * 1e3,
                       "h2d_bytes": int(h2d), "d2h_bytes": int(2 * ng * (ng + 1) // 2 * 16),
                       "api": "build_hs_refined -> hsdla_b200_build_hs"}
                print(json.dumps(rec), flush=True)
                f.write(json.dumps(rec) + "\n")
            del p, H, S


if __name__ == "__main__":
    main()
