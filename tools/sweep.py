"""Single-GPU throughput sweep over BASELINE.json's configs (C1-C4 and the C5 grid
N_L 81 x N_G 2000..20000 x N_A 16..1024).  Device-resident builds on synthetic
device-filled inputs (Engine.fill_synthetic: timing does not depend on the values;
parity at these shapes is covered by tests/ with the reference generator).

    python tools/sweep.py [--algo fused] [--out gpurun_out/sweep.jsonl] [--only c4]

One JSON line per point: ledger TF/s (= pipeline::flop_model / device time of the
whole build, CUDA events on the engine stream), fraction of the in-process DMMA
peak, the S / H contraction kernels' own rates, device bytes.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1712_07206_b200 as hb  # noqa: E402

NAMED = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000), "c4": (512, 121, 13000)}


def points(only):
    pts = [(k, *v) for k, v in NAMED.items()]
    for ng in (2000, 5000, 10000, 15000, 20000):
        for na in (16, 64, 256, 1024):
            pts.append((f"c5_na{na}_ng{ng}", na, 81, ng))
    if only:
        pts = [p for p in pts if p[0] in only.split(",")]
    return pts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="merged", choices=["merged", "fused", "refined", "original"])
    ap.add_argument("--arith", default="3m", choices=["3m", "4m"])
    ap.add_argument("--out", default="gpurun_out/sweep.jsonl")
    ap.add_argument("--only", default="")
    ap.add_argument("--budget", type=float, default=4.0, help="seconds of timed builds per point (>= 2 builds)")
    args = ap.parse_args()
    peak = hb.fp64_peak(0, 1.0)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "a") as f:
        for name, na, nl, ng in points(args.only):
            t0 = time.time()
            e = hb.Engine(0, na, nl, ng)
            e.set_arith(args.arith)
            e.fill_synthetic(1)
            e.build(args.algo)  # warm-up (also allocates X2 for fused / original)
            st = e.sync()
            e.kernel_times(reset=True)
            n = max(2, min(20, int(args.budget / max(st["device_seconds"], 1e-6))))
            dev = []
            for _ in range(n):
                e.build(args.algo)
                dev.append(e.sync()["device_seconds"])
            kt = e.kernel_times()
            led = hb.flop_model(hb.empty_problem(na, nl, ng)).total()
            t = sum(dev) / len(dev)
            rec = {"point": name, "n_atoms": na, "n_l": nl, "n_g": ng, "algo": args.algo, "builds": n,
                   "build_ms": t * 1e3, "min_ms": min(dev) * 1e3, "ledger_flops": led,
                   "tflops": led / t / 1e12, "dmma_peak_tflops": peak,
                   "arith": args.arith, "executed_tflops": bench.executed_flops(na, nl, ng, args.arith, args.algo) / t / 1e12,
                   "executed_frac_of_dmma_peak": bench.executed_flops(na, nl, ng, args.arith, args.algo) / t / 1e12 / peak,
                   "s_kernel_tflops": kt["s_flops"] / kt["s_ms"] / 1e9 if kt["s_ms"] else None,
                   "h_kernel_tflops": kt["h_flops"] / kt["h_ms"] / 1e9 if kt["h_ms"] else None,
                   "phase_ms": {k: v * 1e3 for k, v in st["phase_seconds"].items()},
                   "device_gb": st["peak_device_bytes"] / 1e9, "wall_s": time.time() - t0}
            print(json.dumps(rec), flush=True)
            f.write(json.dumps(rec) + "\n")
            e.close()


if __name__ == "__main__":
    main()
