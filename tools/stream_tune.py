"""Sweep the host-buffer drop-in's streaming knobs (first-chunk floor, chunk-growth
calibration, final-H band ratio) at one config: end-to-end wall ms per call with pinned
inputs (development helper; the knobs are the env vars stream_bounds / make_pieces read).

    python tools/stream_tune.py c2 [--out gpurun_out/stream_tune.jsonl]
"""
import argparse
import itertools
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c2", nargs="?")
    ap.add_argument("--floors", default="0.0625,0.03125,0.015625")
    ap.add_argument("--cs", default="1.84e-14,1.45e-14")
    ap.add_argument("--ratios", default="1.0,0.8,0.7")
    ap.add_argument("--calls", type=int, default=6)
    ap.add_argument("--plans", default="", help="explicit chunk plans 'a,b,c;d,e' (HSDLA_B200_STREAM_PLAN)")
    ap.add_argument("--out", default="gpurun_out/stream_tune.jsonl")
    a = ap.parse_args()
    na, nl, ng = CFG[a.config]
    p = hb.generate_problem(na, nl, ng, 1, 0)
    H = np.zeros((ng, ng), np.complex128, order="F")
    S = np.zeros((ng, ng), np.complex128, order="F")
    bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U, H, S]
    for b in bufs:
        hb.host_register(b)
    led = hb.flop_model(p).total()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "a") as f:
        grid = ([(a.floors.split(",")[0], a.cs.split(",")[0], a.ratios.split(",")[0], pl) for pl in a.plans.split(";")]
                if a.plans else [(*t, "") for t in itertools.product(a.floors.split(","), a.cs.split(","),
                                                                     a.ratios.split(","))])
        for fl, c, r, plan in grid:
            if plan:
                os.environ["HSDLA_B200_STREAM_PLAN"] = plan
            os.environ["HSDLA_B200_STREAM_FLOOR"] = fl
            os.environ["HSDLA_B200_STREAM_C"] = c
            os.environ["HSDLA_B200_BAND_RATIO"] = r
            hb.release_cache()
            hb.build_hs_refined(p, H=H, S=S)
            ts, dev = [], []
            for _ in range(a.calls):
                t = time.perf_counter()
                res = hb.build_hs_refined(p, H=H, S=S)
                ts.append(time.perf_counter() - t)
                dev.append(res.stats["device_seconds"])
            rec = {"config": a.config, "plan": plan, "floor": float(fl), "c": float(c), "band_ratio": float(r),
                   "wall_ms": float(np.median(ts)) * 1e3, "device_ms": float(np.median(dev)) * 1e3,
                   "tflops": led / float(np.median(ts)) / 1e12, "launches": res.stats["kernel_launches"]}
            print(json.dumps(rec), flush=True)
            f.write(json.dumps(rec) + "\n")
    for b in bufs:
        hb.host_unregister(b)


if __name__ == "__main__":
    main()
