"""Sweep the host-buffer drop-in's streaming knobs at one config: end-to-end wall ms per call
(development helper; the knobs are the env vars the chunk planner / make_pieces read).

    python tools/stream_tune.py c2 [--plans "2,4,9,18,31;4,9,20,31"] [--tflops 33e12,30e12]
                                   [--ratios 1.0,0.8] [--pageable] [--out gpurun_out/stream_tune.jsonl]

Without --plans the dynamic-programming planner chooses (HSDLA_B200_STREAM_TFLOPS sets its compute
rate); HSDLA_B200_TRACE=1 prints the plan it picked.
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
    ap.add_argument("--plans", default="", help="explicit chunk plans 'a,b,c;d,e' (HSDLA_B200_STREAM_PLAN)")
    ap.add_argument("--tflops", default="33e12", help="planner compute rates (HSDLA_B200_STREAM_TFLOPS)")
    ap.add_argument("--ratios", default="1.0", help="final-H band ratios (HSDLA_B200_BAND_RATIO)")
    ap.add_argument("--pageable", action="store_true", help="plain numpy inputs (default: page-locked)")
    ap.add_argument("--calls", type=int, default=6)
    ap.add_argument("--out", default="gpurun_out/stream_tune.jsonl")
    a = ap.parse_args()
    na, nl, ng = CFG[a.config]
    p = hb.generate_problem(na, nl, ng, 1, 0)
    H = np.zeros((ng, ng), np.complex128, order="F")
    S = np.zeros((ng, ng), np.complex128, order="F")
    bufs = [] if a.pageable else [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U, H, S]
    for b in bufs:
        hb.host_register(b)
    led = hb.flop_model(p).total()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    plans = a.plans.split(";") if a.plans else [""]
    try:
        with open(a.out, "a") as f:
            for plan, tf, r in itertools.product(plans, a.tflops.split(","), a.ratios.split(",")):
                if plan:
                    os.environ["HSDLA_B200_STREAM_PLAN"] = plan
                else:
                    os.environ.pop("HSDLA_B200_STREAM_PLAN", None)
                os.environ["HSDLA_B200_STREAM_TFLOPS"] = tf
                os.environ["HSDLA_B200_BAND_RATIO"] = r
                hb.release_cache()  # fresh engines: the plans are rebuilt with these knobs
                hb.build_hs_refined(p, H=H, S=S)
                ts, dev = [], []
                for _ in range(a.calls):
                    t = time.perf_counter()
                    res = hb.build_hs_refined(p, H=H, S=S)
                    ts.append(time.perf_counter() - t)
                    dev.append(res.stats["device_seconds"])
                rec = {"config": a.config, "inputs": "pageable" if a.pageable else "pinned", "plan": plan or "dp",
                       "tflops_model": float(tf), "band_ratio": float(r), "wall_ms": float(np.median(ts)) * 1e3,
                       "device_ms": float(np.median(dev)) * 1e3, "tflops": led / float(np.median(ts)) / 1e12,
                       "launches": res.stats["kernel_launches"]}
                print(json.dumps(rec), flush=True)
                f.write(json.dumps(rec) + "\n")
    finally:
        for b in bufs:
            hb.host_unregister(b)
        hb.release_cache()


if __name__ == "__main__":
    main()
