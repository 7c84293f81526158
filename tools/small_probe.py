"""Per-call latency of the host-buffer drop-in on small cells (development helper).

    HSDLA_B200_TRACE=1 python tools/small_probe.py c1 [--calls 20]

Median wall time per build_hs_refined call with pageable and page-locked buffers, and the
stats' split (h2d / device / d2h+unpack).
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "s2": (16, 49, 2000), "s3": (32, 64, 1500), "c2": (64, 81, 3000), "c3": (108, 121, 6000)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1"])
    ap.add_argument("--calls", type=int, default=20)
    a = ap.parse_args()
    for name in a.configs:
        na, nl, ng = CFG[name]
        p = hb.generate_problem(na, nl, ng, 1, 0)
        led = hb.flop_model(p).total()
        H = np.zeros((ng, ng), np.complex128, order="F")
        S = np.zeros((ng, ng), np.complex128, order="F")
        for kind in ("pageable", "pinned"):
            bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U, H, S] if kind == "pinned" else []
            for b in bufs:
                hb.host_register(b)
            try:
                hb.build_hs_refined(p, H=H, S=S)
                ts, sts = [], []
                for _ in range(a.calls):
                    t = time.perf_counter()
                    r = hb.build_hs_refined(p, H=H, S=S)
                    ts.append(time.perf_counter() - t)
                    sts.append(r.stats)
            finally:
                for b in bufs:
                    hb.host_unregister(b)
            i = int(np.argsort(ts)[len(ts) // 2])
            st = sts[i]
            print(f"{name} {kind}: median {ts[i]*1e3:.3f} ms ({led/ts[i]/1e12:.2f} TF/s), min {min(ts)*1e3:.3f}  "
                  f"total {st['total_seconds']*1e3:.3f} h2d {st['h2d_seconds']*1e3:.3f} device "
                  f"{st['device_seconds']*1e3:.3f} d2h+unpack {st['d2h_seconds']*1e3:.3f} launches "
                  f"{st['kernel_launches']}", flush=True)
        hb.release_cache()


if __name__ == "__main__":
    main()
