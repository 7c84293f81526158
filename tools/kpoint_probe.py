"""k-point batch throughput (hsdla_b200_build_hs_kpoints) against per-call drop-in builds
(development helper): n k-points of one cell, pinned and pageable coefficients.

    python tools/kpoint_probe.py [c1|c2|c3] [--nk 8]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000)}
ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--nk", type=int, default=8)
a = ap.parse_args()
na, nl, ng = CFG[a.config]
base = hb.generate_problem(na, nl, ng, 1, 0)
As = [hb.generate_problem(na, nl, ng, 10 + k, 0).A for k in range(a.nk)]
Bs = [hb.generate_problem(na, nl, ng, 10 + k, 0).B for k in range(a.nk)]
Hs = [np.zeros((ng, ng), np.complex128, order="F") for _ in range(a.nk)]
Ss = [np.zeros((ng, ng), np.complex128, order="F") for _ in range(a.nk)]
led = hb.flop_model(base).total()
for pinned in (False, True):
    bufs = As + Bs + Hs + Ss + [base.T_AA, base.T_AB, base.T_BB, base.U]
    if pinned:
        for M in bufs:
            hb.host_register(M)
    hb.build_hs_kpoints(base, As, Bs, Hs=Hs, Ss=Ss)  # warm
    t = time.perf_counter()
    hb.build_hs_kpoints(base, As, Bs, Hs=Hs, Ss=Ss)
    dt = (time.perf_counter() - t) / a.nk
    # per-call drop-in over the same k-points
    p = hb.generate_problem(na, nl, ng, 1, 0)
    p.A, p.B = As[0], Bs[0]
    hb.build_hs_refined(p, H=Hs[0], S=Ss[0])
    t = time.perf_counter()
    for k in range(a.nk):
        p.A, p.B = As[k], Bs[k]
        hb.build_hs_refined(p, H=Hs[k], S=Ss[k])
    dc = (time.perf_counter() - t) / a.nk
    print(f"{a.config} {'pinned' if pinned else 'pageable'}: k-point batch {dt*1e3:.2f} ms per k-point "
          f"({led/dt/1e12:.1f} TF/s), per-call drop-in {dc*1e3:.2f} ms ({led/dc/1e12:.1f} TF/s)", flush=True)
    if pinned:
        for M in bufs:
            hb.host_unregister(M)
    hb.release_cache()
