"""Principal-submatrix parity at the largest BASELINE configs (C4 and C5-hi), against the
UNMODIFIED reference (oracle/_ref, BlockedParallel on every host core) — TEST
INFRASTRUCTURE run as an evidence script (too heavy for the per-round test suite).

H[J,J] and S[J,J] depend only on the columns J of A and B, so the reference's
build_hs_refined on the J-sliced problem yields them exactly; |J| = 512
random G-vectors.  The GPU side is the public drop-in on the FULL problem.
--full: the whole lower triangle against the reference's full run (SURVEY §8d asks for
this at C1-C3).

    python tools/parity_large.py [c4 c5hi] [--j 512] [--out gpurun_out/parity_large.json]
    python tools/parity_large.py c1 c2 c3 --full --out gpurun_out/parity_full.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_07206_b200 as hb  # noqa: E402
from oracle.oracle import Reference, _Problem  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000), "c4": (512, 121, 13000),
       "c5hi": (1024, 81, 20000)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c4", "c5hi"])
    ap.add_argument("--j", type=int, default=512)
    ap.add_argument("--full", action="store_true", help="whole lower triangle vs the reference's full run")
    ap.add_argument("--out", default="gpurun_out/parity_large.json")
    a = ap.parse_args()
    ref = Reference()
    res = []
    for name in a.configs:
        na, nl, ng = CFG[name]
        t0 = time.time()
        p = hb.generate_problem(na, nl, ng, 1, 0)
        t_gen = time.time() - t0
        t0 = time.time()
        r = hb.build_hs_refined(p)
        t_gpu = time.time() - t0
        if a.full:
            t0 = time.time()
            out = ref.build_hs(p, "refined", threads=os.cpu_count() or 1, blocked=True)
            t_ref = time.time() - t0
            eh = hb.rel_frobenius_error_lower(r.H, out["H"])
            es = hb.rel_frobenius_error_lower(r.S, out["S"])
            rec = {"config": name, "n_atoms": na, "n_l": nl, "n_g": ng, "J": "all", "rel_err_H": eh, "rel_err_S": es,
                   "tol": 1e-11, "pass": bool(eh <= 1e-11 and es <= 1e-11), "gen_s": t_gen, "gpu_call_s": t_gpu,
                   "gpu_device_s": r.stats["device_seconds"], "reference_full_s": t_ref,
                   "reference_ledger_tflops": hb.flop_model(p).total() / t_ref / 1e12,
                   "oracle": "oracle/_ref (unmodified reference, Strategy::Cpu BlockedParallel), full problem"}
            print(json.dumps(rec), flush=True)
            res.append(rec)
            del p, r, out
            hb.release_cache()
            continue
        J = np.sort(np.random.default_rng(11).choice(ng, size=a.j, replace=False))
        sl = _Problem(na, nl, a.j, np.asfortranarray(p.A[:, J]), np.asfortranarray(p.B[:, J]), p.T_AA, p.T_AB,
                      p.T_BB, p.U, p.hpd_flags.astype(np.uint8))
        t0 = time.time()
        out = ref.build_hs(sl, "refined", threads=os.cpu_count() or 1, blocked=True)
        t_ref = time.time() - t0
        sub = np.ix_(J, J)
        eh = hb.rel_frobenius_error_lower(np.asfortranarray(r.H[sub]), out["H"])
        es = hb.rel_frobenius_error_lower(np.asfortranarray(r.S[sub]), out["S"])
        rec = {"config": name, "n_atoms": na, "n_l": nl, "n_g": ng, "J": a.j, "rel_err_H": eh, "rel_err_S": es,
               "tol": 1e-11, "pass": bool(eh <= 1e-11 and es <= 1e-11), "gen_s": t_gen, "gpu_call_s": t_gpu,
               "gpu_device_s": r.stats["device_seconds"], "reference_sliced_s": t_ref,
               "oracle": "oracle/_ref (unmodified reference, Strategy::Cpu BlockedParallel) on the J-sliced problem"}
        print(json.dumps(rec), flush=True)
        res.append(rec)
        del p, r, sl, out
        hb.release_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
