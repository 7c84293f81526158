"""One traced drop-in call per buffer kind at a config (development helper; run with HSDLA_B200_TRACE=1 for the timelines)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000)}
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["pageable", "pinned"]
na, nl, ng = CFG[name]
p = hb.generate_problem(na, nl, ng, 1, 0)
H = np.zeros((ng, ng), np.complex128, order="F")
S = np.zeros((ng, ng), np.complex128, order="F")
bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U, H, S]
led = hb.flop_model(p).total()
for kind in kinds:
    if kind == "pinned":
        for b in bufs:
            hb.host_register(b)
    for it in range(6):
        print(f"==== {name} {kind} call {it}", file=sys.stderr, flush=True)
        t = time.perf_counter()
        r = hb.build_hs_refined(p, H=H, S=S)
        dt = time.perf_counter() - t
        ph = " ".join(f"{k} {v * 1e3:.3f}" for k, v in r.stats["phase_seconds"].items() if v)
        print(f"{name} {kind} call {it}: wall {dt*1e3:.3f} ms ({led/dt/1e12:.2f} TF/s) device "
              f"{r.stats['device_seconds']*1e3:.3f}; phases {ph}", flush=True)
    if kind == "pinned":
        for b in bufs:
            hb.host_unregister(b)
