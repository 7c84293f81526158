"""Breakdown of the host-buffer drop-in (hsdla_b200_build_hs) per call (development helper)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000)}
for name in sys.argv[1:] or ["c2"]:
    na, nl, ng = CFG[name]
    p = hb.generate_problem(na, nl, ng, 1, 0)
    H = np.zeros((ng, ng), np.complex128, order="F")
    S = np.zeros((ng, ng), np.complex128, order="F")
    bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U, H, S]
    for b in bufs:
        hb.host_register(b)
    led = hb.flop_model(p).total()
    for it in range(6):
        t = time.perf_counter()
        r = hb.build_hs_refined(p, H=H, S=S)
        dt = time.perf_counter() - t
        st = r.stats
        print(f"{name} call {it}: wall {dt*1e3:.2f} ms ({led/dt/1e12:.2f} TF/s)  total {st['total_seconds']*1e3:.2f}  "
              f"h2d {st['h2d_seconds']*1e3:.2f}  device {st['device_seconds']*1e3:.2f}  d2h+unpack {st['d2h_seconds']*1e3:.2f}"
              f"  launches {st['kernel_launches']}  phases " + " ".join(f"{k}:{v*1e3:.2f}" for k, v in st["phase_seconds"].items()), flush=True)
    e = hb.Engine(0, na, nl, ng)
    for it in range(3):
        e.build_streamed(p, 0)
        st = e.sync()
    print(f"{name} engine streamed: device {st['device_seconds']*1e3:.2f} h2d {st['h2d_seconds']*1e3:.2f} phases " +
          " ".join(f"{k}:{v*1e3:.2f}" for k, v in st["phase_seconds"].items()))
    e.upload(p)
    for it in range(3):
        e.build()
        st = e.sync()
    print(f"{name} engine whole: device {st['device_seconds']*1e3:.2f} phases " +
          " ".join(f"{k}:{v*1e3:.2f}" for k, v in st["phase_seconds"].items()))
    e.close()
    for b in bufs:
        hb.host_unregister(b)
    hb.release_cache()
