"""HSDL file path timing (development helper): raw page-cache read rate vs the
library's streamed build from the file."""
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c2": (64, 81, 3000), "c3": (108, 121, 6000)}
for name in sys.argv[1:] or ["c2"]:
    na, nl, ng = CFG[name]
    p = hb.generate_problem(na, nl, ng, 1, 0)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "p.hsdl")
        hb.save_problem(p, path)
        size = os.path.getsize(path)
        for _ in range(2):
            t = time.perf_counter()
            with open(path, "rb", buffering=0) as f:
                while f.read(64 << 20):
                    pass
            raw = time.perf_counter() - t
        led = hb.flop_model(p).total()
        import numpy as np
        H = np.zeros((ng, ng), np.complex128, order="F")
        S = np.zeros((ng, ng), np.complex128, order="F")
        for it in range(4):
            t = time.perf_counter()
            r = hb.build_hs_file(path, H=H, S=S)
            dt = time.perf_counter() - t
            print(f"{name} call {it}: wall {dt*1e3:.1f} ms ({led/dt/1e12:.2f} TF/s) load {r.stats['h2d_seconds']*1e3:.1f} ms "
                  f"({size/r.stats['h2d_seconds']/1e9:.2f} GB/s) device {r.stats['device_seconds']*1e3:.1f} ms; "
                  f"raw read {raw*1e3:.1f} ms ({size/raw/1e9:.2f} GB/s)", flush=True)
    hb.release_cache()
