"""Quick device-resident timing of the engine (development helper, not the bench contract)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402

cfgs = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000), "c4": (512, 121, 13000)}
for name in sys.argv[1:] or ["c2", "c3"]:
    na, nl, ng = cfgs[name]
    t = time.time()
    p = hb.generate_problem(na, nl, ng, 1, 0)
    tg = time.time() - t
    e = hb.Engine(0, na, nl, ng)
    e.upload(p)
    led_r = hb.flop_model(p).total()
    for algo in ("merged", "fused", "refined", "original"):
        for it in range(4):
            e.build(algo)
            st = e.sync()
        kt = e.kernel_times()
        dev = st["device_seconds"]
        led = led_r
        print(f"{name} {algo}: gen {tg:.1f}s  device {dev*1e3:.2f} ms  {led/dev/1e12:.2f} TF/s(ledger)  "
              f"phases {{{', '.join(f'{k}: {v*1e3:.2f}' for k, v in st['phase_seconds'].items())}}} ms  "
              f"S-kernel {kt['s_flops']/kt['s_ms']/1e9:.2f} TF/s  H-kernel {kt['h_flops']/kt['h_ms']/1e9:.2f} TF/s",
              flush=True)
    e.close()
