import sys, time
sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb
for name, (na, nl, ng) in {"c1": (16, 49, 1000), "c2": (64, 81, 3000)}.items():
    e = hb.Engine(0, na, nl, ng)
    e.fill_synthetic(1)
    for ov in (False, True, False, True):
        e.set_download_overlap(ov)
        ts = []
        for _ in range(8):
            e.build()
            st = e.sync()
            ts.append(st["device_seconds"] * 1e3)
        ts = sorted(ts[2:])
        print(name, "banded" if ov else "whole ", "median %.3f ms" % ts[len(ts) // 2], flush=True)
    e.close()
