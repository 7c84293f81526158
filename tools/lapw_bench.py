"""Times the LAPW setup kernel (HBM-write bound) inside an engine (development helper)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402

cfgs = {"c2": (64, 8, 3000), "c3": (108, 10, 6000), "c4": (512, 10, 13000)}
for name in sys.argv[1:] or ["c2", "c3"]:
    na, lmax, ng = cfgs[name]
    t = time.time()
    s = hb.make_lapw_system(na, lmax, ng, n_types=2, seed=1)
    e = hb.Engine(0, na, s.n_l, ng)
    best = 1e9
    for _ in range(5):
        e.setup_lapw(s)
        e.sync()
        st = e.setup_time()
        best = min(best, st["ms"])
    print(f"{name}: setup kernel {best:.3f} ms, {st['bytes'] / 1e9:.2f} GB written -> "
          f"{st['bytes'] / best / 1e6:.0f} GB/s (gen {time.time() - t:.1f}s)", flush=True)
    e.close()
