"""Small, fixed workload for ncu captures (development helper): `builds` device-resident
builds of a config (default algo merged), or `--lapw` setup passes.  Launch order per
merged build: diag_scale, S (TRI), expand, W = [W_A; W_B] (BATCH, 24-row tiles), H (TRI)."""
import argparse
import sys

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000), "c3": (108, 121, 6000),
       "g2k": (256, 81, 2000), "g10k": (16, 81, 10000), "g20k": (16, 81, 20000)}
ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--builds", type=int, default=3)
ap.add_argument("--algo", default="merged")
ap.add_argument("--lapw", action="store_true")
a = ap.parse_args()
na, nl, ng = CFG[a.config]
if a.lapw:
    lmax = int(round(nl ** 0.5)) - 1
    s = hb.make_lapw_system(na, lmax, ng, n_types=2, seed=1)
    e = hb.Engine(0, na, s.n_l, ng)
    for _ in range(a.builds):
        e.setup_lapw(s)
        e.sync()
else:
    e = hb.Engine(0, na, nl, ng)
    e.fill_synthetic(1)
    for _ in range(a.builds):
        e.build(a.algo)
        e.sync()
e.close()
