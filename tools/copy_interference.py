"""Device-resident build time with and without a concurrent copy on another stream
(development helper): does PCIe traffic slow the contraction kernels?"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402

CFG = {"c1": (16, 49, 1000), "c2": (64, 81, 3000)}
na, nl, ng = CFG[sys.argv[1] if len(sys.argv) > 1 else "c2"]
e = hb.Engine(0, na, nl, ng)
e.fill_synthetic(1)
side = torch.cuda.Stream()
nbytes = 512 << 20
host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dev2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")


def run(label, copy):
    ts, ph = [], []
    for _ in range(6):
        torch.cuda.synchronize()
        if copy:
            with torch.cuda.stream(side):
                for _ in range(8):
                    copy()
        e.build("merged")
        st = e.sync()
        ts.append(st["device_seconds"] * 1e3)
        ph.append(st["phase_seconds"])
        torch.cuda.synchronize()
    ts = sorted(ts[1:])
    last = " ".join(f"{k} {v * 1e3:.3f}" for k, v in ph[-1].items() if v)
    print(f"{label:>10}: build median {ts[len(ts) // 2]:.3f} ms (min {ts[0]:.3f}); last phases {last}", flush=True)


run("alone", None)
run("h2d", lambda: dev.copy_(host, non_blocking=True))
run("d2h", lambda: host.copy_(dev, non_blocking=True))
run("alone", None)
e.close()
