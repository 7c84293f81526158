"""PCIe duplex probe (development helper): pinned H2D and D2H alone and concurrently on two
streams, at the C1 k-point batch's per-k-point sizes (25 MB up, 16 MB down) and larger.

    python tools/duplex_probe.py
"""
import torch


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    for up_mb, dn_mb in ((25, 16), (100, 64), (400, 256)):
        hu = torch.empty(up_mb << 20, dtype=torch.uint8).pin_memory()
        hd = torch.empty(dn_mb << 20, dtype=torch.uint8).pin_memory()
        du = torch.empty(up_mb << 20, dtype=torch.uint8, device="cuda")
        dd = torch.empty(dn_mb << 20, dtype=torch.uint8, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def up():
            du.copy_(hu, non_blocking=True)

        def dn():
            hd.copy_(dd, non_blocking=True)

        def both():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                up()
            with torch.cuda.stream(s2):
                dn()
            cur.wait_stream(s1)
            cur.wait_stream(s2)

        tu, td, tb = timed(up), timed(dn), timed(both)
        print(f"up {up_mb} MB {tu:.3f} ms ({up_mb * 1.048576 / tu:.1f} GB/s)  down {dn_mb} MB {td:.3f} ms "
              f"({dn_mb * 1.048576 / td:.1f} GB/s)  concurrent {tb:.3f} ms (sum alone {tu + td:.3f}, "
              f"{(up_mb + dn_mb) * 1.048576 / tb:.1f} GB/s combined)", flush=True)


if __name__ == "__main__":
    main()
