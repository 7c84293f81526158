#!/usr/bin/env python
"""Benchmark: HSDLA H+S construction per k-point on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--scaling weak|strong]
                    [--reduce scatter|root] [--impl b200|reference]

One "step" = one k-point: the full refined H/S build (pipeline.cpp:281-329) of one
synthetic problem (generate_problem, seed 1: the reference generator, bit-identical).
Default workload = BASELINE.json configs[1] ("NaCl-like cell: 64 atoms, lmax=8, N_G~3000,
single k-point on 1 B200") = (64, 81, 3000).

Multi-GPU (torchrun, one process per GPU): the K = N_A N_L rows of ONE problem are split
evenly over the N ranks (shard_rows: each rank holds the atoms its rows touch and generates only
those, generate_problem_shard) and the partial packed H, S are summed with NCCL inside the timed
region (the path's one exchange step):
  --scaling weak   (default) the problem has 64 N atoms of config c2 -- fixed work per GPU;
  --scaling strong the config's own atom count split N ways (BASELINE configs[2..3]: c3 at
                   N = 1/2/4/8, c4 at N = 8) -- fixed total work.
At N = 1 both are the single-GPU line of the config.  --reduce scatter (default: every GPU
receives its slices of H, S) or root (ncclReduce onto rank 0).

`value` = reference-ledger FLOP/s (flop_model, pipeline.cpp:336-364; complex MAC = 8 flops)
of the whole job with inputs already in HBM, device-timed with CUDA events on the engine
stream, max over ranks.  `fp64_frac_of_peak` = EXECUTED flops per second / (N x the measured
FP64 DMMA peak) -- the efficiency figure (the ledger rate can exceed the peak: the merged
algorithm and the 3M products execute fewer flops than the reference's ledger counts).
`e2e` = the same metric through the public drop-in API with PAGEABLE host buffers (a plain
numpy / std::vector caller) -- H2D of the inputs and D2H of H, S inside the timed region;
`e2e_pinned` is the same with page-locked buffers.  `roofline` = the dominant kernel (the H
contraction) against the FP64 DMMA peak measured in-process.  `cpu_baseline` = the reference
CPU path (oracle/_ref, compiled from the reference sources) on this host.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H+S build time & FP64 TFLOP/s (frac of peak) per k-point at 1/2/4/8 B200"
CONFIGS = {
    "c1": (16, 49, 1000, "small synthetic FLAPW system: 16 atoms, lmax 6 (N_L 49), N_G 1000"),
    "c2": (64, 81, 3000, "NaCl-like cell: 64 atoms, lmax 8 (N_L 81), N_G 3000, single k-point"),
    "c3": (108, 121, 6000, "AuAg-like alloy: 108 atoms, lmax 10 (N_L 121), N_G 6000"),
    "c4": (512, 121, 13000, "CuCd-like large cell: 512 atoms, lmax 10 (N_L 121), N_G 13000"),
}


def executed_flops(na, nl, ng, arith, algo="merged"):
    """Real flops the GPU executes for one build: the complex-MAC work at 8 flops per MAC
    (4M) or 6 (3M) -- 16 K N_G^2 + 32 N_A N_L^2 N_G for the merged algorithm, 20 K N_G^2 +
    24 N_A N_L^2 N_G for the others -- plus 2 K N_G."""
    K = na * nl
    if algo == "merged":
        cmac8 = 16 * K * ng * ng + 32 * na * nl * nl * ng
    else:
        cmac8 = 20 * K * ng * ng + 24 * na * nl * nl * ng
    return (cmac8 // 8 * 6 if arith == "3m" else cmac8) + 2 * K * ng


H_KERNEL = {"merged": "merged H = [A;B]^H [W_A;W_B]", "fused": "fused H = [Z;B;A]^H [B;Z;X]",
            "refined": "her2k [Z;B]^H [B;Z]", "original": "h_aa_update Lft^H W"}


def ledger_flops(na, nl, ng, variant="refined"):
    # pipeline.cpp:336-364, refined: 20 K N_G^2 + 24 N_A N_L^2 N_G + 2 K N_G.  The original
    # variant (generate_problem(..., n_not_hpd=0): every T_AA factorises) swaps the herkx
    # and one hemm for potrf + trmm + herk(B_T).
    K = na * nl
    if variant == "original":
        return (20 * K * ng * ng + 16 * na * nl * nl * ng + 2 * K * ng + na * (4 * nl ** 3 // 3)
                + 4 * na * nl * nl * ng)
    return 20 * K * ng * ng + 24 * na * nl * nl * ng + 2 * K * ng


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max((float(r[3]) for r in self.rows if len(r) >= 9 and
                                    r[3].replace(".", "").isdigit()), default=None)}


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo")  # bootstrap + scalar reductions only; data moves over NCCL
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x):
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def bcast_bytes(self, b):
        if self.world == 1:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
def cpu_reference_sample(na, nl, ng, budget_s, steps=1, warmup=0, mode="atoms"):
    """Time the reference CPU build_hs_refined (Strategy::Cpu, BlockedParallel,
    block 128, all host threads) on a subsampled instance of the workload.

    mode "atoms": same N_L and N_G (so the reference's column-panel parallelism is the
    full-size one), N_A' atoms chosen so one step takes ~budget_s.  H and S are sums
    over atoms, so ledger-flops/s on N_A' atoms is the full-size rate (an upper bound
    when the short K' = N_A' N_L dot products stay in cache).
    mode "columns" (SURVEY section 8d for C4/C5): all atoms, N_G' < N_G columns chosen so
    one step takes ~budget_s; the full-length K dot products of the full-size run."""
    from oracle.oracle import Reference, Restatement
    threads = os.cpu_count() or 1
    if Reference.available():
        ref, kind = Reference(), "reference"
        run = lambda p: ref.build_hs(p, "refined", threads=threads, blocked=True, block=128, want_hs=False)
    else:  # the C restatement (single-threaded port)
        ref, kind, threads = Restatement(), "port", 1
        run = lambda p: ref.build_hs_refined(p)
    na_s, ng_s = na, ng
    if mode == "columns" and kind == "reference":
        # full-size time extrapolated phase by phase: s, her2k, herkx ~ K N_G^2;
        # z_loop, hemm_loop ~ N_A N_L^2 N_G (the sample's N_G' is chosen by the same model)
        quad = ("s", "her2k", "herkx")

        def split(res):
            ph = dict(res["phases"])
            big = sum(v for k, v in ph.items() if k in quad)
            return big, sum(ph.values()) - big

        ng_p = min(ng, 256)
        big, small = split(ref.build_hs(ref.generate_problem(na, nl, ng_p, 1, 0), "refined", threads=threads,
                                        blocked=True, block=128, want_hs=False))
        a_, b_ = big / ng_p ** 2, small / ng_p
        ng_s = int(min(ng, max(ng_p, (-b_ + (b_ * b_ + 4 * a_ * budget_s) ** 0.5) / (2 * a_ + 1e-30))))
        p = ref.generate_problem(na, nl, ng_s, 1, 0)
        for _ in range(warmup):
            run(p)
        ts = []
        for _ in range(steps):
            t = time.perf_counter()
            res = ref.build_hs(p, "refined", threads=threads, blocked=True, block=128, want_hs=False)
            ts.append(time.perf_counter() - t)
            big, small = split(res)
        dt = sum(ts) / len(ts)
        t_full = big * (ng / ng_s) ** 2 + small * (ng / ng_s) + max(0.0, dt - big - small) * (ng / ng_s) ** 2
        return {"value": ledger_flops(na, nl, ng) / t_full / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
                "sample": f"refined H+S of ({na} atoms, N_L {nl}, {ng_s} of {ng} G-vectors), full-size time "
                          f"extrapolated per phase (K N_G^2 phases x (N_G/N_G')^2, per-atom phases x N_G/N_G'): "
                          f"{t_full:.1f} s per k-point; reference Strategy::Cpu BlockedParallel block 128, "
                          f"{threads} threads, {dt:.2f} s per sample",
                "seconds_per_sample": dt, "seconds_full_extrapolated": t_full, "n_atoms_sample": na,
                "n_g_sample": ng_s, "sampling": "columns (extrapolated)"}
    p = ref.generate_problem(1, nl, ng, 1, 0)
    t = time.perf_counter()
    run(p)
    rate = ledger_flops(1, nl, ng) / max(time.perf_counter() - t, 1e-6)
    na_s = int(max(1, min(na, budget_s * rate / ledger_flops(1, nl, ng))))
    p = ref.generate_problem(na_s, nl, ng_s, 1, 0)
    for _ in range(warmup):
        run(p)
    t = time.perf_counter()
    for _ in range(steps):
        run(p)
    dt = (time.perf_counter() - t) / steps
    what = f"{na_s} of {na} atoms, N_L {nl}, N_G {ng}"
    return {"value": ledger_flops(na_s, nl, ng_s) / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
            "sample": f"refined H+S of ({what}); "
                      f"{'reference Strategy::Cpu BlockedParallel block 128' if kind == 'reference' else 'C port'}"
                      f", {threads} threads, {dt:.2f} s per k-point sample",
            "seconds_per_sample": dt, "n_atoms_sample": na_s, "n_g_sample": ng_s, "sampling": mode}


def workload(args, world):
    """(n_atoms_total, n_l, n_g, description) of this run: weak scaling multiplies the config's
    atoms by the rank count, strong scaling keeps them."""
    na, nl, ng, desc = CONFIGS[args.config]
    if world > 1 and args.scaling == "weak":
        return na * world, nl, ng, f"{desc} x {world} (one {na * world}-atom cell, {na} atoms per GPU)"
    return na, nl, ng, desc


def run_reference_arm(args):
    """The reference's own CPU build_hs_refined (oracle/_ref: the unmodified sources compiled
    here; Strategy::Cpu, BlockedParallel, block 128, every host thread) on the B200 arm's
    workload.  Timed steps run the FULL problem when K of them fit ~15 minutes (C2: ~22 s
    each on 16 threads); otherwise an atom-subsampled instance of the same N_L and N_G
    (same_config false).  Warm-up steps run a small atom sample (the code path, not the size)."""
    d = Dist()
    if d.rank != 0:
        d.close()
        return 0
    from oracle.oracle import Reference, Restatement
    na, nl, ng, desc = workload(args, args.gpus)
    threads = os.cpu_count() or 1
    if Reference.available():
        ref, kind = Reference(), "reference"
        run = lambda p: ref.build_hs(p, "refined", threads=threads, blocked=True, block=128, want_hs=False)  # noqa
    else:
        ref, kind, threads = Restatement(), "port", 1
        run = lambda p: ref.build_hs_refined(p)  # noqa: E731
    # rate probe on one atom (same N_L, N_G): predicts the full step
    p1 = ref.generate_problem(1, nl, ng, 1, 0)
    t = time.perf_counter()
    run(p1)
    rate1 = ledger_flops(1, nl, ng) / max(time.perf_counter() - t, 1e-6)
    t_full = ledger_flops(na, nl, ng) / rate1
    full = t_full * args.steps <= args.ref_budget
    na_s = na if full else int(max(1, min(na, 30.0 * rate1 / ledger_flops(1, nl, ng))))
    pw = ref.generate_problem(max(1, min(na_s, 4)), nl, ng, 1, 0)
    for _ in range(args.warmup):
        run(pw)
    p = ref.generate_problem(na_s, nl, ng, 1, 0)
    t = time.perf_counter()
    for _ in range(args.steps):
        run(p)
    dt = (time.perf_counter() - t) / args.steps
    value = ledger_flops(na_s, nl, ng) / dt / 1e12
    sample = (f"refined H+S of the full ({na} atoms, N_L {nl}, N_G {ng}) problem" if full else
              f"refined H+S of ({na_s} of {na} atoms, N_L {nl}, N_G {ng}); H, S are sums over atoms, so the "
              f"ledger rate is the full-size one") + \
        f"; {'reference Strategy::Cpu BlockedParallel block 128' if kind == 'reference' else 'C port'}, " \
        f"{threads} threads, {dt:.2f} s per step"
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generate_problem, seed 1)",
        "impl": "reference",
        "config": {"workload": f"{args.config}: {desc}", "n_atoms": na, "n_l": nl, "n_g": ng,
                   "timed_n_atoms": na_s, "same_config": full,
                   "warmup": f"{pw.n_atoms}-atom sample per warm-up step"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    d.close()
    return 0


# ---------------------------------------------------------------------------
def load_traffic(config, key="dram_bytes_per_launch"):
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(config, {}).get(key)
    except (OSError, ValueError):
        return None


def run_b200(args):
    import torch
    import paper_1712_07206_b200 as hb

    d = Dist()
    P = d.world
    dev = d.local
    torch.cuda.set_device(dev)
    na_total, nl, ng, desc = workload(args, P)
    # this rank's row-balanced shard of ONE problem: the K rows split evenly, the rank holds the
    # atoms its rows touch (bit-identical rows of generate_problem(na_total, ...))
    a0, na_sh, r0, r1 = hb.shard_rows(na_total, nl, P)[d.rank]
    p = (hb.generate_problem(na_total, nl, ng, 1, 0) if P == 1 else
         hb.generate_problem_shard(na_total, nl, ng, a0, a0 + na_sh, 1, 0))
    na = p.n_atoms
    hb.set_default_arith(args.arith)  # kernel layer + any engine created below
    eng = hb.Engine(dev, na, nl, ng, row_begin=r0, row_end=r1)
    eng.set_arith(args.arith)
    multi = P > 1 or args.force_comm
    if multi:
        # N > 1: NCCL sum of the packed partials; --force-comm exercises the same path on one
        # GPU with a 1-rank communicator (plumbing check)
        uid = d.bcast_bytes(hb.nccl_unique_id() if d.rank == 0 else None)
        eng.set_comm(uid, P, d.rank)
        eng.set_reduce_mode(args.reduce)
    eng.upload(p, 0)
    eng.sync()
    stream = torch.cuda.ExternalStream(eng.stream(), device=dev)

    def step():
        eng.build(args.algo)
        eng.reduce(0)

    for _ in range(args.warmup):
        step()
    st_w = eng.sync()
    launches_per_step = st_w["kernel_launches"]
    eng.kernel_times(reset=True)

    # ---- timed region (device-resident inputs) ----
    sampler = ClockSampler(dev)
    d.barrier()
    torch.cuda.synchronize(dev)
    eng.sync()
    sampler.start()
    time.sleep(0.3)  # let the sampler attach before the timed work
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    eng.sync()
    torch.cuda.synchronize(dev)
    d.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms = d.max(ms)
    kt = eng.kernel_times(reset=True)
    st = eng.sync()
    F = ledger_flops(na_total, nl, ng, "original" if args.algo == "original" else "refined")
    value = F / (ms * 1e-3) / 1e12
    exec_tf = executed_flops(na_total, nl, ng, args.arith, args.algo) / (ms * 1e-3) / 1e12

    # the same device-resident build with the plain 4-multiplication arithmetic, for reference
    ms4 = None
    if args.arith == "3m" and not args.no_4m:
        eng.set_arith("4m")
        for _ in range(2):
            step()
        eng.sync()
        d.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
        eng.sync()
        d.barrier()
        ms4 = d.max(ev0.elapsed_time(ev1) / args.steps)
        eng.set_arith("3m")

    # the kernel layer first: host-buffer (un)registration by the e2e legs below leaves the
    # host's page state noisy for a while, which this pageable-input path is sensitive to
    # side legs (kernel layer, HSDL file) only where their host copies stay small
    small = 2 * na * nl * ng * 16 <= (4 << 30)
    klayer = None
    if P == 1 and not args.no_e2e and small:
        klayer = run_kernel_layer(hb, p, nl, ng)

    # ---- e2e through the public API with host buffers ----
    e2e = e2e_pinned = None
    if not args.no_e2e:
        e2e = run_e2e(args, hb, d, p, eng, na_total, nl, ng, pinned=False)
        if P == 1:
            e2e_pinned = run_e2e(args, hb, d, p, eng, na_total, nl, ng, pinned=True)

    lapw = file_leg = kpoints = None
    if P == 1 and not args.no_e2e:
        lapw = run_lapw(args, hb, p, na, nl, ng)
        file_leg = run_file(args, hb, p, na, nl, ng) if small else None
        kpoints = run_kpoints(args, hb, p, na, nl, ng) if small and args.algo != "original" else None

    peak = hb.fp64_peak(dev, 1.0)
    line = None
    if d.rank == 0:
        xf = 0.75 if args.arith == "3m" else 1.0  # executed / ledger flops of a contraction
        h_led = kt["h_flops"] / (kt["h_ms"] * 1e-3) / 1e12
        h_tf = h_led * xf
        traffic = load_traffic(args.config) if P == 1 else None
        roofline = {"bound": "tensor", "achieved": h_tf, "peak": peak, "unit": "TFLOP/s", "frac": h_tf / peak,
                    "traffic": traffic,
                    "kernel": f"ctn_contract_kernel<TRI> {H_KERNEL.get(args.algo, 'H contraction')} (the strictly-lower "
                              "tile launch + the diagonal-tile launch, timed together): "
                              f"{round(kt['h_flops'] / (na * nl * ng * ng))} K N_G^2 "
                              f"flops per contraction at 8 per complex MAC, {'6 per MAC executed (3M)' if xf < 1 else 'all executed (4M)'}; "
                              "achieved = executed flops / mean contraction time (rank 0)",
                    "achieved_ledger": h_led, "arith": args.arith,
                    "kernel_ms": kt["h_ms"], "flops_per_launch": int(kt["h_flops"] * xf),
                    "ledger_flops_per_launch": kt["h_flops"],
                    "s_kernel_tflops": kt["s_flops"] * xf / (kt["s_ms"] * 1e-3) / 1e12,
                    "peak_source": "FP64 DMMA m8n8k4 loop measured in-process after the timed region "
                                   "(MEASURED_PEAKS.json has no FP64 entry)"}
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": P, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling if P > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_problem seed 1, bit-identical to the reference generator; each rank "
                    "generates the atoms of its K-row shard)",
            "config": {"workload": f"{args.config}: {desc}", "n_atoms": na_total, "n_atoms_per_gpu": na_total / P,
                       "n_l": nl, "n_g": ng, "algo": args.algo,
                       "arith": args.arith + (" (Gauss 3-multiplication complex products: 6 executed real "
                                              "flops per complex MAC, all FP64; value counts the reference "
                                              "ledger's 8)" if args.arith == "3m" else " (4 real DMMAs per "
                                              "complex MAC)"),
                       "parallelism": f"K-row-sharded x{P}" + (f" + NCCL {'reduce-scatter' if args.reduce == 'scatter' else 'reduce'}"
                                                              f" of packed H,S (timed)" if multi else ""),
                       "l2": f"inputs A,B {2 * na * nl * ng * 16 / 1e6:.0f} MB per GPU > 126 MB L2 (no flush)"},
            "build_ms": ms,
            "fp64_frac_of_peak": exec_tf / (P * peak),
            "executed_tflops": exec_tf,
            "phase_ms": {k: v * 1e3 for k, v in st["phase_seconds"].items()},
            "reduce_ms": st["reduce_seconds"] * 1e3,
            "roofline": roofline,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        if ms4 is not None:
            line["value_4m"] = F / (ms4 * 1e-3) / 1e12
            line["ms_per_step_4m"] = ms4
        if e2e is not None:
            line["e2e"] = e2e
        if e2e_pinned is not None:
            line["e2e_pinned"] = e2e_pinned
        if lapw is not None:
            line.update(lapw)
        if file_leg is not None:
            line["e2e_file"] = file_leg
        if kpoints is not None:
            line["e2e_kpoints"] = kpoints
        if klayer is not None:
            line["kernel_layer"] = klayer
        if P == 1 and not args.no_cpu_baseline:
            try:
                cb = cpu_reference_sample(na, nl, ng, args.cpu_budget)
                line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            except Exception as ex:  # noqa: BLE001 - reported, never silently replaced
                line["cpu_baseline"] = {"value": None, "error": str(ex)}
        print(json.dumps(line), flush=True)
    eng.close()
    d.close()
    return 0


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s"


def run_lapw(args, hb, p, na, nl, ng):
    """North_star subsystem 1 on the same workload shape: the LAPW matching-coefficient
    setup kernel (HBM-write bound) and the physics-input end-to-end path, where only
    G vectors, atom data, radial values and T operators go host->device and A, B are
    built in HBM (no reference equivalent: the reference takes A, B as inputs)."""
    import torch
    lmax = int(round(nl ** 0.5)) - 1
    if (lmax + 1) ** 2 != nl:
        return None
    s = hb.make_lapw_system(na, lmax, ng, n_types=2, seed=1)
    eng = hb.Engine(torch.cuda.current_device(), na, nl, ng)
    H = np.zeros((ng, ng), np.complex128, order="F")
    S = np.zeros((ng, ng), np.complex128, order="F")
    ops = [p.T_AA, p.T_AB, p.T_BB, H, S]
    for b in ops:
        hb.host_register(b)
    try:
        times, stimes = [], []
        for _ in range(5):
            eng.setup_lapw(s)
            eng.sync()
            t_ = eng.setup_time()
            times.append(t_["ms"])
            stimes.append(t_["stream_ms"])
        nbytes = eng.setup_time()["bytes"]
        ms = float(np.median(times))
        sms = float(np.median(stimes))
        peak, src = hbm_peak()

        def one():
            eng.setup_lapw(s)
            eng.upload_operators(p.T_AA, p.T_AB, p.T_BB)
            eng.build(args.algo)
            eng.download(H, S)

        eng.set_download_overlap(True)  # the download overlaps the build's final H bands
        one()
        eng.sync()
        steps = max(1, min(args.steps, args.e2e_steps))
        t = time.perf_counter()
        for _ in range(steps):
            one()
        eng.sync()
        dt = (time.perf_counter() - t) / steps
    finally:
        for b in ops:
            hb.host_unregister(b)
        eng.close()
    h2d = s.gvec.nbytes + s.tau.nbytes + 6 * s.u.nbytes + 3 * p.T_AA.nbytes
    return {
        "setup_roofline": {"bound": "hbm", "achieved": nbytes / (sms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                           "frac": nbytes / (sms * 1e-3) / 1e9 / peak,
                           "traffic": load_traffic(args.config, "setup_stream_dram_bytes_per_launch"),
                           "kernel": "lapw_stream_kernel (the HBM-write pass: A, B = 2 x K x N_G x 16 B per launch)",
                           "bytes_per_launch": int(nbytes), "kernel_ms": sms, "peak_source": src,
                           "setup_ms_total": ms, "setup_gbs_total": nbytes / (ms * 1e-3) / 1e9,
                           # north_star quotes the setup against the 8 TB/s HBM3e spec
                           "frac_of_spec_8000": nbytes / (sms * 1e-3) / 1e9 / 8000.0,
                           "note": "setup = lapw_tables_kernel (latency-bound per-G tables) + lapw_stream_kernel"},
        "e2e_lapw": {"value": ledger_flops(na, nl, ng) / dt / 1e12, "unit": "TFLOP/s", "ms_per_step": dt * 1e3,
                     "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(2 * (ng * (ng + 1) // 2) * 16),
                     "api": "engine_setup_lapw + engine_upload_operators + engine_build + engine_download (C-ABI, download "
                            "overlap on); "
                            "A, B built in HBM from G vectors / atoms / radial data"},
    }


def run_file(args, hb, p, na, nl, ng):
    """Row f2 (HSDL v1 problem files): the problem written in the reference's file format
    to local disk, then build_hs_file -> hsdla_b200_build_hs_file, which streams the file
    into HBM (pread -> pinned double buffer -> H2D) and builds.  Timed per call with the
    file in the page cache (a warm re-read, as a k-point loop over one file would see)."""
    import tempfile
    H = np.zeros((ng, ng), np.complex128, order="F")
    S = np.zeros((ng, ng), np.complex128, order="F")
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "problem.hsdl")
        hb.save_problem(p, path)
        fbytes = os.path.getsize(path)
        cfg = hb.PipelineConfig(algo=args.algo if args.algo != "original" else "merged", arith=args.arith)
        hb.build_hs_file(path, cfg, H=H, S=S)  # warm: engine cache + page cache
        steps = max(1, min(args.steps, 5))
        t = time.perf_counter()
        loads = []
        for _ in range(steps):
            r = hb.build_hs_file(path, cfg, H=H, S=S)
            loads.append(r.stats["h2d_seconds"])
        dt = (time.perf_counter() - t) / steps
        hb.release_cache()
    load = float(np.median(loads))
    return {"value": ledger_flops(na, nl, ng) / dt / 1e12, "unit": "TFLOP/s", "ms_per_step": dt * 1e3,
            "file_bytes": int(fbytes), "load_ms": load * 1e3, "load_gbs": fbytes / load / 1e9,
            "api": "paper_1712_07206_b200.build_hs_file -> hsdla_b200_build_hs_file (C-ABI)"}


def run_kpoints(args, hb, p, na, nl, ng, nk=8):
    """The k-point batch extension (hsdla_b200_build_hs_kpoints): nk k-points of the cell
    sharing T and U, plain (pageable) numpy coefficients, every k-point's H, S downloaded.
    Informational beside `e2e` (the per-call drop-in, the contract's number)."""
    As = [p.A] + [hb.generate_problem(na, nl, ng, 100 + k, 0).A for k in range(nk - 1)]
    Bs = [p.B] + [hb.generate_problem(na, nl, ng, 100 + k, 0).B for k in range(nk - 1)]
    Hs = [np.zeros((ng, ng), np.complex128, order="F") for _ in range(nk)]
    Ss = [np.zeros((ng, ng), np.complex128, order="F") for _ in range(nk)]
    cfg = hb.PipelineConfig(algo=args.algo, arith=args.arith)
    hb.build_hs_kpoints(p, As, Bs, cfg, Hs=Hs, Ss=Ss)  # warm
    t = time.perf_counter()
    hb.build_hs_kpoints(p, As, Bs, cfg, Hs=Hs, Ss=Ss)
    dt = (time.perf_counter() - t) / nk
    hb.release_cache()
    return {"value": ledger_flops(na, nl, ng) / dt / 1e12, "unit": "TFLOP/s", "ms_per_kpoint": dt * 1e3,
            "k_points": nk, "inputs": "pageable", "h2d_bytes_per_kpoint": int(p.A.nbytes + p.B.nbytes),
            "d2h_bytes_per_kpoint": int(2 * (ng * (ng + 1) // 2) * 16),
            "api": "paper_1712_07206_b200.build_hs_kpoints -> hsdla_b200_build_hs_kpoints (C-ABI; extension: "
                   "k-independent T, U uploaded once, uploads / downloads overlap the builds)"}


def run_kernel_layer(hb, p, nl, ng):
    """The hsdla::kernels layer through its C-ABI with host buffers (upload, one
    contraction-engine launch, download): herk on the workload's A (K x N_G)."""
    from paper_1712_07206_b200 import kernels as K
    A = p.A
    C = np.zeros((ng, ng), np.complex128, order="F")
    K.herk(1.0, A, 0.0, C)  # warm
    t = time.perf_counter()
    n = 3
    for _ in range(n):
        K.herk(1.0, A, 0.0, C)
    dt = (time.perf_counter() - t) / n
    k = A.shape[0]
    return {"herk": {"value": 4 * k * ng * ng / dt / 1e12, "unit": "TFLOP/s", "ms_per_call": dt * 1e3,
                     "shape": f"A {k} x {ng}", "api": "paper_1712_07206_b200.kernels.herk -> hsdla_b200_herk"}}


def run_e2e(args, hb, d, p, eng, na_total, nl, ng, pinned=False):
    """Same metric through the public API with host buffers: every step copies the inputs
    host->device and reads H, S back (packed-lower D2H + unpack).  N = 1: the drop-in
    build_hs_refined -> hsdla_b200_build_hs; N > 1: per rank the engine API (streamed upload of
    its shard, NCCL reduce, download of the ranges it owns into its host H, S).  pinned=False:
    plain pageable numpy buffers (the reference caller's std::vector reality); True: the
    same buffers page-locked (hsdla_b200_host_register) outside the timed region."""
    import torch
    P = d.world
    steps = max(1, min(args.steps, args.e2e_steps))
    H = np.zeros((ng, ng), np.complex128, order="F")
    S = np.zeros((ng, ng), np.complex128, order="F")
    bufs = [p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U, H, S] if pinned else []
    for b in bufs:
        hb.host_register(b)
    h2d = sum(b.nbytes for b in (p.A, p.B, p.T_AA, p.T_AB, p.T_BB, p.U))
    h2d = int(d.sum(h2d)) if P > 1 else h2d
    d2h = 2 * (ng * (ng + 1) // 2) * 16
    try:
        if P == 1:
            if args.algo == "original":
                cfg = hb.PipelineConfig(variant="original", arith=args.arith)
                call = lambda: hb.build_hs_original(p, cfg, H=H, S=S)  # noqa: E731
            else:
                cfg = hb.PipelineConfig(algo=args.algo, arith=args.arith)
                call = lambda: hb.build_hs_refined(p, cfg, H=H, S=S)  # noqa: E731
            call()  # warm the engine cache
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(steps):
                call()
            dt = (time.perf_counter() - t) / steps
            hb.release_cache()
        else:
            eng.set_download_overlap(True)  # band the final H: each band's reduce + D2H overlaps the next

            def one():
                eng.build_streamed(p, 0, args.algo)
                eng.reduce(0)
                eng.download(H, S)
                eng.sync()
            one()
            d.barrier()
            t = time.perf_counter()
            for _ in range(steps):
                one()
            d.barrier()
            dt = d.max((time.perf_counter() - t) / steps)
            eng.set_download_overlap(False)
    finally:
        for b in bufs:
            hb.host_unregister(b)
    return {"value": ledger_flops(na_total, nl, ng) / dt / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3, "steps": steps,
            "host_buffers": "page-locked" if pinned else "pageable",
            "api": "paper_1712_07206_b200.build_hs_refined -> hsdla_b200_build_hs (C-ABI)" if P == 1
            else f"hsdla_b200_engine_build_streamed / reduce ({args.reduce}) / download (C-ABI), one process per GPU"}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--algo", default="merged", choices=["merged", "fused", "refined", "original"])
    ap.add_argument("--arith", default="3m", choices=["3m", "4m"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = 64 N atoms of c2 (fixed work per GPU); strong = the config's atoms split N ways")
    ap.add_argument("--reduce", default="scatter", choices=["scatter", "root"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-4m", action="store_true", help="skip the 4M re-timing of the device-resident build")
    ap.add_argument("--force-comm", action="store_true", help="NCCL communicator even at N=1 (plumbing check)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU work for cpu_baseline")
    ap.add_argument("--ref-budget", type=float, default=900.0,
                    help="--impl reference: run the full problem when K steps are predicted to fit this many seconds")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus and not (ws == 1 and args.gpus == 1):
        if ws == 1 and args.gpus > 1:
            ap.error("--gpus N>1 must be launched with torchrun --nproc-per-node N")
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
