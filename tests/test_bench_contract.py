"""bench.py's one-JSON-line contract (the driver parses it): the reference arm on CPU
(oracle/_ref, no GPU needed) and the B200 arm on a GPU, on the small C1 workload."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libhsdla_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3"], 600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "TFLOP/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_warmup_floor_enforced():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--warmup", "1"], capture_output=True,
                       text=True, timeout=120, cwd=ROOT)
    assert r.returncode != 0 and "--warmup must be >= 3" in r.stderr


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "2"], 900)
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 1.0 and d["dtype"] == "f64" and d["scaling"] == "weak"
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and 0 < rf["frac"] <= 1.05 and rf["unit"] == "TFLOP/s"
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["host_buffers"] == "pageable" and d["e2e_pinned"]["host_buffers"] == "page-locked"
    # every "fraction of peak" is an executed-flop efficiency (<= 1); the ledger rate is `value`
    assert 0 < d["fp64_frac_of_peak"] <= 1.0 and "ledger_frac_of_peak" not in d
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert d["setup_roofline"]["bound"] == "hbm" and d["e2e_file"]["value"] > 0


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libhsdla_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_under_torchrun_world_2():
    """The driver launches the reference arm like its own at N > 1: rank 0 alone times the
    reference and prints the one JSON line; the other rank exits 0 without work (gloo, CPU)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.gpu
def test_b200_arm_under_torchrun_with_nccl_plumbing():
    """bench.py as the driver launches it for N > 1 (torchrun, env rendezvous), here with one
    rank and --force-comm: the NCCL reduce path (comm stream, banded H reduce) in the timed
    region and the multi-rank e2e leg (build_streamed + reduce + rank-0 download)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "1", "--config", "c1", "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
                        "--force-comm", "--e2e-steps", "2"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 1.0 and d["e2e"]["value"] > 0
    assert "reduce-scatter" in d["config"]["parallelism"]
