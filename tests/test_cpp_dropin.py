"""The C++ drop-in (include/hsdla_b200/pipeline.hpp) driven through the reference's
own C++ types against the reference's own CPU pipeline (oracle/_ref/parity_cpp,
built from the reference sources by oracle/Makefile)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "parity_cpp")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/parity_cpp not built")


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(2, 3, 16, 1, 0), (8, 5, 128, 99, 4), (16, 49, 1000, 1, 0), (5, 121, 700, 3, 2)])
def test_cpp_dropin_matches_reference_cpu(dims):
    r = subprocess.run([BIN, *map(str, dims), str(os.cpu_count() or 1)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


def test_cpp_dropin_no_gpu_is_config_error():
    from paper_1712_07206_b200 import device_count
    if device_count() > 0:
        pytest.skip("GPU present")
    r = subprocess.run([BIN, "2", "3", "16", "1", "0"], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0 and "ConfigError" in r.stderr
