import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "case_*.npz")))


def load_case(path):
    """Golden fixture -> (problem-like namespace, dict of arrays)."""
    z = np.load(path)
    d = {k: z[k] for k in z.files}
    na, nl, ng, seed, nnh = (int(x) for x in d["dims"])
    return (na, nl, ng, seed, nnh), d


def as_problem(d, dims):
    import paper_1712_07206_b200 as hb
    na, nl, ng = dims[:3]
    f = np.asfortranarray
    return hb.ProblemInstance(na, nl, ng, f(d["A"]), f(d["B"]), f(d["T_AA"]), f(d["T_AB"]), f(d["T_BB"]), f(d["U"]),
                              d["hpd"].astype(bool))


def gpu_available():
    try:
        import paper_1712_07206_b200 as hb
        return hb.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def restatement():
    from oracle.oracle import Restatement
    return Restatement()
