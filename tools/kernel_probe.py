"""Kernel-layer (hsdla::kernels on the GPU) host-buffer timing (development helper)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1712_07206_b200 as hb  # noqa: E402
from paper_1712_07206_b200 import kernels as K  # noqa: E402

p = hb.generate_problem(64, 81, 3000, 1, 0)
A, B = p.A, p.B
k, n = A.shape
C = np.zeros((n, n), np.complex128, order="F")
G = np.zeros((n, n), np.complex128, order="F")
for name, fn, fl in (("herk", lambda: K.herk(1.0, A, 0.0, C), 4 * k * n * n),
                     ("her2k", lambda: K.her2k(1.0, A, B, 0.0, C), 8 * k * n * n),
                     ("gemm", lambda: K.gemm(1.0, A, K.CONJ_TRANS, B, K.NONE, 0.0, G), 8 * k * n * n)):
    fn()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {dt*1e3:.1f} ms per call, {fl/dt/1e12:.2f} TF/s (host buffers)", flush=True)
