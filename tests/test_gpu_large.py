"""Parity at BASELINE.md §3's measurement sizes, against the UNMODIFIED reference (oracle/_ref,
Strategy::Cpu BlockedParallel on every host core), plus 3M-arithmetic stress cases.

* Config 3 (108 atoms, N_L 121, N_G 6000) in FULL: the whole lower triangle of H and S.
* Configs 4 (512, 121, 13000) and 5-hi (1024, 81, 20000) by principal-submatrix sampling
  with |J| = 2048 random G-vectors: H[J,J], S[J,J] depend only on the columns J
  of A and B, so the reference's build_hs_refined on the J-sliced problem yields them
  exactly.  The GPU side is the public drop-in on the FULL problem (26 / 53 GB of pageable
  inputs through the host-buffer path).
The reference run (minutes on the host cores) overlaps the GPU work: ctypes releases the GIL.

Bar (north_star): relative Frobenius error of the lower triangle <= 1e-11
(rel_frobenius_error_lower, complex_matrix.cpp:106-118; tests/test_pipeline.cpp:30-52,
acceptance.cpp:58-136 for the reference's own bar)."""
import os
import threading

import numpy as np
import pytest

import paper_1712_07206_b200 as hb

pytestmark = pytest.mark.gpu
TOL = 1e-11


def rel(x, y):
    return hb.rel_frobenius_error_lower(x, y)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    assert hb.device_count() > 0, "GPU tests need a CUDA device"
    yield
    hb.release_cache()


def _reference():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    return Reference()


class _Bg(threading.Thread):
    """Run the reference build on a worker thread (the GIL is released inside the C call)."""

    def __init__(self, fn):
        super().__init__(daemon=True)
        self.fn, self.out, self.err = fn, None, None
        self.start()

    def run(self):
        try:
            self.out = self.fn()
        except Exception as ex:  # noqa: BLE001 - re-raised in result()
            self.err = ex

    def result(self):
        self.join()
        if self.err is not None:
            raise self.err
        return self.out


@pytest.mark.timeout(1800)
def test_config3_full_vs_unmodified_reference():
    """Config 3 in full (the whole lower triangle), merged and reference-order algorithms."""
    ref = _reference()
    p = hb.generate_problem(108, 121, 6000, 1, 0)
    bg = _Bg(lambda: ref.build_hs(p, "refined", threads=os.cpu_count() or 1, blocked=True))
    got = {algo: hb.build_hs_refined(p, hb.PipelineConfig(algo=algo)) for algo in ("merged", "refined")}
    out = bg.result()
    for algo, r in got.items():
        assert rel(r.H, out["H"]) <= TOL and rel(r.S, out["S"]) <= TOL, algo
        assert r.ledger == hb.flop_model(p)
    hb.release_cache()


@pytest.mark.timeout(2400)
@pytest.mark.parametrize("dims", [(512, 121, 13000), (1024, 81, 20000)], ids=["config4", "config5hi"])
def test_sampled_2048_vs_unmodified_reference(dims):
    from oracle.oracle import _Problem
    ref = _reference()
    na, nl, ng = dims
    p = hb.generate_problem(na, nl, ng, 1, 0)
    J = np.sort(np.random.default_rng(11).choice(ng, size=2048, replace=False))
    sl = _Problem(na, nl, J.size, np.asfortranarray(p.A[:, J]), np.asfortranarray(p.B[:, J]), p.T_AA, p.T_AB,
                  p.T_BB, p.U, p.hpd_flags.astype(np.uint8))
    bg = _Bg(lambda: ref.build_hs(sl, "refined", threads=os.cpu_count() or 1, blocked=True))
    r = hb.build_hs_refined(p)
    sub = np.ix_(J, J)
    Hs, Ss = np.asfortranarray(r.H[sub]), np.asfortranarray(r.S[sub])
    del r
    hb.release_cache()
    out = bg.result()
    assert rel(Hs, out["H"]) <= TOL and rel(Ss, out["S"]) <= TOL


def _adversarial(kind):
    """Problems that stress Gauss's 3M product (t3 = (a_r - a_i)(b_r + b_i), Im = t3 - t1 + t2):
      scale    real and imaginary parts of A and B a factor 1e6 apart (1e3 / 1e-3), so the
               imaginary part of every product is a small difference of large t3, t1 terms;
      cancel   B = A with T_AB = -(1 - 1e-3)(T_AA + T_BB) / 2 (per atom), so the operator
               blocks cancel to 1e-3 of their size and H is the residual of large terms;
      both     the two at once."""
    p = hb.generate_problem(8, 49, 700, 5, 0)
    if kind in ("scale", "both"):
        for M in (p.A, p.B):
            M[...] = M.real * 1e3 + 1j * M.imag * 1e-3
    if kind in ("cancel", "both"):
        p.B[...] = p.A
        for a in range(p.n_atoms):
            taa = p.T_AA[:, :, a]
            tbb = p.T_BB[:, :, a]
            full = lambda t: np.tril(t) + np.tril(t, -1).conj().T  # noqa: E731 - lower authoritative
            p.T_AB[:, :, a] = -(1.0 - 1e-3) * (full(taa) + full(tbb)) / 2.0
    return p


@pytest.mark.parametrize("kind", ["scale", "cancel", "both"])
def test_3m_adversarial_operands(restatement, kind):
    """3M stays within the bar on operands built to stress it; its error stays within a small
    factor of the 4M (plain product) error.  Each error is against the reference-bit-identical C
    restatement; the imaginary parts are also checked on their own."""
    p = _adversarial(kind)
    H0, S0, _ = restatement.build_hs_refined(p)
    err = {}
    for arith in ("3m", "4m"):
        for algo in ("merged", "refined"):
            r = hb.build_hs_refined(p, hb.PipelineConfig(algo=algo, arith=arith))
            err[(arith, algo)] = (rel(r.H, H0), rel(r.S, S0))
            il = np.tril_indices(p.n_g)
            im_err = np.linalg.norm((r.H - H0)[il].imag) / max(np.linalg.norm(H0[il].imag), 1e-300)
            # 3M's known weak spot: the imaginary part alone, when it is tiny next to the real part,
            # carries the rounding of t3 - t1 (it still meets the bar as part of H)
            assert im_err <= 1e-6, (kind, arith, algo, im_err)
            err[(arith, algo, "im")] = im_err
            assert err[(arith, algo)][0] <= TOL and err[(arith, algo)][1] <= TOL, (kind, arith, algo, err)
    for algo in ("merged", "refined"):
        e3, e4 = err[("3m", algo)][0], err[("4m", algo)][0]
        assert e3 <= max(100.0 * e4, 1e-13), (kind, algo, e3, e4)
    print(f"3M/4M H error ({kind}): " + ", ".join(
        f"{a}: {err[('3m', a)][0]:.2e}/{err[('4m', a)][0]:.2e} (imag {err[('3m', a, 'im')]:.2e}/"
        f"{err[('4m', a, 'im')]:.2e})" for a in ("merged", "refined")))
