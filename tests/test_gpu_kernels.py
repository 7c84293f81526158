"""The reference kernel layer (hsdla::kernels, kernels.hpp) on the GPU, pinned like the
reference's tests/test_kernels.cpp: each kernel against a numpy complex128 reference
(<= 1e-13 relative, FP64), NaN-poisoned upper triangles survive (:76-109), beta = 0
never reads C (:111-134), alpha = 0 reduces to a scale of C, bit-exact at beta = 1
(:136-148), hemm reads the lower triangle only (:173-187), trmm both modes (:189-201),
potrf factors / failing pivot (:203-227), diag_scale incl. aliasing (:229-240), ledger
closed forms (:242-274), dimension errors (:276-284)."""
import numpy as np
import pytest

import paper_1712_07206_b200 as hb
from paper_1712_07206_b200 import kernels as K

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    assert hb.device_count() > 0, "GPU tests need a CUDA device"


def rnd(r, c, seed):
    g = np.random.default_rng(seed)
    return np.asfortranarray(g.uniform(-1, 1, (r, c)) + 1j * g.uniform(-1, 1, (r, c)))


def close(x, y, tol=1e-13):
    return np.linalg.norm(x - y) <= tol * max(np.linalg.norm(y), 1e-300)


def lower(x):
    return np.tril(x)


@pytest.mark.parametrize("n,k", [(1, 1), (9, 5), (70, 33), (130, 200)])
def test_herk_her2k_herkx_vs_numpy_and_upper_untouched(n, k):
    a, b = rnd(k, n, 1), rnd(k, n, 2)
    c0 = rnd(n, n, 3)
    c0 = np.asfortranarray(c0 + c0.conj().T)  # Hermitian start so beta * C keeps diag real-ish
    iu = np.triu_indices(n, 1)
    for beta in (0.0, 0.5):
        c = c0.copy(order="F")
        c[iu] = np.nan
        K.herk(1.5, a, beta, c)
        want = lower(1.5 * a.conj().T @ a + beta * c0)
        np.fill_diagonal(want, want.diagonal().real + 1j * (beta * c0.diagonal().imag))
        assert close(lower(np.nan_to_num(c)), want) and np.all(np.isnan(c[iu]))
        alpha = 0.7 - 0.3j
        c = c0.copy(order="F")
        c[iu] = np.nan
        K.her2k(alpha, a, b, beta, c)
        full = alpha * a.conj().T @ b + np.conj(alpha) * b.conj().T @ a
        want = lower(full + beta * c0)
        np.fill_diagonal(want, full.diagonal().real + beta * c0.diagonal())
        assert close(lower(np.nan_to_num(c)), want) and np.all(np.isnan(c[iu]))
        c = c0.copy(order="F")
        c[iu] = np.nan
        K.herkx(alpha, a, b, beta, c)
        full = alpha * a.conj().T @ b
        want = lower(full + beta * c0)
        np.fill_diagonal(want, full.diagonal().real + beta * c0.diagonal())
        assert close(lower(np.nan_to_num(c)), want) and np.all(np.isnan(c[iu]))


@pytest.mark.parametrize("ta", [K.NONE, K.CONJ_TRANS])
@pytest.mark.parametrize("tb", [K.NONE, K.CONJ_TRANS])
def test_gemm_all_transpose_combinations(ta, tb):
    m, n, k = 37, 150, 19
    a = rnd(m, k, 4) if ta == K.NONE else rnd(k, m, 4)
    b = rnd(k, n, 5) if tb == K.NONE else rnd(n, k, 5)
    oa = a if ta == K.NONE else a.conj().T
    ob = b if tb == K.NONE else b.conj().T
    c0 = rnd(m, n, 6)
    for alpha, beta in ((1.0, 0.0), (0.5 + 2j, -1 + 0.25j)):
        c = c0.copy(order="F")
        K.gemm(alpha, a, ta, b, tb, beta, c)
        assert close(c, alpha * oa @ ob + beta * c0)


def test_beta_zero_never_reads_destination():
    n, k = 9, 5
    a, b = rnd(k, n, 1), rnd(k, n, 2)
    c = np.full((n, n), np.nan + 1j * np.nan, order="F")
    K.gemm(1.0, a, K.CONJ_TRANS, b, K.NONE, 0.0, c)
    assert np.all(np.isfinite(c))
    for f in (lambda h: K.herk(1.0, a, 0.0, h), lambda h: K.her2k(1.0, a, b, 0.0, h)):
        h = np.full((n, n), np.nan + 1j * np.nan, order="F")
        f(h)
        assert np.all(np.isfinite(h[np.tril_indices(n)]))


def test_alpha_zero_scales_c_bit_exact():
    n, k = 6, 4
    a = rnd(k, n, 1)
    c = rnd(n, n, 2)
    before = c.copy()
    K.gemm(0.0, a, K.CONJ_TRANS, a, K.NONE, 1.0, c)
    assert np.array_equal(c, before)
    h = before.copy(order="F")
    K.herk(0.0, a, 1.0, h)
    assert np.array_equal(np.tril(h), np.tril(before)) and np.array_equal(np.triu(h, 1), np.triu(before, 1))
    h = before.copy(order="F")
    K.herk(0.0, a, 0.0, h)
    assert np.all(np.tril(h) == 0) and np.array_equal(np.triu(h, 1), np.triu(before, 1))


def test_hemm_reads_lower_only():
    n, m = 21, 40
    hl = rnd(n, n, 7)
    full = np.tril(hl) + np.tril(hl, -1).conj().T
    np.fill_diagonal(full, full.diagonal())
    b, c0 = rnd(n, m, 8), rnd(n, m, 9)
    h = hl.copy(order="F")
    h[np.triu_indices(n, 1)] = np.nan
    c = c0.copy(order="F")
    K.hemm(K.LEFT, 0.5 - 1j, h, b, 2.0, c)
    assert close(c, (0.5 - 1j) * full @ b + 2.0 * c0)


@pytest.mark.parametrize("n", [1, 3, 9, 81])
def test_trmm_both_modes(n):
    m = 6
    t = rnd(n, n, 8)
    lt = np.tril(t)
    for tr in (K.NONE, K.CONJ_TRANS):
        b = rnd(n, m, 9)
        want = (2 + 1j) * ((lt if tr == K.NONE else lt.conj().T) @ b)
        K.trmm(K.LEFT, tr, 2 + 1j, t, b)
        assert close(b, want, 1e-12 * n)


def test_potrf_factor_and_failing_pivot():
    g = rnd(6, 6, 12)
    h = np.asfortranarray(g.conj().T @ g + 6 * np.eye(6))
    r = K.potrf(h)
    assert r.ok()
    c = r.factor
    assert close(np.tril(c @ c.conj().T), np.tril(h), 1e-12)
    assert np.all(c[np.triu_indices(6, 1)] == 0)
    bad = np.zeros((3, 3), np.complex128, order="F")
    bad[0, 0], bad[1, 1], bad[2, 2] = 4.0, -1.0, 1.0  # negative pivot at index 1
    f = K.potrf(bad)
    assert not f.ok() and f.pivot == 1


def test_diag_scale_and_aliasing():
    b = rnd(3, 4, 5)
    orig = b.copy()
    u = np.array([2.0, -1.0, 0.5])
    x = K.diag_scale(u, b)
    assert np.array_equal(x, u[:, None] * orig)
    K.diag_scale(u, b, b)  # in place
    assert np.array_equal(b, x)


def test_ledger_closed_forms():
    led = hb.FlopLedger()
    a, b = rnd(5, 3, 1), rnd(5, 3, 2)
    c = np.zeros((3, 3), np.complex128, order="F")
    K.gemm(1.0, a, K.CONJ_TRANS, b, K.NONE, 0.0, c, led)
    assert led.count("gemm") == 8 * 3 * 3 * 5
    K.herk(1.0, a, 0.0, c, led)
    assert led.count("herk") == 4 * 5 * 3 * 3
    K.her2k(1.0, a, b, 0.0, c, led)
    assert led.count("her2k") == 8 * 5 * 3 * 3
    K.herkx(1.0, a, b, 0.0, c, led)
    assert led.count("herkx") == 4 * 5 * 3 * 3
    g = rnd(3, 3, 3)
    hm = np.asfortranarray(g.conj().T @ g + 3 * np.eye(3))
    bm = rnd(3, 7, 4)
    K.hemm(K.LEFT, 1.0, hm, bm, 0.0, np.zeros((3, 7), np.complex128, order="F"), led)
    assert led.count("hemm") == 8 * 3 * 3 * 7
    K.trmm(K.LEFT, K.CONJ_TRANS, 1.0, hm, bm, led)
    assert led.count("trmm") == 4 * 3 * 3 * 7
    K.potrf(hm, led)
    assert led.count("potrf") == 4 * 27 // 3
    K.diag_scale(np.array([1.0, 2.0, 3.0]), bm, None, led)
    assert led.count("scaling") == 2 * 3 * 7
    z = hb.FlopLedger()
    K.herk(0.0, a, 1.0, c, z)  # alpha = 0 still charges the full closed form
    assert z.count("herk") == 4 * 5 * 3 * 3


def test_dimension_errors():
    a, b, c = rnd(2, 3, 1), rnd(4, 5, 2), np.zeros((2, 5), np.complex128, order="F")
    with pytest.raises(hb.DimensionError):
        K.gemm(1.0, a, K.NONE, b, K.NONE, 0.0, c)
    with pytest.raises(hb.DimensionError):
        K.herk(1.0, rnd(3, 5, 1), 0.0, np.zeros((4, 4), np.complex128, order="F"))
