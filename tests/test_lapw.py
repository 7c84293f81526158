"""LAPW matching-coefficient setup (north_star subsystem 1).

NO REFERENCE IMPLEMENTATION exists: parity is SELF-PINNED.
The CPU oracle (oracle/hsdla_oracle.c:orc_lapw_coefficients, different Y_lm / j_l
algorithms than the GPU) is pinned against scipy.special.sph_harm_y / spherical_jn
and against the matching conditions it must satisfy; the GPU kernel is checked
against that oracle and against the plane-wave (Rayleigh) reconstruction at the
muffin-tin sphere.
"""
import numpy as np
import pytest
import scipy.special as sps

import paper_1712_07206_b200 as hb


def _angles(K):
    kx, ky, kz = K
    kn = np.sqrt(kx * kx + ky * ky + kz * kz)
    return (np.arccos(kz / kn) if kn > 0 else 0.0), (np.arctan2(ky, kx) if kx or ky else 0.0), kn


DIRS = [(0.3, -1.2, 0.7), (0, 0, 1.5), (0, 0, -2.0), (1e-9, 0, 0), (2.5, 1.0, -0.2), (-0.4, -0.4, 0.01),
        (0.0, 0.0, 0.0)]


@pytest.mark.parametrize("K", DIRS)
def test_oracle_ylm_vs_scipy(restatement, K):
    lmax = 12
    th, ph, kn = _angles(K)
    Y = restatement.ylm(lmax, K)
    ref = np.array([sps.sph_harm_y(l, m, th, ph) for l in range(lmax + 1) for m in range(-l, l + 1)])
    assert np.max(np.abs(Y - ref)) < 1e-13


@pytest.mark.parametrize("x", [0.0, 1e-7, 1e-3, 0.3, 0.999, 1.0, 2.5, 7.3, 11.0, 13.5, 25.0, 60.0])
def test_oracle_sph_bessel_vs_scipy(restatement, x):
    lmax = 13
    j = restatement.sph_bessel(lmax, x)
    ref = sps.spherical_jn(np.arange(lmax + 1), x)
    scale = np.maximum(np.abs(ref), 1e-300)
    big = np.abs(ref) > 1e-200
    assert np.all(np.abs(j - ref)[big] / scale[big] < 1e-12)


@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("d", [-1e-6, -1e-9, 0.0, 1e-9, 1e-6])
def test_oracle_sph_bessel_next_to_zeros_of_j0(restatement, n, d):
    """x = n pi + d: j_0 vanishes there, so a downward recurrence normalised by j_0 alone loses
    every digit (3e-4 relative at 2 pi + 1e-12); normalising by the larger of |j_0|, |j_1| keeps
    the 1e-12 bar (the GPU kernel uses the same normalisation, lapw_setup.cuh)."""
    x = n * np.pi + d
    j = restatement.sph_bessel(13, x)
    ref = sps.spherical_jn(np.arange(14), x)
    big = np.abs(ref) > 1e-200
    # j_0 itself is ~|d| / x next to its zero: compare it absolutely
    assert abs(j[0] - ref[0]) <= 1e-15
    assert np.all(np.abs(j - ref)[1:][big[1:]] / np.abs(ref[1:][big[1:]]) < 1e-12)


def _matching_residual(s, A, B, a, lm, g):
    """|A u + B udot - c j_l(KR)| and |A u' + B udot' - c K j_l'(KR)| with scipy values."""
    l = int(np.floor(np.sqrt(lm)))
    m = lm - l * (l + 1)
    K = s.kpt + s.gvec[g]
    th, ph, kn = _angles(K)
    t = s.atom_type[a]
    R = s.rmt[t]
    c = 4 * np.pi / np.sqrt(s.omega) * np.exp(1j * K @ s.tau[a]) * (1j ** l) * np.conj(sps.sph_harm_y(l, m, th, ph))
    j = sps.spherical_jn(l, kn * R)
    jd = kn * sps.spherical_jn(l, kn * R, derivative=True)
    row = a * s.n_l + lm
    r1 = A[row, g] * s.u[t, l] + B[row, g] * s.udot[t, l] - c * j
    r2 = A[row, g] * s.du[t, l] + B[row, g] * s.dudot[t, l] - c * jd
    return abs(r1), abs(r2), abs(c)


def test_oracle_satisfies_matching_conditions(restatement):
    s = hb.make_lapw_system(5, 8, 60, n_types=3, seed=4)
    A, B, U = restatement.lapw_coefficients(s)
    rng = np.random.default_rng(0)
    for _ in range(200):
        a, lm, g = rng.integers(s.n_atoms), rng.integers(s.n_l), rng.integers(s.n_g)
        r1, r2, c = _matching_residual(s, A, B, a, lm, g)
        assert r1 <= 1e-13 * max(c, 1e-3) + 1e-15 and r2 <= 1e-13 * max(c, 1e-3) + 1e-15
    l_of = np.floor(np.sqrt(np.arange(s.n_l))).astype(int)
    assert np.array_equal(U, s.udot_norm[s.atom_type][:, l_of].T)


def test_synthetic_system_generator():
    s = hb.make_lapw_system(9, 6, 250, n_types=2, seed=3)
    kn = np.linalg.norm(s.gvec + s.kpt, axis=1)
    assert s.n_g == 250 and np.all(np.diff(kn) >= -1e-12)
    det = s.u * s.dudot - s.udot * s.du
    assert np.allclose(det * s.rmt[:, None] ** 2, -1.0)
    assert s.n_l == 49 and s.tau.shape == (9, 3)


def test_lapw_dimension_errors():
    s = hb.make_lapw_system(2, 3, 10)
    s.atom_type = np.array([0, 7], np.int32)
    with pytest.raises((hb.DimensionError, hb.ConfigError)):
        hb.lapw_coefficients(s)


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(1, 0, 1, 1), (3, 6, 64, 2), (7, 10, 300, 3), (16, 8, 1000, 2)])
def test_gpu_coefficients_vs_oracle(restatement, dims):
    na, lmax, ng, nt = dims
    s = hb.make_lapw_system(na, lmax, ng, n_types=nt, seed=na + lmax)
    A, B, U = hb.lapw_coefficients(s)
    Ar, Br, Ur = restatement.lapw_coefficients(s)
    rel = lambda x, y: np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)
    assert rel(A, Ar) <= 1e-13 and rel(B, Br) <= 1e-13
    assert np.array_equal(U, Ur)


@pytest.mark.gpu
def test_gpu_coefficients_next_to_zeros_of_j0(restatement):
    """Muffin-tin radii set so that |k+G| R_mt = pi + 1e-9 and 2 pi - 1e-9 for two G vectors (the
    zeros of j_0, where the j_l recurrence needs the j_0 / j_1 normalisation): the GPU coefficients
    equal the oracle's and satisfy the matching conditions with scipy's j_l there."""
    s = hb.make_lapw_system(4, 8, 80, n_types=2, seed=7)
    kn = np.linalg.norm(s.kpt + s.gvec, axis=1)
    g1, g2 = 5, 41
    s.rmt = np.array([(np.pi + 1e-9) / kn[g1], (2 * np.pi - 1e-9) / kn[g2]])
    A, B, U = hb.lapw_coefficients(s)
    Ar, Br, Ur = restatement.lapw_coefficients(s)
    rel = lambda x, y: np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)
    assert rel(A, Ar) <= 1e-13 and rel(B, Br) <= 1e-13
    for g, t in ((g1, 0), (g2, 1)):
        for a in range(s.n_atoms):
            if s.atom_type[a] != t:
                continue
            for lm in range(s.n_l):
                r1, r2, c = _matching_residual(s, A, B, a, lm, g)
                assert r1 <= 1e-12 * max(c, 1e-3) + 1e-15 and r2 <= 1e-12 * max(c, 1e-3) + 1e-15, (g, a, lm)


@pytest.mark.gpu
def test_gpu_plane_wave_reconstruction():
    """Sum_lm (A u_l + B udot_l) Y_lm(r^) at |r_a| = R reproduces Omega^-1/2 e^{iK.(tau+R r^)}
    (Rayleigh expansion truncated at lmax = 14; only G with |K| R <= 2.5, where the
    truncation error is < 1e-10)."""
    s = hb.make_lapw_system(2, 14, 40, n_types=2, seed=2)
    A, B, _ = hb.lapw_coefficients(s)
    rng = np.random.default_rng(1)
    kn = np.linalg.norm(s.gvec + s.kpt, axis=1)
    checked = 0
    for _ in range(200):
        a, g = rng.integers(s.n_atoms), rng.integers(s.n_g)
        t = s.atom_type[a]
        if kn[g] * s.rmt[t] > 2.5:
            continue
        checked += 1
        th, ph = np.arccos(rng.uniform(-1, 1)), rng.uniform(0, 2 * np.pi)
        rhat = np.array([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)])
        val = 0j
        for l in range(s.lmax + 1):
            for m in range(-l, l + 1):
                row = a * s.n_l + l * (l + 1) + m
                val += (A[row, g] * s.u[t, l] + B[row, g] * s.udot[t, l]) * sps.sph_harm_y(l, m, th, ph)
        K = s.kpt + s.gvec[g]
        want = np.exp(1j * K @ (s.tau[a] + s.rmt[t] * rhat)) / np.sqrt(s.omega)
        assert abs(val - want) < 1e-9 * abs(want)
    assert checked >= 10


@pytest.mark.gpu
def test_build_hs_lapw_matches_oracle_path(restatement):
    """Full physics path: GPU setup + GPU build == CPU oracle setup + CPU oracle build."""
    na, lmax, ng = 6, 6, 200
    s = hb.make_lapw_system(na, lmax, ng, n_types=2, seed=5)
    q = hb.generate_problem(na, s.n_l, ng, 9, 0)  # T operators from the reference generator
    r = hb.build_hs_lapw(s, q.T_AA, q.T_AB, q.T_BB)
    A, B, U = restatement.lapw_coefficients(s)
    p = hb.ProblemInstance(na, s.n_l, ng, A, B, q.T_AA, q.T_AB, q.T_BB, U)
    H, S, _ = restatement.build_hs_refined(p)
    assert hb.rel_frobenius_error_lower(r.H, H) <= 1e-11
    assert hb.rel_frobenius_error_lower(r.S, S) <= 1e-11
    assert r.ledger == hb.flop_model(p)
