"""The CPU oracle (oracle/hsdla_oracle.c) pinned against the reference.

Golden vectors come from the UNMODIFIED reference library (tests/golden/make_golden.py);
the restatement must reproduce them BIT FOR BIT (it replays the reference's
operation order), and the reference's own known-answer tests:
  hand unit problem H=[[6]], S=[[2]]           test_oracle.cpp:11-47
  flop model at unit dims totals 46            test_pipeline.cpp:75-85
  NaCl her2k = 1,021,490,233,344               test_pipeline.cpp:87-95
  ledger == flop_model, closed-form delta       test_pipeline.cpp:97-113
  grouped == ungrouped (<= 1e-13)              test_oracle.cpp:76-83
  refined vs direct oracle <= 1e-10 sqrt(N_G)  test_pipeline.cpp:42-52
"""
import numpy as np
import pytest

from conftest import GOLDEN as GOLDEN_DIR, golden_cases, load_case
from oracle.oracle import LEDGER_KEYS, Reference, Restatement, alloc_problem


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1][:-4])
def test_restatement_bitwise_vs_reference_golden(path, restatement):
    dims, d = load_case(path)
    na, nl, ng, seed, nnh = dims
    p = restatement.generate_problem(na, nl, ng, seed, nnh)
    for k in ("A", "B", "T_AA", "T_AB", "T_BB", "U"):
        assert np.array_equal(getattr(p, k), d[k]), k
    assert np.array_equal(p.hpd_flags, d["hpd"])
    H, S, led = restatement.build_hs_refined(p)
    assert np.array_equal(H, d["H"]) and np.array_equal(S, d["S"])
    assert [led.get(k, 0) for k in LEDGER_KEYS] + [led["total"]] == d["ledger"].tolist()
    if ng <= 512:
        assert np.array_equal(restatement.direct_H(p), d["Hd"])
        assert np.array_equal(restatement.direct_S(p), d["Sd"])
        tol = 1e-10 * np.sqrt(ng)
        assert restatement.rel_frobenius_error_lower(H, d["Hd"]) < tol
        assert restatement.rel_frobenius_error_lower(S, d["Sd"]) < tol
    if "Hg" in d:
        assert np.array_equal(restatement.direct_H_grouped(p), d["Hg"])
        assert restatement.rel_frobenius_error_lower(d["Hg"], d["Hd"]) < 1e-13
    # the refined pipeline never touches the upper triangles (test_pipeline.cpp:136-147)
    iu = np.triu_indices(ng, 1)
    assert np.all(H[iu] == 0) and np.all(S[iu] == 0)
    assert np.all(np.diag(H).imag == 0) and np.all(np.diag(S).imag == 0)


def test_hand_unit_problem(restatement):
    p = alloc_problem(1, 1, 1)
    p.A[0, 0] = 1.0
    p.B[0, 0] = 1j
    p.T_AA[0, 0, 0] = 2.0
    p.T_AB[0, 0, 0] = 1.0
    p.T_BB[0, 0, 0] = 4.0
    p.U[0, 0] = 1.0
    assert restatement.direct_H(p)[0, 0] == pytest.approx(6.0, abs=1e-14)
    assert restatement.direct_S(p)[0, 0] == pytest.approx(2.0, abs=1e-14)
    H, S, _ = restatement.build_hs_refined(p)
    assert H[0, 0] == pytest.approx(6.0, abs=1e-14) and S[0, 0] == pytest.approx(2.0, abs=1e-14)


def test_flop_model_known_answers(restatement):
    m = restatement.flop_model(1, 1, 1)
    assert m == {"gemm": 8, "hemm": 16, "her2k": 8, "herk": 8, "scaling": 2, "herkx": 4, "total": 46}
    assert restatement.flop_model(512, 49, 2256)["her2k"] == 1021490233344
    # original vs refined closed-form delta (test_pipeline.cpp:97-113)
    for nnh in (0, 2, 4):
        na, nl, ng = 4, 6, 40
        o = restatement.flop_model(na, nl, ng, "original", n_hpd=na - nnh)
        r = restatement.flop_model(na, nl, ng, "refined")
        delta = 4 * nnh * nl * ng * ng + na * (4 * nl ** 3 // 3) - 4 * (na - nnh) * nl * nl * ng
        assert o["total"] - r["total"] == delta


def test_sampled_principal_submatrix(restatement):
    p = restatement.generate_problem(3, 7, 40, 4, 0)
    H, S, _ = restatement.build_hs_refined(p)
    J = np.array([0, 3, 5, 17, 18, 39], np.uint64)
    Hs, Ss = restatement.build_hs_sampled(p, J)
    Ji = J.astype(int)
    il = np.tril_indices(len(J))
    assert np.array_equal(Hs[il], H[np.ix_(Ji, Ji)][il])
    assert np.array_equal(Ss[il], S[np.ix_(Ji, Ji)][il])


def test_direct_oracle_refuses_oversized(restatement):
    p = alloc_problem(1, 1, 513)
    with pytest.raises(ValueError):
        restatement.direct_H(p)


@pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built (needs /root/reference at build time)")
def test_compiled_reference_matches_golden():
    ref = Reference()
    path = golden_cases()[3]
    dims, d = load_case(path)
    p = ref.generate_problem(*dims)
    r = ref.build_hs(p, "refined", threads=2, blocked=True)
    assert np.array_equal(r["H"], d["H"]) and np.array_equal(r["S"], d["S"])
    assert [ph[0] for ph in r["phases"]] == ["s", "z_loop", "her2k", "hemm_loop", "herkx"]


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1][:-4])
def test_original_restatement_vs_reference_golden(path, restatement):
    """Algorithm 1 (pipeline.cpp:189-279) restated: bit-identical H, S and the
    original-variant ledger (test_pipeline.cpp:97-113), equal to the refined result
    within 1e-11 (test_pipeline.cpp:30-40)."""
    dims, d = load_case(path)
    na, nl, ng, seed, nnh = dims
    p = restatement.generate_problem(na, nl, ng, seed, nnh)
    H, S, led, n_hpd = restatement.build_hs_original(p)
    assert n_hpd == na - nnh
    assert [led.get(k, 0) for k in LEDGER_KEYS] + [led["total"]] == d["ledger_original"].tolist()
    if "Ho" in d:
        assert np.array_equal(H, d["Ho"]) and np.array_equal(S, d["So"])
    assert restatement.rel_frobenius_error_lower(H, d["H"]) < 1e-11
    assert restatement.rel_frobenius_error_lower(S, d["S"]) < 1e-11
    iu = np.triu_indices(ng, 1)
    assert np.all(H[iu] == 0) and np.all(S[iu] == 0)


def test_potrf_restatement_vs_reference_golden(restatement):
    """kernels::potrf (kernels.cpp:417-436): factors bit-identical, failing pivots equal."""
    z = np.load(f"{GOLDEN_DIR}/potrf_blocks.npz")
    piv = z["pivots"]
    assert sorted(set(piv.tolist())) == [-1, 0, 7, 30]
    for i, want in enumerate(piv):
        L, got = restatement.potrf(z[f"T{i}"][:, :, None])
        assert got[0] == want
        if want < 0:
            assert np.array_equal(L[:, :, 0], z[f"L{i}"])
            Lf = z[f"L{i}"]
            assert np.all(Lf[np.triu_indices(Lf.shape[0], 1)] == 0)


def test_original_restatement_hpd_mixes(restatement):
    """original == refined across seeds and hpd mixes (test_pipeline.cpp:30-40) and
    the closed-form ledger delta (test_pipeline.cpp:105-112)."""
    for seed in range(1, 11):
        na, nl, ng = 4, 5, 32
        nnh = seed % (na + 1)
        p = restatement.generate_problem(na, nl, ng, seed, nnh)
        Ho, So, lo, n_hpd = restatement.build_hs_original(p)
        Hr, Sr, lr = restatement.build_hs_refined(p)
        assert restatement.rel_frobenius_error_lower(Ho, Hr) < 1e-11
        assert restatement.rel_frobenius_error_lower(So, Sr) < 1e-11
        delta = 4 * nnh * nl * ng * ng + na * (4 * nl ** 3 // 3) - 4 * n_hpd * nl * nl * ng
        assert lo["total"] - lr["total"] == delta


def test_parity_checker_negative_control(restatement):
    """The reference CLI's --corrupt-h negative control (hsdla_cli.cpp:120,346-347): a single
    perturbed lower-triangle element must push the relative Frobenius error past the 1e-11
    bar, and an upper-triangle change must not count (lower triangle authoritative)."""
    import paper_1712_07206_b200 as hb
    dims, d = load_case(golden_cases()[-1])
    H = d["H"].copy()
    assert hb.rel_frobenius_error_lower(H, d["H"]) == 0.0
    i, j = H.shape[0] - 1, 0
    H[i, j] += 1e-9 * np.linalg.norm(np.tril(d["H"]))
    assert hb.rel_frobenius_error_lower(H, d["H"]) > 1e-11
    assert restatement.rel_frobenius_error_lower(H, d["H"]) > 1e-11
    U = d["H"].copy()
    U[0, U.shape[0] - 1] += 1.0
    assert hb.rel_frobenius_error_lower(U, d["H"]) == 0.0
