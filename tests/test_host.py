"""Host-side logic of the product package (no GPU): generator, HSDL I/O, presets,
flop model, config errors, helpers."""
import os

import numpy as np
import pytest

import paper_1712_07206_b200 as hb
from conftest import GOLDEN, as_problem, golden_cases, load_case


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1][:-4])
def test_generate_problem_bitwise_vs_reference(path):
    dims, d = load_case(path)
    p = hb.generate_problem(*dims)
    for k in ("A", "B", "T_AA", "T_AB", "T_BB", "U"):
        assert np.array_equal(getattr(p, k), d[k]), k
    assert np.array_equal(p.hpd_flags, d["hpd"].astype(bool))
    assert p.A.flags.f_contiguous


@pytest.mark.parametrize("dims,lo,hi", [((7, 6, 48, 3, 2), 0, 7), ((7, 6, 48, 3, 2), 2, 5), ((7, 6, 48, 3, 2), 6, 7),
                                         ((5, 9, 97, 11, 5), 1, 3), ((16, 49, 200, 1, 0), 8, 16)])
def test_generate_problem_shard_is_the_full_instance_rows(dims, lo, hi):
    """Each rank of a multi-GPU run generates only its atoms: bit-identical to the same rows /
    blocks of the full generate_problem (the generator stream of other atoms is skipped)."""
    na, nl, ng, seed, nnh = dims
    full = hb.generate_problem(*dims)
    sh = hb.generate_problem_shard(na, nl, ng, lo, hi, seed, nnh)
    assert sh.n_atoms == hi - lo and sh.atom_begin == lo and sh.n_atoms_total == na
    assert np.array_equal(sh.A, full.A[lo * nl:hi * nl]) and np.array_equal(sh.B, full.B[lo * nl:hi * nl])
    for k in ("T_AA", "T_AB", "T_BB", "U"):
        assert np.array_equal(getattr(sh, k), getattr(full, k)[..., lo:hi]), k
    assert np.array_equal(sh.hpd_flags, full.hpd_flags[lo:hi])
    with pytest.raises(hb.DimensionError):
        hb.generate_problem_shard(na, nl, ng, hi, lo, seed, nnh)


def test_generate_problem_dimension_errors():
    with pytest.raises(hb.DimensionError):
        hb.generate_problem(0, 1, 1)
    with pytest.raises(hb.DimensionError):
        hb.generate_problem(2, 1, 1, 1, 3)


def test_hsdl_reference_file_roundtrip(tmp_path):
    p = hb.load_problem(os.path.join(GOLDEN, "small_2_3_16_s1_nh1.hsdl"))
    q = hb.generate_problem(2, 3, 16, 1, 1)
    for k in ("A", "B", "T_AA", "T_AB", "T_BB", "U"):
        assert np.array_equal(getattr(p, k), getattr(q, k)), k
    assert list(p.hpd_flags) == [True, False]
    out = tmp_path / "rt.hsdl"
    hb.save_problem(p, str(out))
    assert out.read_bytes() == open(os.path.join(GOLDEN, "small_2_3_16_s1_nh1.hsdl"), "rb").read()


def test_hsdl_malformed(tmp_path):
    bad = tmp_path / "bad.hsdl"
    bad.write_bytes(b"NOPE" + b"\0" * 40)
    with pytest.raises(hb.IoError):
        hb.load_problem(str(bad))
    src = open(os.path.join(GOLDEN, "small_2_3_16_s1_nh1.hsdl"), "rb").read()
    (tmp_path / "trunc.hsdl").write_bytes(src[:100])
    with pytest.raises(hb.IoError):
        hb.load_problem(str(tmp_path / "trunc.hsdl"))
    (tmp_path / "ver.hsdl").write_bytes(src[:4] + b"\x02\0\0\0" + src[8:])
    with pytest.raises(hb.IoError):
        hb.load_problem(str(tmp_path / "ver.hsdl"))
    with pytest.raises(hb.IoError):
        hb.load_problem(str(tmp_path / "missing.hsdl"))


def test_presets():
    names = [p.name for p in hb.presets()]
    assert len(names) == 12 and "auag-4.0" in names
    p = hb.find_preset("tio2-3.5", 0.5)
    assert (p.n_atoms, p.n_l, p.n_g) == (192, 41, 9777)
    assert hb.find_preset("nope") is None


def test_flop_model_matches_reference_ledger():
    for path in golden_cases():
        dims, d = load_case(path)
        led = hb.flop_model(as_problem(d, dims))
        keys = ("gemm", "hemm", "her2k", "herk", "scaling", "herkx", "potrf", "trmm")
        assert [led.count(k) for k in keys] + [led.total()] == d["ledger"].tolist()
    unit = hb.empty_problem(1, 1, 1)
    assert hb.flop_model(unit).total() == 46


def test_config_errors():
    p = hb.generate_problem(1, 2, 4, 81, 0)
    with pytest.raises(hb.ConfigError):
        hb.build_hs(p, hb.PipelineConfig(strategy="dynamic"))
    with pytest.raises(hb.ConfigError):
        hb.build_hs(p, hb.PipelineConfig(variant="original"))
    with pytest.raises(hb.ConfigError):
        hb.parse_variant("x")
    with pytest.raises(hb.ConfigError):
        hb.build_hs_refined(p, hb.PipelineConfig(algo="bogus"))
    # the C-ABI algorithm numbering the Python mirror relies on (include/hsdla_b200.h)
    from paper_1712_07206_b200.pipeline import ALGOS
    assert ALGOS == {"merged": 0, "refined": 1, "original": 2, "fused": 3}
    assert hb.PipelineConfig().algo == "merged"
    with pytest.raises(hb.DimensionError):
        bad = hb.generate_problem(1, 2, 4, 81, 0)
        bad.A = np.ascontiguousarray(bad.A)  # C order is not the reference layout
        bad.validate()


def test_no_cpu_fallback_without_gpu():
    if hb.device_count() > 0:
        pytest.skip("GPU present")
    p = hb.generate_problem(1, 2, 4, 81, 0)
    with pytest.raises(hb.ConfigError):
        hb.build_hs_refined(p)


def test_mirror_and_rel_error():
    rng = np.random.default_rng(0)
    M = np.tril(rng.standard_normal((5, 5)) + 1j * rng.standard_normal((5, 5))).astype(np.complex128)
    M = np.asfortranarray(M)
    X = hb.mirror(M.copy())
    assert np.allclose(X, X.conj().T) and np.all(np.diag(X).imag == 0)
    assert hb.rel_frobenius_error_lower(M, M) == 0.0


def test_native_hsdl_header_reader(tmp_path):
    """The library's own HSDL v1 header reader (the streaming loader's front end,
    problem.cpp:197-225) on the reference-written file and on malformed files
    (test_io.cpp:47-63): IoError for bad magic, bad version, truncation, no file."""
    ref = os.path.join(GOLDEN, "small_2_3_16_s1_nh1.hsdl")
    na, nl, ng, hpd = hb.problem_file_info(ref)
    assert (na, nl, ng) == (2, 3, 16) and list(hpd) == [True, False]
    src = open(ref, "rb").read()
    cases = {"bad.hsdl": b"NOPE" + b"\0" * 64, "ver.hsdl": src[:4] + b"\x02\0\0\0" + src[8:],
             "trunc.hsdl": src[: len(src) // 2], "hdr.hsdl": src[:20]}
    for name, data in cases.items():
        (tmp_path / name).write_bytes(data)
        with pytest.raises(hb.IoError):
            hb.problem_file_info(str(tmp_path / name))
    with pytest.raises(hb.IoError):
        hb.problem_file_info("/nonexistent/nowhere.hsdl")
    with pytest.raises(hb.IoError):
        hb.build_hs_file(str(tmp_path / "trunc.hsdl"))  # rejected before any device work
    big = hb.generate_problem(37, 5, 9, 4, 11)
    hb.save_problem(big, str(tmp_path / "big.hsdl"))
    na, nl, ng, hpd = hb.problem_file_info(str(tmp_path / "big.hsdl"))
    assert (na, nl, ng) == (37, 5, 9) and np.array_equal(hpd, big.hpd_flags)
