"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (where /root/reference exists) after
`make -C oracle ref`:

    python tests/golden/make_golden.py

Every array comes from oracle/_ref/libhsdla_ref.so, i.e. the reference sources
compiled in place (proj/src/*.cpp):
  problem   generate_problem          proj/src/problem.cpp:79-142
  H, S      build_hs_refined (Cpu, Variant::Reference)  proj/src/pipeline.cpp:281-329
  Ho, So    build_hs_original                           proj/src/pipeline.cpp:189-279
  Hd, Sd    oracle::direct_H / direct_S                 proj/src/oracle.cpp:72-103
  ledger    the measured refined ledger (== flop_model, pipeline.cpp:336-364)
The HSDL v1 file is written by the reference's own save_problem (problem.cpp:172-195).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import LEDGER_KEYS, Reference  # noqa: E402

CASES = [
    # (n_atoms, n_l, n_g, seed, n_not_hpd)
    (1, 1, 1, 1, 0),
    (2, 3, 16, 1, 0),
    (4, 7, 64, 2, 2),
    (8, 5, 128, 99, 4),
    (3, 49, 50, 5, 1),
    (2, 81, 40, 7, 0),
    (1, 121, 24, 3, 0),
    (5, 9, 97, 11, 0),
]


def main():
    ref = Reference()
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for na, nl, ng, seed, nnh in CASES:
        p = ref.generate_problem(na, nl, ng, seed, nnh)
        r = ref.build_hs(p, "refined", threads=1, blocked=False)
        o = ref.build_hs(p, "original", threads=1, blocked=False)
        led = r["ledger"]
        name = f"case_{na}_{nl}_{ng}_s{seed}_nh{nnh}.npz"
        extra = {}
        if ng <= 64:  # keep the fixture tree small: the cross-variant arrays only for small cases
            extra = dict(Ho=o["H"], So=o["S"], Hg=ref.direct_H_grouped(p))
        np.savez_compressed(
            os.path.join(out_dir, name),
            dims=np.array([na, nl, ng, seed, nnh], np.uint64),
            A=p.A, B=p.B, T_AA=p.T_AA, T_AB=p.T_AB, T_BB=p.T_BB, U=p.U, hpd=p.hpd_flags,
            H=r["H"], S=r["S"], Hd=ref.direct_H(p), Sd=ref.direct_S(p), **extra,
            ledger=np.array([led.get(k, 0) for k in LEDGER_KEYS] + [led["total"]], np.uint64),
            ledger_original=np.array([o["ledger"].get(k, 0) for k in LEDGER_KEYS] + [o["ledger"]["total"]],
                                     np.uint64),
        )
        print("wrote", name)
    # kernels::potrf known answers (kernels.cpp:417-436): HPD blocks of the
    # generator's T_AA at N_L 1/5/49/81/121 plus indefinite blocks that fail at
    # pivots 0 (the generator's non-HPD shift), 7 and 30.
    blocks = []
    for nl, seed, nnh in ((1, 3, 0), (5, 4, 1), (49, 5, 1), (81, 6, 0), (121, 7, 0)):
        q = ref.generate_problem(1 + nnh, nl, 1, seed, nnh)
        blocks += [q.T_AA[:, :, a] for a in range(q.n_atoms)]
    for nl, bad in ((16, 7), (49, 30)):
        q = ref.generate_problem(1, nl, 1, 8 + bad, 0)
        t = q.T_AA[:, :, 0].copy()
        t[bad, bad] -= 1e3  # indefinite from column `bad` on
        blocks.append(t)
    ls, pivs, ts = [], [], []
    for t in blocks:
        L, piv = ref.potrf(t[:, :, None])
        ts.append(t)
        ls.append(L[:, :, 0])
        pivs.append(int(piv[0]))
    np.savez_compressed(os.path.join(out_dir, "potrf_blocks.npz"),
                        **{f"T{i}": t for i, t in enumerate(ts)}, **{f"L{i}": l for i, l in enumerate(ls)},
                        pivots=np.array(pivs, np.int64))
    print("wrote potrf_blocks.npz", pivs)
    p = ref.generate_problem(2, 3, 16, 1, 1)
    ref.save_problem(p, os.path.join(out_dir, "small_2_3_16_s1_nh1.hsdl"))
    print("wrote small_2_3_16_s1_nh1.hsdl")


if __name__ == "__main__":
    main()
