"""TEST INFRASTRUCTURE ONLY — CPU oracles for the HSDLA H/S construction.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the reported CPU baseline.  The product package ``paper_1712_07206_b200`` never
imports it.
"""
