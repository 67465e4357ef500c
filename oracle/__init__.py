"""CPU oracle for the speculate-vote-verify hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import this package, and only as the checker or as
the timed CPU baseline.  The product package (`paper_2402_15678_b200`) never
imports it: the product path runs the sm_100a kernels and fails loudly when
the CUDA extension is missing.
"""
