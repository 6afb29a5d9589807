"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A numpy/scipy + plain-C restatement of the reference `paradiff` solvers
(`/root/reference/pkg/src/paradiff`), used to check the CUDA path.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU baseline / reference
arm may import it, and only as the checker or the timed CPU baseline — the
product package `paper_2006_12883_b200` never imports or calls it.

Pinning: `tests/test_oracle_golden.py` checks this restatement against golden
vectors produced by running the real reference in the build container
(`tests/golden/make_golden.py`, fixtures in `tests/golden/*.npz`).
"""
