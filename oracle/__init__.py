"""CPU oracle for the ARCHES UL channel-estimation hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package,
and only as the checker or the timed CPU baseline -- never as the product path.

`oracle.ref_path` is a numpy/scipy restatement of the reference's algorithm
(`/root/reference/pkg/src/ranswitch`, cited per function).  It is pinned against
golden vectors produced by the unmodified reference (`tools/make_golden.py`,
fixtures under `tests/golden/`, checked by `tests/test_oracle_golden.py`).
"""
