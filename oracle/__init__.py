"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the IVFPQ search path.

Nothing in `paper_2301_06672_b200/` imports this package.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu-baseline / `--impl reference`
legs may use it, and only as the checker or the timed CPU baseline -- never
as the thing measured or shipped.

Contents
  * `ivfpq_np`  -- numpy restatement of the reference `ivfpq8` search path
                   (search.py:91-221, minifloat.py:91-169, datasets.py:166-176),
                   same per-query loop structure, so it is also the "port" CPU
                   baseline.
  * `c_oracle`  -- ctypes binding of `ivfpq_oracle.c`, a plain-C restatement of
                   the same arithmetic (compiled with -ffp-contract=off), used
                   for parity at sizes the numpy loop is too slow for.

Parity pinning: both restatements are checked against golden vectors that
`tests/golden/make_golden.py` produced by running the reference package itself
(`/root/reference/pkg/src`, importable in the build container) -- see
tests/test_oracle_golden.py.
"""
