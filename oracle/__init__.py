"""CPU oracle for satsweep-b200 -- TEST INFRASTRUCTURE ONLY.

This package restates the reference algorithm (the `satsweep` package under
/root/reference/pkg, pure Python on numpy) so the GPU path can be checked and
the reference's CPU cost can be timed.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline / `--impl reference` legs may import it, and only
as the checker or the timed CPU baseline -- never as a product code path.

Parity is pinned: tests/test_oracle_golden.py checks every function here
against golden vectors produced by the reference itself
(tests/golden/make_golden.py, run in the survey container where the reference
is importable).
"""
