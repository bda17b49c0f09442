"""CPU oracle for the MOR frequency-sweep hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy, the reference `vibrofem` algorithms
on the north-star path (SURVEY.md §8a rows A1–A15).  Every function cites the
reference file:line it follows (paths relative to /root/reference/pkg/src/
vibrofem/).

Who may import it: `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs — and only as the CHECKER or the
timed CPU baseline.  The product package `paper_2310_04734_b200` never
imports anything from here; its compute runs through the CUDA C-ABI library
and fails loudly when that library is missing.

Parity pin: the restatement is checked against golden vectors produced by the
unmodified reference (tests/golden/make_golden.py, run in the build
container with PYTHONPATH=/root/reference/pkg/src) — see DESIGN.md §3.
"""
