"""CPU oracle for the low-rank MEG hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `specmeg` algorithm
(arXiv 2012.10469; reference files cited per function) used as the parity
checker for the B200 implementation in `paper_2012_10469_b200`.

Only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may import it, and only as the
checker or the timed CPU baseline.  The product package never imports it;
the CUDA path fails loudly when its extension is missing.

Pinning: `tests/golden/make_golden.py` runs the unmodified reference
(`/root/reference/pkg/src/specmeg`, importable in the build container) on
the seeded inputs of `oracle.inputs` and commits the outputs under
`tests/golden/`; `tests/test_oracle_pins.py` checks this restatement against
those fixtures and against every known-answer test the reference's own test
suite holds for the path.
"""
