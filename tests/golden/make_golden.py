"""Generate golden fixtures by running the UNMODIFIED reference `specmeg` package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--only NAME ...]

It imports the reference from $SPECMEG_SRC (default
/root/reference/pkg/src), drives `specmeg.meg.lowrank_meg_step` on the seeded
inputs of `oracle.inputs` with the factored driver of `oracle.objectives`
(exactly the driver the survey measured), and writes one
compressed .npz per case into tests/golden/.  The GPU box never needs the
reference: the fixtures travel with the repo.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("SPECMEG_SRC", "/root/reference/pkg/src"))

from specmeg import linalg as ref_linalg  # noqa: E402
from specmeg import meg as ref_meg  # noqa: E402
from specmeg import objectives as ref_obj  # noqa: E402

from oracle import inputs, objectives  # noqa: E402

REF = types.SimpleNamespace(
    SymmetricOperator=ref_linalg.SymmetricOperator,
    lanczos_top_r=ref_linalg.lanczos_top_r,
    project_simplex=ref_linalg.project_simplex,
    warm_start_wrap=ref_meg.warm_start_wrap,
    lowrank_meg_step=ref_meg.lowrank_meg_step,
)

OUT = os.path.join(ROOT, "tests", "golden")

# (name, config, n override, iterations, probe iterations)
CASES = [
    ("cfg1_full", "cfg1", None, 200, (0, 49, 99, 199)),
    ("cfg2_prefix", "cfg2", None, 5, (0, 4)),
    ("cfg2_n1024", "cfg2", 1024, 30, (0, 29)),
    ("cfg3_n2048", "cfg3", 2048, 20, (0, 19)),
    ("cfg3_prefix", "cfg3", None, 3, (0, 2)),
    ("cfg4_n2048", "cfg4", 2048, 30, (0, 29)),
    ("cfg4_prefix", "cfg4", None, 3, (0, 2)),
    ("cfg5_n2048", "cfg5", 2048, 20, (0, 19)),
]


def dual_gap_reference(obj, x, seed):
    """Reference `_dual_gap_core` on the dense gradient X - M (objectives.py:332-335)."""
    grad = x.densify() - obj.m
    trace_term = float(np.sum(x.densify() * grad))
    return ref_obj._dual_gap_core(grad, trace_term, tau=1.0, seed=seed)


def make_case(name, cfg_name, n, iters, probe_at):
    cfg = inputs.CONFIGS[cfg_name]
    if n is not None:
        cfg = cfg.scaled(n, iters)
    t0 = time.time()
    obj = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(REF, cfg, obj)
    t1 = time.time()
    rec, x = objectives.run_trajectory(REF, cfg, obj, x0, iters, probe_at=probe_at)
    t2 = time.time()
    z = objectives.probes(cfg.n)
    rec["x0_probe"] = objectives.x_apply(x0, z)
    rec["x0_lam"] = np.asarray(x0.lam)
    rec["x0_eps"] = np.float64(x0.eps)
    rec["f0"] = np.float64(obj.value(x0))
    rec["n"] = np.int64(cfg.n)
    rec["iters"] = np.int64(iters)
    rec["seconds_per_iter"] = np.float64((t2 - t1) / iters)
    if cfg.cert_every and n is not None:
        # dual gap at the final iterate (small n only: needs the dense gradient)
        rec["dual_gap_final"] = np.float64(dual_gap_reference(obj, x, seed=0))
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"{name}: n={cfg.n} iters={iters} init {t1 - t0:.1f}s, {(t2 - t1) / iters:.3f}s/iter -> {path}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    for case in CASES:
        if args.only and case[0] not in args.only:
            continue
        make_case(*case)


if __name__ == "__main__":
    main()
