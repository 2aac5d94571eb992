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
    ("cfg3_prefix", "cfg3", None, 8, (0, 7)),
    ("cfg4_n2048", "cfg4", 2048, 30, (0, 29)),
    ("cfg4_prefix", "cfg4", None, 8, (0, 7)),
    ("cfg5_n2048", "cfg5", 2048, 20, (0, 19)),
    # the benched window: full-size cfg2 past the bench's warm-up into its steady one-pass regime
    ("cfg2_long", "cfg2", None, 45, (0, 22, 44)),
    # full-size cfg5 (n = 32768, the 4 GiB fp32 operand) with the dual-gap certificate
    ("cfg5_full", "cfg5", None, 3, (0, 2)),
]

# cases whose GPU tests start from the stored reference warm start instead of re-deriving it
STORE_X0 = {"cfg2_long", "cfg3_prefix", "cfg4_prefix", "cfg5_full"}


def dual_gap_reference(obj, x, seed, consume_m=False):
    """Reference `_dual_gap_core` on the dense gradient X - M (objectives.py:332-335).

    The dense gradient is built row chunk by row chunk from the factors (X rows minus M rows),
    never via densify(); with consume_m the gradient is formed in M's own storage (n = 32768)."""
    grad = obj.m if consume_m else obj.m.copy()
    if consume_m:
        obj.m = None
    trace_term = 0.0
    for i0 in range(0, x.n, 1024):
        i1 = min(x.n, i0 + 1024)
        xr = objectives.x_rows(x, i0, i1)
        grad[i0:i1] = xr - grad[i0:i1]
        trace_term += float(np.einsum("ij,ij->", xr, grad[i0:i1]))
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
    if hasattr(obj, "value_direct"):
        rec["f0_direct"] = np.float64(obj.value_direct(x0))
    if name in STORE_X0:
        rec["V0"] = np.asarray(x0.V)
        # checksums of the (fp32-rounded) operand the device generator must reproduce
        if hasattr(obj, "m"):
            rec["m_probe"] = obj.m @ z
            rec["m_trace"] = np.float64(np.trace(obj.m))
            rec["m_norm2"] = np.float64(obj.m_norm2)
    if cfg.cert_every:
        # dual gap at the final iterate (objectives.py:332-335 on the dense X - M)
        t3 = time.time()
        rec["dual_gap_final"] = np.float64(dual_gap_reference(obj, x, seed=0, consume_m=n is None))
        print(f"{name}: dual gap {float(rec['dual_gap_final']):.12g} in {time.time() - t3:.1f}s", flush=True)
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
