"""Sweep block width / svd_subspace of a multi-pass config (dev tool): steady ms/step and passes/step.

    [MEGB200_BASIS_BLOCKS=.. MEGB200_KEEP=..] python tools/cfg_sweep.py cfg3 --blocks 12,18,24 --subspaces 0,64
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import warnings  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs  # noqa: E402
from config_profile import objective_for  # noqa: E402

warnings.simplefilter("ignore")
ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--blocks", default="")
ap.add_argument("--subspaces", default="")
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--t0", type=int, default=20)
a = ap.parse_args()
w = configs.WORKLOADS[a.name]
obj, init = objective_for(w)
tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
if isinstance(init, torch.Tensor):
    x = inputs.initial_iterate(w, init, tol=tol)
else:
    top = pb.lanczos_top_r(init, w.r, tol=tol, seed=w.seed, subspace=64, return_device=True)
    lam = pb.project_simplex(top.eigenvalues, 1.0)
    lam = np.maximum(lam / lam.sum(), 1e-12)
    x = pb.warm_start_wrap(top.eigenvectors, lam / lam.sum(), w.eps(0))
# common prefix so every variant starts from the same iterate
pre = driver.run(x, obj, a.t0, eta=w.eta0, eta_decay=w.eta_decay, svd_subspace=w.subspace, block=w.block)
blocks = [int(b) for b in a.blocks.split(",") if b] or [w.block]
subs = [int(s) for s in a.subspaces.split(",") if s] or [w.subspace or 0]
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("MEGB200_"))
for b in blocks:
    for sub in subs:
        try:
            x1 = pb.LowRankIterate(w.n, w.r, pre.iterate.V, pre.iterate.lam, pre.iterate.eps)
            rr = driver.run(x1, obj, a.steps, t0=a.t0, eta=w.eta0, eta_decay=w.eta_decay,
                            svd_subspace=sub or None, block=b)
            h = a.steps // 2
            print(f"{a.name} [{env}] block={b} subspace={sub}: {np.mean(rr.step_ms[h:]):8.3f} ms/step "
                  f"passes {np.mean(rr.passes[h:]):6.2f}  it/s {1e3 / np.mean(rr.step_ms[h:]):7.1f} lhs {rr.lhs[-1]:.12f}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{a.name} [{env}] block={b} subspace={sub}: FAILED {type(e).__name__}: {str(e)[:120]}", flush=True)
