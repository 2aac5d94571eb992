"""Per-config device performance: passes/step and ms/step of the native run loop (dev tool).

    python tools/config_profile.py [cfg1 cfg2 cfg3 cfg4 cfg5] [--steps 20]
"""

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs, runtime  # noqa: E402


def objective_for(w):
    if w.kind == "dense":
        m = inputs.dense_target(w)
        return pb.FrobeniusObjective.from_device(m, w.dtype), m
    if w.kind == "stochastic":
        m = inputs.dense_target(w)
        return pb.StochasticFrobeniusObjective.from_device(m, w.dtype, batch=w.batch, sigma=w.sigma, seed=w.seed), m
    from oracle import inputs as oin  # host CSR generation (dev tool only)

    inst = oin.sampled_instance(oin.CONFIGS[w.name], keep_planted=False)
    obj = pb.SampledObjective(w.n, inst.rowptr, inst.col, inst.obs)
    init = pb.SymmetricOperator.from_csr(w.n, inst.rowptr, inst.col, inst.obs / w.sample_p)
    return obj, init


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    for name in args.names:
        w = configs.WORKLOADS[name]
        t0 = time.time()
        obj, init = objective_for(w)
        tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
        if isinstance(init, torch.Tensor):
            x = inputs.initial_iterate(w, init, tol=tol)
        else:
            top = pb.lanczos_top_r(init, w.r, tol=tol, seed=w.seed, subspace=64, return_device=True)
            lam = pb.project_simplex(top.eigenvalues, 1.0)
            lam = np.maximum(lam / lam.sum(), 1e-12)
            x = pb.warm_start_wrap(top.eigenvectors, lam / lam.sum(), w.eps(0))
        torch.cuda.synchronize()
        setup = time.time() - t0
        s = runtime.solver_for(w.n)
        # cold start (first step) outside the trace; the traced run continues warm from its Ritz block
        r0 = driver.run(x, obj, 1, eta=w.eta0, eta_decay=w.eta_decay, svd_subspace=w.subspace, block=w.block)
        s.lib.megb200_trace_enable(s.handle, 1)
        rr = driver.run(r0.iterate, obj, args.steps, t0=1, eta=w.eta0, eta_decay=w.eta_decay,
                        svd_subspace=w.subspace, block=w.block)
        buf = C.create_string_buffer(4096)
        s.lib.megb200_trace_report(s.handle, buf, 4096)
        s.lib.megb200_trace_enable(s.handle, 0)
        steady = rr.step_ms
        print(json.dumps({"config": name, "n": w.n, "r": w.r, "dtype": w.dtype, "setup_s": round(setup, 2),
                          "first_step_ms": float(r0.step_ms[0]), "first_step_passes": int(r0.passes[0]),
                          "steady_ms_per_step": float(np.mean(steady)), "steady_passes": float(np.mean(rr.passes)),
                          "it_per_s": 1e3 / float(np.mean(steady)), "lhs_last": float(rr.lhs[-1])}), flush=True)
        print(buf.value.decode(), flush=True)
        del obj, init
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
