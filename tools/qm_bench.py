"""Quadratic-measurement MEG steps/s on the device vs the CPU oracle port (dev tool).

    python tools/qm_bench.py [--steps 200]

The paper's experiment sizes (§7): n = 100, r = 1 / 5 / 20, m = 20 n r, kappa = 1/2,
eta = 1 / (0.4 sqrt(r n)).  Device: per-step public API (lowrank_meg_step with
QuadMeasObjective.grad_operator: residual kernel, gradient kernels, pass + fused Rayleigh-Ritz),
inputs resident in HBM.  CPU: oracle/cpu_meg.lowrank_meg_step + oracle/qm (numpy/OpenBLAS).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import inputs  # noqa: E402


def eps(t):
    return min(0.6 / (t + 11.0) ** 2, 0.75)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    ap.add_argument("--sizes", default="100x1,100x5,100x20", help="comma-separated n x r list")
    ap.add_argument("--split", action="store_true", help="also time gradient and step separately (host clock)")
    args = ap.parse_args()
    from oracle import cpu_meg as om  # CPU comparison leg only
    from oracle import qm as oq

    for n, r in (tuple(int(v) for v in nr.split("x")) for nr in args.sizes.split(",")):
        a, b, y, tau = inputs.quad_meas_instance(n, r, seed=0)
        obj = pb.QuadMeasObjective(a, b, y, tau)
        eta = 1.0 / pb.QuadMeasObjective.preset_beta(n, r)
        rng = np.random.default_rng(1000)
        q, _ = np.linalg.qr(rng.standard_normal((n, r)))
        x0 = pb.warm_start_wrap(q, np.full(r, 1.0 / r), eps(0))
        x = x0
        for t in range(5):
            x = pb.lowrank_meg_step(x, obj.grad_operator(x), eta, eps(t + 1), svd_seed=t).iterate
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        passes = 0
        for t in range(5, 5 + args.steps):
            res = pb.lowrank_meg_step(x, obj.grad_operator(x), eta, eps(t + 1), svd_seed=t)
            x, passes = res.iterate, passes + res.passes
        e1.record()
        torch.cuda.synchronize()
        gpu = args.steps / (e0.elapsed_time(e1) / 1e3)
        split = {}
        if args.split:
            tg = ts = 0.0
            for t in range(5 + args.steps, 5 + 2 * args.steps):
                h0 = time.perf_counter()
                op = obj.grad_operator(x)
                torch.cuda.synchronize()
                h1 = time.perf_counter()
                x = pb.lowrank_meg_step(x, op, eta, eps(t + 1), svd_seed=t).iterate
                torch.cuda.synchronize()
                h2 = time.perf_counter()
                tg, ts = tg + h1 - h0, ts + h2 - h1
            split = {"grad_ms": round(1e3 * tg / args.steps, 4), "step_ms": round(1e3 * ts / args.steps, 4)}
        inst = oq.generate_instance(n, r, seed=0)
        ox = om.warm_start_wrap(q, np.full(r, 1.0 / r), eps(0))
        done, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < args.cpu_seconds:
            G = oq.dense_gradient(inst, oq.residuals(inst, ox), inst.tau)
            ox = om.lowrank_meg_step(ox, lambda u, G=G: G @ u, eta, eps(done + 1), svd_seed=done).iterate
            done += 1
        cpu = done / (time.perf_counter() - t0)
        print(json.dumps({"n": n, "r": r, "m": 20 * n * r, "gpu_it_per_s": round(gpu, 1),
                          "passes_per_step": passes / args.steps, "cpu_port_it_per_s": round(cpu, 2),
                          "cpu_cores": len(os.sched_getaffinity(0)), **split}), flush=True)


if __name__ == "__main__":
    main()
