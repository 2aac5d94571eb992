"""Host-side cost of the per-step public API with host buffers (the bench e2e loop), by cProfile (dev tool)."""

import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, inputs  # noqa: E402

w = configs.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
m = inputs.dense_target(w)
obj = pb.FrobeniusObjective.from_device(m, w.dtype)
x = inputs.initial_iterate(w, m)


def step(xi, t):
    return pb.lowrank_meg_step(xi, obj.grad_operator(xi), w.eta(t), w.eps(t + 1), svd_seed=t,
                               svd_subspace=w.subspace, block=w.block)


t = 0
for _ in range(5):
    x = step(x, t).iterate
    t += 1
torch.cuda.synchronize()
Vh = torch.empty((w.n, w.r), dtype=torch.float64).pin_memory()
Vh.copy_(x.V_device)
Vn = torch.empty_like(Vh).pin_memory()
lam, eps, warm, werr = x.lam.copy(), x.eps, x.warm_block, x.warm_orth_err


def loop(K):
    global Vh, Vn, lam, eps, warm, werr, t
    for _ in range(K):
        res = pb.lowrank_meg_step_host(Vh, lam, eps, obj, w.eta(t), w.eps(t + 1), svd_seed=t,
                                       svd_subspace=w.subspace, block=w.block, warm=warm, warm_orth_err=werr, out=Vn)
        Vh, Vn = Vn, Vh
        lam, eps, warm, werr = res.lam, res.eps, res.warm_block, res.warm_orth_err
        t += 1


loop(20)
torch.cuda.synchronize()
t0 = time.perf_counter()
loop(300)
torch.cuda.synchronize()
print(f"wall per step: {(time.perf_counter() - t0) / 300 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
loop(300)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
