"""Adapters that drive the B200 package with the oracle's trajectory driver (tests only)."""

from __future__ import annotations

import types

import numpy as np

from oracle import inputs, objectives


class GpuObjective:
    """Wraps a device objective so `oracle.objectives.run_trajectory` can drive it."""

    def __init__(self, cfg: inputs.MegConfig, host_obj):
        import paper_2012_10469_b200 as pb

        self.cfg = cfg
        if cfg.kind == "dense":
            self.dev = pb.FrobeniusObjective(host_obj.m, dtype=cfg.dtype)
        elif cfg.kind == "sampled":
            inst = host_obj.inst
            self.dev = pb.SampledObjective(cfg.n, inst.rowptr, inst.col, inst.obs)
        elif cfg.kind == "stochastic":
            self.dev = pb.StochasticFrobeniusObjective(host_obj.m, batch=cfg.batch, sigma=cfg.sigma, seed=cfg.seed,
                                                       dtype=cfg.dtype)
        else:
            raise ValueError(cfg.kind)
        if cfg.kind != "sampled":
            self.value_direct = self.dev.value  # the device value is the entry-by-entry sum

    def grad_apply(self, x, t: int = 0):
        return self.dev.grad_operator(x, t)

    def value(self, x) -> float:
        return self.dev.value(x)


def gpu_api():
    import paper_2012_10469_b200 as pb

    return types.SimpleNamespace(lowrank_meg_step=pb.lowrank_meg_step)


def upload_iterate(x0):
    import paper_2012_10469_b200 as pb

    return pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps)


def run_gpu(cfg, host_obj, x0, iters, probe_at=(), **kw):
    gobj = GpuObjective(cfg, host_obj)
    rec, x = objectives.run_trajectory(gpu_api(), cfg, gobj, upload_iterate(x0), iters, probe_at=probe_at,
                                       step_kwargs=kw)
    return rec, x, gobj


def f_scale(host_obj) -> float:
    if hasattr(host_obj, "m_norm2"):
        return 0.5 * host_obj.m_norm2
    return 0.5 * float(host_obj.inst.obs @ host_obj.inst.obs)


def random_lowrank_iterate_np(n, r, rng, eps=None):
    """test_entropy.py:28-35 fixture (host arrays)."""
    q, _ = np.linalg.qr(rng.standard_normal((n, r)))
    lam = np.sort(rng.dirichlet(np.ones(r) * 3))[::-1]
    lam = np.maximum(lam, 1e-6)
    lam /= lam.sum()
    lam = np.sort(lam)[::-1]
    if eps is None:
        eps = float(rng.uniform(0.01, 0.5))
    return q, lam, eps
