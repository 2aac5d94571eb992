"""Native run loop: T low-rank MEG steps in one call (megb200_meg_run).

The reference has no driver in its code -- the loop lives in its tests
(test_meg.py:150-156) and in the spec's absent harness (SPEC.md:433-450,
SURVEY.md 8f rank 2).  `run` is that loop, executed natively: the iterate,
the warm Ritz block and (for the stochastic objective) the minibatch stay on
the device between steps, the schedules are evaluated in C++, and the
per-step records come back in one batch.  Step t uses eta_t, eps_next =
eps_{t+1}, svd_seed = t -- the same convention as oracle.objectives.run_trajectory.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, runtime
from .errors import ParameterError
from .linalg import _eig_opts
from .meg import EpsilonSchedule, LowRankIterate, StepConfig
from .objectives import FrobeniusObjective, SampledObjective, StochasticFrobeniusObjective


@dataclass
class RunResult:
    iterate: LowRankIterate
    shift: np.ndarray  # (T,)
    y: np.ndarray  # (T, r+1) exp(mu - mu_1)
    lam: np.ndarray  # (T, r)
    eps: np.ndarray  # (T,)
    lhs: np.ndarray  # (T,) cheap certificate
    holds: np.ndarray  # (T,) bool
    passes: np.ndarray  # (T,) operand passes per step
    step_ms: np.ndarray  # (T,) device time per step (flush excluded)


def _schedule(eps_schedule: EpsilonSchedule, eta, eta_decay: bool, objective) -> _lib.Schedule:
    sc = _lib.Schedule()
    if eps_schedule.kind not in _lib.EPS_KINDS:
        raise ParameterError(f"unknown epsilon schedule {eps_schedule.kind!r}")
    sc.eps_kind = _lib.EPS_KINDS[eps_schedule.kind]
    sc.eps0_tilde, sc.G, sc.c = eps_schedule.eps0_tilde, eps_schedule.G, eps_schedule.c
    eta0 = eta.eval(0) if isinstance(eta, StepConfig) else float(eta)
    if not eta0 > 0:
        raise ParameterError(f"eta must be positive, got {eta0}")
    sc.eta_kind = 1 if eta_decay else 0
    sc.eta0 = eta0
    if isinstance(objective, StochasticFrobeniusObjective):
        sc.minibatch_seed = objective.seed
        sc.minibatch_round_f32 = 1 if objective.dtype == "f32" else 0
    return sc


def run(
    x0: LowRankIterate,
    objective,
    T: int,
    *,
    t0: int = 0,
    eps_schedule: EpsilonSchedule | None = None,
    eta=1.0,
    eta_decay: bool = False,
    svd_tol: float = 1e-10,
    svd_subspace: int | None = None,
    block: int | None = None,
    flush_bytes: int = 0,
    timing: bool = True,
) -> RunResult:
    """Run T MEG steps from x0 on `objective` (Frobenius, sampled or stochastic).

    timing=False skips the per-step CUDA events (step_ms is then all zeros)."""
    if not isinstance(objective, (FrobeniusObjective, SampledObjective)):
        raise TypeError("run() needs a device objective (FrobeniusObjective, StochasticFrobeniusObjective, "
                        "SampledObjective)")
    eps_schedule = eps_schedule or EpsilonSchedule.experiment(10.0)
    n, r = x0.n, x0.r
    g = objective.grad_operator(x0, t0)
    s = g.solver()
    hold: list = []
    xs, gs = x0.struct(hold), g.struct(hold)
    warm = x0.warm_block if isinstance(x0.warm_block, torch.Tensor) and x0.warm_block.shape[0] == n else None
    opts = _eig_opts(max(svd_tol, g.tol_floor), None, 0, svd_subspace, 12, block, None, warm,
                     warm_orthonormal=warm is not None and x0.warm_orth_err <= 1e-13)
    sc = _schedule(eps_schedule, eta, eta_decay, objective)
    T = int(T)
    out = {k: np.zeros(T) for k in ("shift", "eps", "lhs", "step_ms")}
    out["y"] = np.zeros((T, r + 1))
    out["lam"] = np.zeros((T, r))
    holds = np.zeros(T, dtype=np.int32)
    passes = np.zeros(T, dtype=np.int32)
    rec = _lib.RunRecord()
    for k in ("shift", "eps", "lhs", "step_ms", "y", "lam"):
        if k == "step_ms" and not timing:
            continue
        setattr(rec, k, _lib.dptr(out[k]))
    rec.holds = holds.ctypes.data_as(_lib.c_int32_p)
    rec.passes = passes.ctypes.data_as(_lib.c_int32_p)
    v_out = torch.empty((n, r), dtype=torch.float64, device=runtime.device())
    ritz = torch.empty((n, runtime.MAX_BLOCK), dtype=torch.float64, device=runtime.device())
    rec.ritz_block = ritz.data_ptr()
    rec.ld_ritz = ritz.stride(0)
    rec.ritz_cap = ritz.shape[1]
    lam_out = np.zeros(r)
    eps_out = C.c_double()
    runtime.check(s.lib.megb200_meg_run(s.handle, C.byref(xs), C.byref(gs), C.byref(sc), int(t0), T, C.byref(opts),
                                        int(flush_bytes), v_out.data_ptr(), r, _lib.dptr(lam_out),
                                        C.byref(eps_out), C.byref(rec)))
    # the final iterate carries the warm Ritz block, so a later run or step continues warm
    x = (LowRankIterate(n, r, v_out, lam_out, eps_out.value, warm_block=ritz[:, : rec.ritz_cols],
                        warm_orth_err=rec.ritz_orth_err) if T > 0 else x0)
    return RunResult(iterate=x, holds=holds.astype(bool), passes=passes, **out)
