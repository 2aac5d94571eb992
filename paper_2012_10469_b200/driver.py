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
from .meg import EpsilonSchedule, LowRankIterate, StepConfig, effective_settings
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
    timed_ms: float = 0.0  # device time of steps [timed_from, timed_from + timed_count) (CUDA events, in loop)
    timed_launches: int = 0  # kernels enqueued for those steps
    gap: np.ndarray | None = None  # (T,) dual gap of X_{t+1} at certificate steps, NaN elsewhere
    lmin: np.ndarray | None = None  # (T,) lambda_min(grad f(X_{t+1})) at certificate steps


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
    timed_from: int = 0,
    timed_count: int = 0,
    cert_every: int = 0,
) -> RunResult:
    """Run T MEG steps from x0 on `objective` (Frobenius, sampled or stochastic).

    timing=False skips the per-step CUDA events (step_ms is then all zeros).  timed_count > 0
    brackets steps [timed_from, timed_from + timed_count) with CUDA events on the solver stream
    inside the loop (RunResult.timed_ms): the device time of exactly those steps, the steps
    before them serving as warm-up of the same pipelined loop.  cert_every > 0 (Frobenius
    objectives) computes the dual-gap certificate (_dual_gap_core, objectives.py:332-335) of
    X_{t+1} after every step t with (t + 1) % cert_every == 0, inside the native loop, each
    solve warm-started from the previous certificate's Ritz block (RunResult.gap / .lmin)."""
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
    tol_eff, sub_eff = effective_settings(svd_tol, svd_subspace, g)
    opts = _eig_opts(tol_eff, None, 0, sub_eff, 12, block, None, warm,
                     warm_orthonormal=warm is not None and x0.warm_orth_err <= 1e-13)
    sc = _schedule(eps_schedule, eta, eta_decay, objective)
    if cert_every < 0:
        raise ParameterError("cert_every must be >= 0")
    sc.cert_every = int(cert_every)
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
    gap = np.full(T, np.nan)
    lmin = np.full(T, np.nan)
    if cert_every:
        rec.gap, rec.lmin = _lib.dptr(gap), _lib.dptr(lmin)
    rec.holds = holds.ctypes.data_as(_lib.c_int32_p)
    rec.passes = passes.ctypes.data_as(_lib.c_int32_p)
    v_out = torch.empty((n, r), dtype=torch.float64, device=runtime.device())
    ritz = torch.empty((n, runtime.MAX_BLOCK), dtype=torch.float64, device=runtime.device())
    rec.ritz_block = ritz.data_ptr()
    rec.ld_ritz = ritz.stride(0)
    rec.ritz_cap = ritz.shape[1]
    if timed_count > 0:
        if timed_from < 0 or timed_from + timed_count > T:
            raise ParameterError("timed steps must lie inside [0, T)")
        rec.timed_from, rec.timed_count = int(timed_from), int(timed_count)
    lam_out = np.zeros(r)
    eps_out = C.c_double()
    runtime.check(s.lib.megb200_meg_run(s.handle, C.byref(xs), C.byref(gs), C.byref(sc), int(t0), T, C.byref(opts),
                                        int(flush_bytes), v_out.data_ptr(), r, _lib.dptr(lam_out),
                                        C.byref(eps_out), C.byref(rec)))
    # the final iterate carries the warm Ritz block, so a later run or step continues warm
    x = (LowRankIterate(n, r, v_out, lam_out, eps_out.value, warm_block=ritz[:, : rec.ritz_cols],
                        warm_orth_err=rec.ritz_orth_err) if T > 0 else x0)
    return RunResult(iterate=x, holds=holds.astype(bool), passes=passes, timed_ms=rec.timed_ms,
                     timed_launches=rec.timed_launches, gap=gap if cert_every else None,
                     lmin=lmin if cert_every else None, **out)


# ---------------------------------------------------------------------------
# Recovery runs (the paper's experiment): a step loop over the
# quadratic-measurement objective with the RunRecord rows of SPEC.md's harness
# (t, f_value, eps_t, eta_t, cheap certificate, lambda_{r+1}, elapsed) and an optional dual gap
# every k rows, emitted as the spec's CSV.  The full-certificate / Bregman columns need the
# dense shadow (out of scope) and are left empty, as the spec prescribes for missing fields.

RUN_CSV_HEADER = ("t,f_value,eps_t,eta_t,cert_cheap_lhs,cert_cheap_holds,cert_full_lhs,cert_full_holds,"
                  "bregman_to_exact,lambda_rsp1,elapsed_ns")


@dataclass
class RecoveryRun:
    iterate: LowRankIterate
    rows: list  # dicts keyed by the CSV columns (+ "dual_gap" where computed)
    summary: dict


def run_recovery(objective, x0: LowRankIterate, T: int, *, eta: float, eps_schedule: EpsilonSchedule | None = None,
                 oracle=None, gap_every: int = 0, svd_subspace: int | None = None, block: int | None = None,
                 seed: int = 0, shadow: bool = False, dense_cap: int = 400) -> RecoveryRun:
    """T MEG steps on a QuadMeasObjective (deterministic, or mini-batch when `oracle` is a
    QuadMeasStochasticOracle): step t uses eta, eps_{t+1}, svd_seed = t; row t logs f(tau X_{t+1}),
    the cheap certificate and lambda_{r+1} of the step and its wall time; every `gap_every` rows
    (and at the end) the dual gap of X_{t+1}.

    shadow=True is the spec's lockstep / dense-shadow mode (n <= dense_cap): the
    full certificate from the whole spectrum of log X_t - eta grad (shadow_lowrank_step +
    certificate_full, meg.py:240-262, 367-385) and B(W_{t+1}, X_{t+1}) against the exact MEG
    sequence W_{t+1} = exact_meg_step(W_t, grad(W_t), eta) from W_0 = X_0 (Fig. 1-2; entropy.py:128-142);
    the elapsed time then covers only the low-rank step."""
    import time

    from .meg import certificate_full, lowrank_meg_step

    if shadow:
        from . import shadow as sh

        if x0.n > dense_cap:
            raise ParameterError(f"dense shadow allowed only for n <= {dense_cap}, got n={x0.n}")
        if oracle is not None:
            raise ParameterError("the lockstep shadow follows the deterministic gradient (oracle must be None)")
        W = x0.densify() if hasattr(x0, "densify") else None
    eps_schedule = eps_schedule or EpsilonSchedule.experiment(10.0)
    rows = []
    x = x0
    for t in range(int(T)):
        t0 = time.perf_counter_ns()
        g = oracle.grad_operator(x, oracle.sample_batch()) if oracle is not None else objective.grad_operator(x)
        eps_next = eps_schedule.eval(t + 1)
        res = lowrank_meg_step(x, g, float(eta), eps_next, svd_seed=t, svd_subspace=svd_subspace,
                               block=block)
        elapsed = time.perf_counter_ns() - t0
        row = {"t": t + 1, "f_value": objective.value(res.iterate), "eps_t": float(res.iterate.eps),
               "eta_t": float(eta), "cert_cheap_lhs": float(res.cert.lhs_cheap),
               "cert_cheap_holds": int(res.cert.holds_cheap), "cert_full_lhs": None, "cert_full_holds": None,
               "bregman_to_exact": None, "lambda_rsp1": float(res.lambda_r_plus_1), "elapsed_ns": elapsed}
        if shadow:
            _, _, yfull = sh.shadow_lowrank_step(x.densify(), g.dense, float(eta), eps_next, x.r)
            cf = certificate_full(yfull.cpu().numpy(), eps_next, x.n, x.r, iteration=t)
            W = sh.exact_meg_step(W, objective.gradient_dense(W), float(eta))
            row["cert_full_lhs"] = float(cf.lhs_full)
            row["cert_full_holds"] = int(cf.holds_full)
            row["bregman_to_exact"] = float(sh.bregman_structured(W, res.iterate))
        x = res.iterate
        if gap_every and ((t + 1) % gap_every == 0 or t + 1 == T):
            row["dual_gap"] = objective.dual_gap(x, seed=seed)
        rows.append(row)
    holds = [r["t"] for r in rows if r["cert_cheap_holds"]]
    summary = {"T": int(T), "f_final": rows[-1]["f_value"] if rows else objective.value(x0),
               "first_iter_cert_cheap": holds[0] if holds else -1}
    if shadow:
        holds_full = [r["t"] for r in rows if r["cert_full_holds"]]
        summary["first_iter_cert_full"] = holds_full[0] if holds_full else -1
    gaps = [r["dual_gap"] for r in rows if "dual_gap" in r]
    if gaps:
        summary["dual_gap"] = gaps[-1]
    return RecoveryRun(iterate=x, rows=rows, summary=summary)


def emit_metrics(run: RecoveryRun, path: str) -> None:
    """SPEC.md harness emit_metrics: the exact header row, one row per iteration (17 significant
    digits, empty cells for absent fields), the summary as trailing `# key = value` comments."""
    cols = RUN_CSV_HEADER.split(",")

    def fmt(v):
        if v is None:
            return ""
        if isinstance(v, (int, np.integer)):
            return str(int(v))
        return repr(float(v)) if np.isfinite(v) else ("-inf" if v < 0 else "inf" if v > 0 else "nan")

    try:
        with open(path, "w") as fh:
            fh.write(RUN_CSV_HEADER + "\n")
            for r in run.rows:
                fh.write(",".join(fmt(r.get(c)) for c in cols) + "\n")
            for k, v in run.summary.items():
                fh.write(f"# {k} = {fmt(v)}\n")
    except OSError as e:
        raise OSError(f"{path}: {e}") from e
