"""Numpy objectives and trajectory driver for the oracle -- TEST INFRASTRUCTURE ONLY.

The objectives are plain `grad_apply` callables, the boundary the reference
step consumes (meg.py:327-335, example `frobenius_objective`
test_meg.py:28-35 used as `lambda u: g @ u` at :153).  The dense driver is
the factored "lean" driver of SURVEY.md section 6: X u from the factors
minus M u.  The driver `run_trajectory` works with any module exposing the
reference step API (the oracle port, or the reference itself when the
golden fixtures are generated).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import inputs


def x_apply(x, u: np.ndarray) -> np.ndarray:
    """X u for a structured iterate, from its factors (meg.py:84-87 without densifying)."""
    tail = x.eps / (x.n - x.r)
    coeff = (1.0 - x.eps) * x.lam - tail
    c = x.V.T @ u
    c = c * (coeff if u.ndim == 1 else coeff[:, None])
    return x.V @ c + tail * u


def x_entries(x, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """X_ij at the listed positions, from the factors."""
    tail = x.eps / (x.n - x.r)
    coeff = (1.0 - x.eps) * x.lam - tail
    vals = np.einsum("ik,k,ik->i", x.V[rows], coeff, x.V[cols])
    return vals + tail * (rows == cols)


def frob_value(x, m: np.ndarray, m_norm2: float | None = None, mv: np.ndarray | None = None) -> float:
    """1/2 ||X - M||_F^2 from the factors: needs M V."""
    n, r = x.n, x.r
    tail = x.eps / (n - r)
    kept = (1.0 - x.eps) * x.lam
    coeff = kept - tail
    if mv is None:
        mv = m @ x.V
    x_norm2 = float(np.sum(kept**2) + tail**2 * (n - r))
    inner = float(np.sum(coeff * np.einsum("ik,ik->k", x.V, mv)) + tail * np.trace(m))
    if m_norm2 is None:
        m_norm2 = float(np.sum(m * m))
    return 0.5 * (x_norm2 - 2.0 * inner + m_norm2)


def x_rows(x, i0: int, i1: int) -> np.ndarray:
    """Rows i0:i1 of the dense X from its factors (row-chunked densify, meg.py:84-87)."""
    tail = x.eps / (x.n - x.r)
    coeff = (1.0 - x.eps) * x.lam - tail
    rows = (x.V[i0:i1] * coeff) @ x.V.T
    rows[np.arange(i1 - i0), np.arange(i0, i1)] += tail
    return rows


def frob_value_direct(x, m: np.ndarray, chunk: int = 1024) -> float:
    """1/2 sum_ij (X_ij - M_ij)^2 summed entry by entry (no cancellation between the
    1/2(||X||^2 - 2<X,M> + ||M||^2) summands), row chunks of X from the factors."""
    total = 0.0
    for i0 in range(0, x.n, chunk):
        i1 = min(x.n, i0 + chunk)
        d = x_rows(x, i0, i1) - m[i0:i1]
        total += float(np.einsum("ij,ij->", d, d))
    return 0.5 * total


class DenseFrobenius:
    """f(X) = 1/2 ||X - M||_F^2; grad f(X) u = X u - M u."""

    def __init__(self, m: np.ndarray):
        self.m = np.ascontiguousarray(m, dtype=np.float64)
        self.n = self.m.shape[0]
        self.m_norm2 = float(np.sum(self.m * self.m))

    def grad_apply(self, x, t: int = 0):
        m = self.m
        return lambda u: x_apply(x, u) - m @ u

    def value(self, x) -> float:
        return frob_value(x, self.m, self.m_norm2)

    def value_direct(self, x) -> float:
        return frob_value_direct(x, self.m)

    def init_apply(self):
        m = self.m
        return lambda u: m @ u


class SampledEntries:
    """f(X) = 1/2 sum_{(i,j) in Omega} (X_ij - Mobs_ij)^2; grad = P_Omega(X - Mobs)."""

    def __init__(self, inst: inputs.SampledInstance, p: float):
        self.inst = inst
        self.n = inst.n
        counts = np.diff(inst.rowptr.astype(np.int64))
        self.rows = np.repeat(np.arange(inst.n), counts)
        self.cols = inst.col.astype(np.int64)
        self.p = p

    def _grad_matrix(self, x):
        vals = x_entries(x, self.rows, self.cols) - self.inst.obs
        return sp.csr_matrix((vals, self.inst.col, self.inst.rowptr), shape=(self.n, self.n))

    def grad_apply(self, x, t: int = 0):
        g = self._grad_matrix(x)
        return lambda u: g @ u

    def value(self, x) -> float:
        d = x_entries(x, self.rows, self.cols) - self.inst.obs
        return 0.5 * float(d @ d)

    def init_apply(self):
        """Spectral init operator (1/p) P_Omega(Mobs)."""
        g = sp.csr_matrix((self.inst.obs / self.p, self.inst.col, self.inst.rowptr), shape=(self.n, self.n))
        return lambda u: g @ u


class StochasticFrobenius(DenseFrobenius):
    """grad estimate (X - M) + sigma((1/b) A_t A_t^T - I/n), A_t from `inputs.minibatch`."""

    def __init__(self, m: np.ndarray, cfg: inputs.MegConfig):
        super().__init__(m)
        self.cfg = cfg

    def grad_apply(self, x, t: int = 0):
        m, cfg = self.m, self.cfg
        a = inputs.minibatch(cfg, t)
        s, b, n = cfg.sigma, cfg.batch, cfg.n
        return lambda u: x_apply(x, u) - m @ u + s * (a @ (a.T @ u) / b - u / n)


def make_objective(cfg: inputs.MegConfig):
    if cfg.kind == "dense":
        return DenseFrobenius(inputs.dense_target(cfg))
    if cfg.kind == "sampled":
        return SampledEntries(inputs.sampled_instance(cfg, keep_planted=False), cfg.sample_p)
    if cfg.kind == "stochastic":
        return StochasticFrobenius(inputs.dense_target(cfg), cfg)
    raise ValueError(cfg.kind)


def initial_iterate(api, cfg: inputs.MegConfig, obj):
    """Warm start: top-r eigenpairs of M (or (1/p) P_Omega Mobs), simplex weights,
    warm_start_wrap with eps0 = schedule(0)."""
    op = api.SymmetricOperator(cfg.n, obj.init_apply())
    top = api.lanczos_top_r(op, cfg.r, seed=cfg.seed, subspace=64)
    w = api.project_simplex(np.asarray(top.eigenvalues, dtype=float), 1.0)
    w = w / w.sum()
    w = np.maximum(w, 1e-12)
    w = w / w.sum()
    return api.warm_start_wrap(top.eigenvectors, w, cfg.eps(0))


def probes(n: int, k: int = 2, seed: int = 99) -> np.ndarray:
    key = inputs.stream_key(seed, 7)
    return inputs.gaussian(key, np.arange(n * k, dtype=np.uint64)).reshape(n, k) / math.sqrt(n)


def run_trajectory(api, cfg: inputs.MegConfig, obj, x0, iters: int, probe_at=(), step_kwargs=None):
    """Drive `api.lowrank_meg_step` for `iters` iterations from x0 (driver of test_meg.py:150-156).

    Iteration t uses eta_t = cfg.eta(t), eps_next = cfg.eps(t + 1), svd_seed = t.
    Records per iteration: shift, y (r+1), lam, eps, lhs_cheap, f(X_{t+1});
    at iterations in `probe_at`, X_{t+1} Z for a fixed probe block Z.
    """
    step_kwargs = dict(step_kwargs or {})
    z = probes(cfg.n)
    rec = {k: [] for k in ("shift", "y", "lam", "eps", "lhs", "f")}
    if hasattr(obj, "value_direct"):
        rec["f_direct"] = []
    probe = {}
    x = x0
    for t in range(iters):
        res = api.lowrank_meg_step(
            x, obj.grad_apply(x, t), cfg.eta(t), cfg.eps(t + 1),
            svd_tol=1e-10, svd_seed=t, svd_subspace=cfg.subspace, **step_kwargs,
        )
        x = res.iterate
        rec["shift"].append(res.shift)
        rec["y"].append(np.asarray(res.top_eigenvalues))
        rec["lam"].append(np.asarray(x.lam))
        rec["eps"].append(x.eps)
        rec["lhs"].append(res.cert.lhs_cheap)
        rec["f"].append(obj.value(x))
        if "f_direct" in rec:
            rec["f_direct"].append(obj.value_direct(x))
        if t in probe_at:
            probe[t] = x_apply(x, z)
    out = {k: np.asarray(v) for k, v in rec.items()}
    for t, v in probe.items():
        out[f"probe_{t}"] = v
    return out, x
