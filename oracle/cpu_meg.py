"""Numpy restatement of the reference low-rank MEG step -- TEST INFRASTRUCTURE ONLY.

Every public function names the reference lines it restates.  Reference root:
`/root/reference/pkg/src/specmeg/` (files `linalg.py`, `meg.py`).  The
restatement keeps the reference's numerical recipe (full-reorthogonalisation
Lanczos, CGS2, Rayleigh-Ritz through cached images, thick restart, max-shift
exponentiation, cheap certificate) so converged outputs agree with the
reference to rounding; tests/test_oracle_pins.py pins it against fixtures
produced by the reference itself.

Implementation differences that do not change the converged result:
the Krylov basis lives in a preallocated (n, m + 1) buffer instead of being
re-stacked with `np.column_stack` on every application.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np


# ---------------------------------------------------------------------------
# error types -- linalg.py:23-52


class ParameterError(ValueError):
    """Structurally invalid argument (linalg.py:23-24)."""


class EighError(RuntimeError):
    """Dense eigendecomposition failure (linalg.py:27-28)."""


class LanczosError(RuntimeError):
    """Residual tolerance not reached; carries best residuals (linalg.py:43-52)."""

    def __init__(self, message: str, residual_norms: np.ndarray):
        self.residual_norms = residual_norms
        super().__init__(message)


def symmetrize(a) -> np.ndarray:
    """(A + A^T)/2 in float64 (linalg.py:55-60)."""
    a = np.asarray(a, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ParameterError(f"expected a square matrix, got shape {a.shape}")
    return 0.5 * (a + a.T)


@dataclass(frozen=True)
class TopREigen:
    """Top-r eigenpairs, eigenvalues non-increasing (linalg.py:71-78)."""

    r: int
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    residual_norms: np.ndarray


class SymmetricOperator:
    """Symmetric map given by block application (linalg.py:81-103)."""

    def __init__(self, dim: int, apply_fn: Callable[[np.ndarray], np.ndarray]):
        self.dim = int(dim)
        self._fn = apply_fn

    def apply(self, u: np.ndarray) -> np.ndarray:
        return self._fn(u)

    @classmethod
    def from_dense(cls, a) -> "SymmetricOperator":
        s = symmetrize(a)
        return cls(s.shape[0], lambda u: s @ u)

    def to_dense(self) -> np.ndarray:
        return symmetrize(self.apply(np.eye(self.dim)))


def full_eigh(a):
    """Full spectrum, sorted non-increasing (linalg.py:106-119)."""
    s = symmetrize(a)
    try:
        w, v = np.linalg.eigh(s)
    except np.linalg.LinAlgError as exc:  # pragma: no cover - LAPACK failure
        raise EighError(str(exc)) from exc
    idx = np.argsort(-w, kind="stable")
    return w[idx], v[:, idx]


def _cgs2(q: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Classical Gram-Schmidt applied twice against span(q) (linalg.py:122-127)."""
    if q.shape[1]:
        for _ in range(2):
            v = v - q @ (q.T @ v)
    return v


class _Krylov:
    """Basis/image store for `lanczos_top_r` (replaces linalg.py:164-180 stacking)."""

    def __init__(self, op: SymmetricOperator, cap: int):
        n = op.dim
        self.op = op
        self.q = np.zeros((n, cap))
        self.aq = np.zeros((n, cap))
        self.size = 0
        self.applies = 0

    @property
    def basis(self) -> np.ndarray:
        return self.q[:, : self.size]

    @property
    def images(self) -> np.ndarray:
        return self.aq[:, : self.size]

    def push(self, v: np.ndarray) -> None:
        self.q[:, self.size] = v
        self.aq[:, self.size] = self.op.apply(v)
        self.size += 1
        self.applies += 1

    def reset(self, q: np.ndarray, aq: np.ndarray) -> None:
        k = q.shape[1]
        self.q[:, :k] = q
        self.aq[:, :k] = aq
        self.size = k


def lanczos_top_r(
    op: SymmetricOperator,
    r: int,
    tol: float = 1e-10,
    max_iter: int | None = None,
    seed: int = 0,
    subspace: int | None = None,
    restarts: int = 12,
) -> TopREigen:
    """Algebraically largest r eigenpairs (linalg.py:130-241).

    Basis size m = min(n, max(2r+10, 30)) unless given (:158-159); budget
    restarts*m applications (:160-161); random unit start from
    default_rng(seed) (:162, :168-174); Krylov expansion with CGS2 and
    breakdown restart (:189-201); Rayleigh-Ritz on cached images
    (:205-211); convergence iff every residual <= tol*max(1, max|theta_all|)
    (:214-216); thick restart keeping r+2 Ritz vectors and continuing from
    the orthogonalised image of the worst one (:220-235); LanczosError with
    the best residuals otherwise (:237-241).
    """
    n = op.dim
    if not 1 <= r < n:
        raise ParameterError(f"need 1 <= r < n, got r={r}, n={n}")
    m = subspace if subspace is not None else min(n, max(2 * r + 10, 30))
    m = min(n, max(m, r + 1))
    budget = restarts * m if max_iter is None else max_iter
    rng = np.random.default_rng(seed)
    ks = _Krylov(op, m + 1)

    def random_direction():
        for _ in range(20):
            v = _cgs2(ks.basis, rng.standard_normal(n))
            nv = np.linalg.norm(v)
            if nv > 1e-8 * np.sqrt(n):
                return v / nv
        return None

    start = random_direction()
    assert start is not None
    ks.push(start)
    best = np.full(r, np.inf)
    for _ in range(restarts):
        while ks.size < m and ks.applies < budget + 1:
            w = _cgs2(ks.basis, ks.images[:, -1].copy())
            nw = np.linalg.norm(w)
            if nw <= 1e-13 * max(1.0, float(np.abs(ks.images).max())):
                if ks.size >= n:
                    break
                fresh = random_direction()
                if fresh is None:
                    break
                ks.push(fresh)
            else:
                ks.push(w / nw)
        basis, images = ks.basis, ks.images
        theta_all, s = np.linalg.eigh(symmetrize(basis.T @ images))
        order = np.argsort(-theta_all, kind="stable")
        top = order[:r]
        theta = theta_all[top]
        vecs = basis @ s[:, top]
        resid = np.linalg.norm(images @ s[:, top] - vecs * theta, axis=0)
        if resid.max() < best.max():
            best = resid
        scale = max(1.0, float(np.abs(theta_all).max()))
        if np.all(resid <= tol * scale) or ks.size >= n:
            return TopREigen(r=r, eigenvalues=theta, eigenvectors=vecs, residual_norms=resid)
        if ks.applies >= budget:
            break
        keep = order[: min(ks.size, r + 2)]
        ks.reset(basis @ s[:, keep], images @ s[:, keep])
        worst = int(np.argmax(resid))
        w = _cgs2(ks.basis, ks.images[:, worst].copy())
        nw = np.linalg.norm(w)
        if nw > 1e-13 * max(1.0, float(np.abs(ks.images).max())):
            ks.push(w / nw)
        else:
            fresh = random_direction()
            if fresh is None:
                break
            ks.push(fresh)
    raise LanczosError(
        f"residual tolerance {tol:g} not reached after {ks.applies} applications",
        residual_norms=best,
    )


def project_simplex(z, tau: float = 1.0) -> np.ndarray:
    """Euclidean projection onto {w >= 0, sum w = tau} (linalg.py:244-261)."""
    z = np.asarray(z, dtype=float).ravel()
    if z.size < 1:
        raise ParameterError("need at least one coordinate")
    if not tau > 0:
        raise ParameterError(f"tau must be positive, got {tau}")
    srt = np.sort(z)[::-1]
    csum = np.cumsum(srt)
    cand = (csum - tau) / np.arange(1, z.size + 1)
    k = int(np.flatnonzero(srt - cand > 0).max()) + 1
    return np.maximum(z - (csum[k - 1] - tau) / k, 0.0)


# ---------------------------------------------------------------------------
# iterate, schedules, certificates -- meg.py


@dataclass(frozen=True)
class LowRankIterate:
    """(1-eps) V diag(lam) V^T + eps/(n-r)(I - V V^T) (meg.py:47-92)."""

    n: int
    r: int
    V: np.ndarray
    lam: np.ndarray
    eps: float
    warm: object = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        if not 1 <= self.r < self.n:
            raise ParameterError(f"need 1 <= r < n, got r={self.r}, n={self.n}")
        if self.V.shape != (self.n, self.r):
            raise ParameterError(f"V must be {self.n}x{self.r}, got {self.V.shape}")
        if not 0 < self.eps <= 0.75:
            raise ParameterError(f"eps must lie in (0, 3/4], got {self.eps}")
        err = float(np.max(np.abs(self.V.T @ self.V - np.eye(self.r))))
        if err > 1e-10:
            raise ParameterError(f"V columns not orthonormal (error {err:.3e})")
        if abs(self.lam.sum() - 1.0) > 1e-10:
            raise ParameterError(f"lam must sum to 1, got {self.lam.sum()!r}")
        if np.any(np.diff(self.lam) > 0):
            raise ParameterError("lam must be sorted non-increasing")
        if not self.lam[-1] > 0:
            raise ParameterError("lam must be strictly positive")

    @property
    def tail_value(self) -> float:
        return self.eps / (self.n - self.r)

    def densify(self) -> np.ndarray:
        coeff = (1.0 - self.eps) * self.lam - self.tail_value
        return symmetrize((self.V * coeff) @ self.V.T + self.tail_value * np.eye(self.n))

    def eigenvalues_full(self) -> np.ndarray:
        vals = np.concatenate([(1.0 - self.eps) * self.lam, np.full(self.n - self.r, self.tail_value)])
        return np.sort(vals)[::-1]

    def apply(self, u: np.ndarray) -> np.ndarray:
        """X u from the factors (the factored driver of SURVEY.md section 6)."""
        coeff = (1.0 - self.eps) * self.lam - self.tail_value
        c = self.V.T @ u
        c = c * (coeff if u.ndim == 1 else coeff[:, None])
        return self.V @ c + self.tail_value * u


@dataclass(frozen=True)
class EpsilonSchedule:
    """Complement-mass schedules, clamped to 3/4 (meg.py:114-197)."""

    kind: str
    eps0_tilde: float = 0.0
    G: float = 0.0
    c: float = 0.0

    @classmethod
    def experiment(cls, c: float = 10.0) -> "EpsilonSchedule":
        return cls(kind="experiment", c=c)

    @classmethod
    def cubic_det(cls, eps0_tilde, G, c):
        return cls(kind="cubic_det", eps0_tilde=eps0_tilde, G=G, c=c)

    @classmethod
    def cubic_det_general(cls, eps0_tilde, G, c):
        return cls(kind="cubic_det_general", eps0_tilde=eps0_tilde, G=G, c=c)

    @classmethod
    def quadratic_stoch(cls, eps0_tilde, c):
        return cls(kind="quadratic_stoch", eps0_tilde=eps0_tilde, c=c)

    def eval(self, t: int) -> float:
        g2 = max(self.G**2, 1.0)
        if self.kind == "cubic_det":
            raw = self.eps0_tilde / (2.0 * g2) / (t + 1 + self.c) ** 3
        elif self.kind == "cubic_det_general":
            raw = 3.0 * self.eps0_tilde / (2.0 * g2) / (t + self.c + 1) ** 3
        elif self.kind == "quadratic_stoch":
            raw = (9.0 / 32.0) * self.eps0_tilde / (t + self.c + 1) ** 2
        elif self.kind == "experiment":
            raw = 0.6 / (t + self.c + 1) ** 2
        else:
            raise ParameterError(f"unknown epsilon schedule {self.kind!r}")
        return min(raw, 0.75)


@dataclass(frozen=True)
class CertificateRecord:
    """Certificate evaluation against threshold 2 eps (meg.py:204-219)."""

    iteration: int | None
    lhs_cheap: float
    holds_cheap: bool
    threshold: float
    lhs_full: float | None = None
    holds_full: bool | None = None


def _cert_lhs(lam_rp1: float, b: float, eps: float, n: int, r: int) -> float:
    """log((n-r) lambda_{r+1} / (eps b)) (meg.py:222-229)."""
    if not b > 0:
        raise ParameterError(f"partial trace must be positive, got {b}")
    if lam_rp1 < 0:
        raise ParameterError(f"lambda_(r+1) must be non-negative, got {lam_rp1}")
    if lam_rp1 == 0.0:
        return -math.inf
    return math.log((n - r) * lam_rp1 / (eps * b))


def certificate_cheap(lambda_r_plus_1, b_r_plus_1, eps, n, r, iteration=None) -> CertificateRecord:
    """Cheap certificate from the top r+1 eigenvalues (meg.py:232-239)."""
    lhs = _cert_lhs(lambda_r_plus_1, b_r_plus_1, eps, n, r)
    return CertificateRecord(iteration=iteration, lhs_cheap=lhs, holds_cheap=lhs <= 2.0 * eps, threshold=2.0 * eps)


def certificate_full(y_spectrum, eps, n, r, iteration=None) -> CertificateRecord:
    """Full certificate from the whole exponential spectrum (meg.py:242-262)."""
    y = np.sort(np.asarray(y_spectrum, dtype=float))[::-1]
    if y.size != n:
        raise ParameterError(f"expected a full spectrum of length {n}, got {y.size}")
    full = _cert_lhs(float(y[r]), float(y.sum()), eps, n, r)
    cheap = _cert_lhs(float(y[r]), float(y[: r + 1].sum()), eps, n, r)
    return CertificateRecord(iteration, cheap, cheap <= 2.0 * eps, 2.0 * eps, full, full <= 2.0 * eps)


# ---------------------------------------------------------------------------
# the step -- meg.py:287-364


def logmap_operator(x: LowRankIterate, grad_apply, eta: float) -> SymmetricOperator:
    """u -> (log X - eta grad) u, matrix-free (meg.py:287-307)."""
    lk = np.log((1.0 - x.eps) * x.lam)
    lt = math.log(x.tail_value)

    def apply(u):
        c = x.V.T @ u
        kept = x.V @ ((lk if u.ndim == 1 else lk[:, None]) * c)
        return kept + lt * (u - x.V @ c) - eta * grad_apply(u)

    return SymmetricOperator(x.n, apply)


@dataclass(frozen=True)
class LowRankStepResult:
    """Step outputs (meg.py:310-324); top_eigenvalues holds y = exp(mu - mu_1)."""

    iterate: LowRankIterate
    cert: CertificateRecord
    lambda_r_plus_1: float
    b_r_plus_1: float
    shift: float
    top_eigenvalues: np.ndarray | None = field(repr=False, default=None)
    mu: np.ndarray | None = field(repr=False, default=None)
    residual_norms: np.ndarray | None = field(repr=False, default=None)


def lowrank_meg_step(
    x: LowRankIterate,
    grad_apply,
    eta: float,
    eps_next: float,
    svd_tol: float = 1e-10,
    svd_seed: int = 0,
    svd_subspace: int | None = None,
) -> LowRankStepResult:
    """One low-rank MEG update (meg.py:327-364; Algorithm 2)."""
    if not 0 < eps_next <= 0.75:
        raise ParameterError(f"eps_next must lie in (0, 3/4], got {eps_next}")
    top = lanczos_top_r(logmap_operator(x, grad_apply, eta), x.r + 1, tol=svd_tol, seed=svd_seed, subspace=svd_subspace)
    mu = top.eigenvalues
    shift = float(mu[0])
    y = np.exp(mu - shift)
    kept = float(y[: x.r].sum())
    assert kept > 1e-290, "kept mass vanished despite max-shift"
    lam = y[: x.r] / kept
    lam = lam / lam.sum()
    nxt = LowRankIterate(n=x.n, r=x.r, V=top.eigenvectors[:, : x.r], lam=lam, eps=eps_next)
    lam_rp1, b_rp1 = float(y[x.r]), float(y.sum())
    return LowRankStepResult(
        iterate=nxt,
        cert=certificate_cheap(lam_rp1, b_rp1, eps_next, x.n, x.r),
        lambda_r_plus_1=lam_rp1,
        b_r_plus_1=b_rp1,
        shift=shift,
        top_eigenvalues=y,
        mu=mu,
        residual_norms=top.residual_norms,
    )


def shadow_lowrank_step(x_dense, grad_dense, eta, eps_next, r):
    """Dense recomputation via two full eighs (meg.py:367-385).  Test oracle only."""
    w, v = full_eigh(x_dense)
    log_x = (v * np.log(np.maximum(w, 1e-300))) @ v.T
    mu, ev = full_eigh(symmetrize(log_x - eta * grad_dense))
    y = np.exp(mu - mu[0])
    n = x_dense.shape[0]
    exact = symmetrize((ev * (y / y.sum())) @ ev.T)
    kept = ev[:, :r]
    low = (1.0 - eps_next) * (kept * (y[:r] / y[:r].sum())) @ kept.T
    low += eps_next / (n - r) * (np.eye(n) - kept @ kept.T)
    return symmetrize(low), exact, y


def warm_start_wrap(V0, lam0, eps0) -> LowRankIterate:
    """(1-eps0) V0 diag(lam0) V0^T + eps0/n I in canonical form (meg.py:392-411)."""
    if not 0 < eps0 <= 0.75:
        raise ParameterError(f"eps0 must lie in (0, 3/4], got {eps0}")
    V0 = np.asarray(V0, dtype=float)
    lam0 = np.asarray(lam0, dtype=float).ravel()
    n, r = V0.shape
    if abs(lam0.sum() - 1.0) > 1e-10 or not np.all(lam0 > 0):
        raise ParameterError("lam0 must be strictly positive and sum to 1")
    order = np.argsort(-lam0, kind="stable")
    lam0, V0 = lam0[order], V0[:, order]
    eps_p = eps0 * (n - r) / n
    lam = ((1.0 - eps0) * lam0 + eps0 / n) / (1.0 - eps_p)
    return LowRankIterate(n=n, r=r, V=V0, lam=lam / lam.sum(), eps=eps_p)


def init_weights_from_top_eigs(top_eigs, tau: float = 1.0, floor: float = 1e-12) -> np.ndarray:
    """Simplex projection, floor, renormalise (objectives.py:312-317 pattern)."""
    w = project_simplex(np.asarray(top_eigs, dtype=float), tau)
    w = w / w.sum()
    w = np.maximum(w, floor)
    return w / w.sum()


def dual_gap_core(grad: np.ndarray, trace_term: float, tau: float = 1.0, seed: int = 0) -> float:
    """Tr(X grad) - tau lambda_min(grad) via the top eigenpair of -grad (objectives.py:332-335)."""
    top = lanczos_top_r(SymmetricOperator.from_dense(-grad), 1, seed=seed)
    v = top.eigenvectors[:, 0]
    return trace_term - tau * float(v @ grad @ v)


# ---------------------------------------------------------------------------
# dense-shadow diagnostics -- test oracle only


def exact_meg_step(z, grad, eta):
    """exp(log Z - eta grad) / trace (meg.py:269-284)."""
    w, v = full_eigh(z)
    if w[-1] <= 0:
        raise ParameterError(f"iterate must be positive definite, min eigenvalue {w[-1]:.3e}")
    log_z = (v * np.log(w)) @ v.T
    mu, ev = full_eigh(symmetrize(log_z - eta * np.asarray(grad, dtype=float)))
    y = np.exp(mu - mu[0])
    y /= y.sum()
    return symmetrize((ev * y) @ ev.T)


EIG_CLAMP = 1e-300  # entropy.py:21
MASS_TOL = 1e-14  # entropy.py:22


def entropy_sum(w):
    """sum lambda log lambda, 0 log 0 = 0 (entropy.py:54-58)."""
    w = np.maximum(w, 0.0)
    m = w > EIG_CLAMP
    return float(np.sum(w[m] * np.log(w[m])))


def bregman(x, y):
    """(value, finite, clamped) of Tr(X log X - X log Y) (entropy.py:76-96)."""
    x, y = symmetrize(x), symmetrize(y)
    wx, _ = full_eigh(x)
    wy, vy = full_eigh(y)
    mass = np.einsum("ij,ji->i", vy.T @ x, vy)
    heavy = mass > MASS_TOL
    if np.any(heavy & (wy <= 0.0)):
        return math.inf, False, True
    clamped = bool(np.any(heavy & (wy <= EIG_CLAMP)))
    cross = float(np.sum(mass * np.log(np.maximum(wy, EIG_CLAMP))))
    return entropy_sum(wx) - cross, True, clamped


def structured_log_trace(x, y):
    """Tr(X log Y), Y structured; X dense or structured (entropy.py:108-125)."""
    log_kept = np.log((1.0 - y.eps) * y.lam)
    log_tail = math.log(y.eps / (y.n - y.r))
    if isinstance(x, np.ndarray):
        mass = np.einsum("ij,ij->j", y.V, x @ y.V)
        trace_x = float(np.trace(x))
    else:
        sq = (x.V.T @ y.V) ** 2
        mass = (1.0 - x.eps) * (x.lam @ sq) + (x.eps / (x.n - x.r)) * (1.0 - sq.sum(axis=0))
        trace_x = 1.0
    return float(np.sum(mass * (log_kept - log_tail))) + log_tail * trace_x


def bregman_structured(x, y):
    """Tr(X log X - X log Y), Y structured (entropy.py:128-142)."""
    if isinstance(x, np.ndarray):
        own = entropy_sum(full_eigh(symmetrize(x))[0])
    else:
        kept = (1.0 - x.eps) * x.lam
        own = entropy_sum(kept) + x.eps * math.log(x.eps / (x.n - x.r))
    return own - structured_log_trace(x, y)
