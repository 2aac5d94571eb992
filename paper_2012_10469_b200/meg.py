"""Low-rank MEG step on the B200, mirroring `specmeg.meg` (meg.py:1-495) for the hot path.

Same names, arguments, return types and error behaviour as the reference:
`LowRankIterate`, `logmap_operator`, `lowrank_meg_step`, `LowRankStepResult`,
`CertificateRecord`, `certificate_cheap`, `warm_start_wrap`,
`EpsilonSchedule`, `StepConfig`.  The iterate's factor V lives in HBM
(float64 n x r); lam and eps are host scalars.  The step is one native call
(csrc/megb200_runtime.cu): it builds the matrix-free operator
log X - eta grad, extracts the top r + 1 eigenpairs with the block solver,
exponentiates with the max-shift and evaluates the cheap certificate on the
device.

Warm start: each step returns, inside the next iterate, the top Ritz block of
the operator it solved (`iterate.warm_block`).  The next step seeds its
Krylov block with it; without one it seeds with the iterate's own V.  Seeds
change only the number of passes, never the converged result (the
convergence rule is the reference's, linalg.py:214-215).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib, runtime
from .callbacks import checked
from .errors import ParameterError
from .linalg import SymmetricOperator, _eig_opts, symmetrize  # noqa: F401
from .objectives import GradientOperator


class LowRankIterate:
    """(1-eps) V diag(lam) V^T + eps/(n-r) (I - V V^T), stored as factors (meg.py:47-92).

    V may be given as numpy or torch; it is kept on the device
    (`V_device`).  `V` returns a host copy (numpy), like the reference field.
    Validation matches meg.py:62-77 (the V^T V check runs on the device).
    """

    __slots__ = ("n", "r", "lam", "eps", "_vd", "_vh", "warm_block", "warm_orth_err")

    def __init__(self, n: int, r: int, V, lam, eps: float, *, warm_block=None, warm_orth_err: float = 1.0,
                 _gram_err: float | None = None):
        n, r = int(n), int(r)
        if not 1 <= r < n:
            raise ParameterError(f"need 1 <= r < n, got r={r}, n={n}")
        shape = tuple(V.shape)
        if shape != (n, r):
            raise ParameterError(f"V must be {n}x{r}, got {shape}")
        if not 0 < eps <= 0.75:
            raise ParameterError(f"eps must lie in (0, 3/4], got {eps}")
        lam = np.array(lam, dtype=float).ravel()
        vd = runtime.as_device_f64(V)
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "r", r)
        object.__setattr__(self, "_vd", vd)
        object.__setattr__(self, "_vh", V.copy() if isinstance(V, np.ndarray) else None)
        object.__setattr__(self, "lam", lam)
        object.__setattr__(self, "eps", float(eps))
        object.__setattr__(self, "warm_block", warm_block)
        object.__setattr__(self, "warm_orth_err", float(warm_orth_err))
        if _gram_err is None:
            s = runtime.solver_for(n)
            err = C.c_double()
            runtime.check(s.lib.megb200_gram_error(s.handle, vd.data_ptr(), vd.stride(0), r, C.byref(err)))
            _gram_err = err.value
        if _gram_err > 1e-10:
            raise ParameterError(f"V columns not orthonormal (error {_gram_err:.3e})")
        if abs(lam.sum() - 1.0) > 1e-10:
            raise ParameterError(f"lam must sum to 1, got {lam.sum()!r}")
        if np.any(np.diff(lam) > 0):
            raise ParameterError("lam must be sorted non-increasing")
        if not lam[-1] > 0:
            raise ParameterError("lam must be strictly positive")

    def __setattr__(self, name, value):
        raise AttributeError("LowRankIterate is immutable")

    @property
    def V_device(self) -> torch.Tensor:
        return self._vd

    @property
    def V(self) -> np.ndarray:
        """Host copy of the factor (one device-to-host read, cached)."""
        if self._vh is None:
            object.__setattr__(self, "_vh", self._vd.cpu().numpy())
        return self._vh

    @property
    def tail_value(self) -> float:
        """The (n-r)-fold eigenvalue eps/(n-r) on the complement (meg.py:79-82)."""
        return self.eps / (self.n - self.r)

    def densify(self) -> np.ndarray:
        """Materialise the n x n matrix on the host.  Test and dense-shadow use only (meg.py:84-87)."""
        v = self.V
        kept = (v * ((1.0 - self.eps) * self.lam - self.tail_value)) @ v.T
        return symmetrize(kept + self.tail_value * np.eye(self.n))

    def eigenvalues_full(self) -> np.ndarray:
        vals = np.concatenate([(1.0 - self.eps) * self.lam, np.full(self.n - self.r, self.tail_value)])
        return np.sort(vals)[::-1]

    def struct(self, keep: list) -> _lib.Iterate:
        it = _lib.Iterate()
        lam = runtime.host_f64(self.lam)
        keep.append(lam)
        it.n, it.r = self.n, self.r
        it.V = self._vd.data_ptr()
        it.ldv = self._vd.stride(0)
        it.lam = _lib.dptr(lam)
        it.eps = self.eps
        return it


def dense_iterate(x):  # pragma: no cover - API parity; exact-step path is out of scope
    raise NotImplementedError("the dense exact step (meg.py:95-107, 269-284) is an O(n^3) oracle, out of scope")


# ---------------------------------------------------------------------------
# schedules (meg.py:114-197) -- host scalars


@dataclass(frozen=True)
class StepConfig:
    """Step-size rule; all supported rules evaluate to a constant eta (meg.py:114-150)."""

    kind: str
    eta: float = 0.0
    beta: float = 0.0
    R0: float = 0.0
    G: float = 0.0
    T: int = 0

    @classmethod
    def fixed(cls, eta: float) -> "StepConfig":
        if not eta > 0:
            raise ParameterError(f"eta must be positive, got {eta}")
        return cls(kind="fixed", eta=eta)

    @classmethod
    def one_over_beta(cls, beta: float) -> "StepConfig":
        if not beta > 0:
            raise ParameterError(f"beta must be positive, got {beta}")
        return cls(kind="one_over_beta", beta=beta)

    @classmethod
    def stochastic_fixed(cls, R0: float, G: float, T: int) -> "StepConfig":
        if not (R0 > 0 and G > 0 and T >= 1):
            raise ParameterError(f"need R0 > 0, G > 0, T >= 1, got {R0}, {G}, {T}")
        return cls(kind="stochastic_fixed", R0=R0, G=G, T=T)

    def eval(self, t: int) -> float:
        if self.kind == "fixed":
            return self.eta
        if self.kind == "one_over_beta":
            return 1.0 / self.beta
        if self.kind == "stochastic_fixed":
            return self.R0 / (2.0 * self.G * math.sqrt(self.T))
        raise ParameterError(f"unknown step rule {self.kind!r}")


def step_eval(config: StepConfig, t: int) -> float:
    return config.eval(t)


@dataclass(frozen=True)
class EpsilonSchedule:
    """Complement-mass schedule eps_t clamped into (0, 3/4] (meg.py:153-197)."""

    kind: str
    eps0_tilde: float = 0.0
    G: float = 0.0
    c: float = 0.0

    @classmethod
    def cubic_det(cls, eps0_tilde: float, G: float, c: float) -> "EpsilonSchedule":
        return cls(kind="cubic_det", eps0_tilde=eps0_tilde, G=G, c=c)

    @classmethod
    def cubic_det_general(cls, eps0_tilde: float, G: float, c: float) -> "EpsilonSchedule":
        return cls(kind="cubic_det_general", eps0_tilde=eps0_tilde, G=G, c=c)

    @classmethod
    def quadratic_stoch(cls, eps0_tilde: float, c: float) -> "EpsilonSchedule":
        return cls(kind="quadratic_stoch", eps0_tilde=eps0_tilde, c=c)

    @classmethod
    def experiment(cls, c: float = 10.0) -> "EpsilonSchedule":
        return cls(kind="experiment", c=c)

    def eval(self, t: int) -> float:
        g2 = max(self.G**2, 1.0)
        if self.kind == "cubic_det":
            raw = self.eps0_tilde / (2.0 * g2) / (t + 1 + self.c) ** 3
        elif self.kind == "cubic_det_general":
            raw = 3.0 * self.eps0_tilde / (2.0 * g2) / (t + self.c + 1) ** 3
        elif self.kind == "quadratic_stoch":
            raw = (9.0 / 32.0) * self.eps0_tilde / (t + self.c + 1) ** 2
        elif self.kind == "experiment":
            raw = (3.0 / 5.0) / (t + self.c + 1) ** 2
        else:
            raise ParameterError(f"unknown epsilon schedule {self.kind!r}")
        return min(raw, 0.75)


def eps_schedule_eval(schedule: EpsilonSchedule, t: int) -> float:
    return schedule.eval(t)


# ---------------------------------------------------------------------------
# certificates (meg.py:200-262)


@dataclass(frozen=True)
class CertificateRecord:
    """One step's certificate against the threshold 2 eps (meg.py:204-219)."""

    iteration: int | None
    lhs_cheap: float
    holds_cheap: bool
    threshold: float
    lhs_full: float | None = None
    holds_full: bool | None = None


def certificate_cheap(lambda_r_plus_1: float, b_r_plus_1: float, eps: float, n: int, r: int,
                      iteration: int | None = None) -> CertificateRecord:
    """log((n-r) lambda_{r+1} / (eps b)) <= 2 eps from the top r+1 eigenvalues (meg.py:222-239)."""
    lib = _lib.load()
    lhs, holds, thr = C.c_double(), C.c_int32(), C.c_double()
    runtime.check(lib.megb200_certificate_cheap(float(lambda_r_plus_1), float(b_r_plus_1), float(eps), int(n), int(r),
                                                C.byref(lhs), C.byref(holds), C.byref(thr)))
    return CertificateRecord(iteration=iteration, lhs_cheap=lhs.value, holds_cheap=bool(holds.value),
                             threshold=thr.value)


def certificate_full(y_spectrum, eps: float, n: int, r: int, iteration: int | None = None) -> CertificateRecord:
    """Both certificate sides from a full exponential spectrum (meg.py:242-262; shadow mode, host arithmetic)."""
    y = np.sort(np.asarray(y_spectrum, dtype=float))[::-1]
    if y.size != n:
        raise ParameterError(f"expected a full spectrum of length {n}, got {y.size}")
    full = certificate_cheap(float(y[r]), float(y.sum()), eps, n, r)
    cheap = certificate_cheap(float(y[r]), float(y[: r + 1].sum()), eps, n, r)
    return CertificateRecord(iteration, cheap.lhs_cheap, cheap.holds_cheap, cheap.threshold, full.lhs_cheap,
                             full.holds_cheap)


def merge_certificates(cheap: CertificateRecord, full: CertificateRecord) -> CertificateRecord:
    return replace(cheap, lhs_full=full.lhs_full, holds_full=full.holds_full)


# ---------------------------------------------------------------------------
# operator and step (meg.py:287-364)


def _as_gradient(x: LowRankIterate, grad_apply) -> GradientOperator:
    """A device descriptor as is; any other callable through the callback operator (the
    reference's `grad_apply` contract, meg.py:327-335: numpy blocks in and out, or torch CUDA
    tensors when marked with callbacks.device_callable)."""
    if isinstance(grad_apply, GradientOperator):
        if grad_apply.n != x.n:
            raise ParameterError(f"gradient dimension {grad_apply.n} does not match n={x.n}")
        return grad_apply
    if callable(grad_apply):
        from .objectives import CallbackGradient

        return CallbackGradient(x.n, grad_apply)
    raise TypeError("grad_apply must be a device gradient descriptor or a callable u -> grad f(X) u")


class LogmapOperator:
    """u -> (log X - eta grad) u without materialising log X (meg.py:287-307)."""

    def __init__(self, x: LowRankIterate, grad: GradientOperator, eta: float):
        self.x, self.grad, self.eta = x, grad, float(eta)
        self.dim = x.n

    def apply(self, u):
        is_np = not isinstance(u, torch.Tensor)
        vec = u.ndim == 1
        ut = runtime.as_device_f64(u)
        if vec:
            ut = ut.reshape(-1, 1).contiguous()
        w = torch.empty_like(ut)
        s = self.grad.solver()
        keep: list = []
        xs, gs = self.x.struct(keep), self.grad.struct(keep)
        checked(s.lib.megb200_logmap_apply(s.handle, C.byref(xs), C.byref(gs), self.eta, ut.data_ptr(),
                                           ut.stride(0), ut.shape[1], w.data_ptr(), w.stride(0)), [self.grad.callback])
        if vec:
            w = w.reshape(-1)
        return w.cpu().numpy() if is_np else w

    def to_dense(self) -> np.ndarray:
        return symmetrize(self.apply(np.eye(self.dim)))


def logmap_operator(x: LowRankIterate, grad_apply, eta: float) -> LogmapOperator:
    return LogmapOperator(x, _as_gradient(x, grad_apply), eta)


@dataclass(frozen=True)
class LowRankStepResult:
    """Next iterate plus certificate inputs (meg.py:310-324).

    `top_eigenvalues` holds y = exp(mu - mu_1) (length r+1), as in the
    reference; `mu`, `residual_norms`, `passes`, `restarts` are solver
    telemetry added by this implementation.
    """

    iterate: LowRankIterate
    cert: CertificateRecord
    lambda_r_plus_1: float
    b_r_plus_1: float
    shift: float
    top_eigenvalues: np.ndarray | None = field(repr=False, default=None)
    mu: np.ndarray | None = field(repr=False, default=None)
    residual_norms: np.ndarray | None = field(repr=False, default=None)
    passes: int = 0
    restarts: int = 0
    svd_tol_effective: float = 0.0  # the residual rule's tol as applied (float32 operands: >= F32_TOL_FLOOR)
    svd_subspace_effective: int | None = None  # the Krylov basis bound as applied (<= runtime.MAX_BASIS)


class SolverSettingWarning(UserWarning):
    """A solver setting was applied in a modified form (reported in the step result as well)."""


def effective_settings(svd_tol: float, svd_subspace: int | None, g) -> tuple[float, int | None]:
    """(tol, basis bound) the device solver applies: float32 operands raise the residual rule's tol
    to objectives.F32_TOL_FLOOR (their product noise sits above 1e-10); the basis is bounded by the
    shared-memory Rayleigh-Ritz limit runtime.MAX_BASIS (the block solver then restarts: the same
    rule linalg.py:214-216, more passes).  Either change is reported once per call site."""
    import warnings

    tol = max(float(svd_tol), g.tol_floor)
    if tol > svd_tol:
        warnings.warn(f"svd_tol={svd_tol:g} raised to {tol:g} for a float32 operand", SolverSettingWarning,
                      stacklevel=3)
    sub = svd_subspace
    if sub is not None and sub > runtime.MAX_BASIS:
        warnings.warn(f"svd_subspace={sub} bounded by the device Rayleigh-Ritz limit {runtime.MAX_BASIS}",
                      SolverSettingWarning, stacklevel=3)
        sub = runtime.MAX_BASIS
    return tol, sub


def lowrank_meg_step(
    x: LowRankIterate,
    grad_apply,
    eta: float,
    eps_next: float,
    svd_tol: float = 1e-10,
    svd_seed: int = 0,
    svd_subspace: int | None = None,
    *,
    block: int | None = None,
    keep: int | None = None,
    max_passes: int | None = None,
) -> LowRankStepResult:
    """One low-rank MEG update (meg.py:327-364; Algorithm 2).

    r + 1 eigenpairs of log X - eta grad by the device block solver
    (svd_subspace = Krylov basis size, svd_tol = residual rule, svd_seed =
    random directions), max-shift exponentiation, renormalised kept mass
    1 - eps_next, cheap certificate.  Raises ParameterError for eps_next
    outside (0, 3/4] before any launch, LanczosError with the best residuals
    if the solver does not converge.
    """
    if not 0 < eps_next <= 0.75:
        raise ParameterError(f"eps_next must lie in (0, 3/4], got {eps_next}")
    g = _as_gradient(x, grad_apply)
    n, r = x.n, x.r
    if r + 1 >= n:
        raise ParameterError(f"need r + 1 < n, got r={r}, n={n}")
    s = g.solver()
    dev = runtime.device()
    hold: list = []
    xs, gs = x.struct(hold), g.struct(hold)
    warm = x.warm_block if isinstance(x.warm_block, torch.Tensor) and x.warm_block.shape[0] == n else None
    tol_eff, sub_eff = effective_settings(svd_tol, svd_subspace, g)
    opts = _eig_opts(tol_eff, max_passes, svd_seed, sub_eff, 12, block, keep, warm,
                     warm_orthonormal=warm is not None and x.warm_orth_err <= 1e-13)
    v_next = torch.empty((n, r), dtype=torch.float64, device=dev)
    ritz = torch.empty((n, runtime.MAX_BLOCK), dtype=torch.float64, device=dev)
    lam = np.zeros(r)
    y = np.zeros(r + 1)
    mu = np.zeros(r + 1)
    res = np.zeros(r + 1)
    out = _lib.StepResult()
    out.V_next = v_next.data_ptr()
    out.ld_next = r
    out.lam_next = _lib.dptr(lam)
    out.y = _lib.dptr(y)
    out.mu = _lib.dptr(mu)
    out.residual_norms = _lib.dptr(res)
    out.ritz_block = ritz.data_ptr()
    out.ld_ritz = ritz.stride(0)
    rc = s.lib.megb200_lowrank_meg_step(s.handle, C.byref(xs), C.byref(gs), float(eta), float(eps_next),
                                        C.byref(opts), C.byref(out))
    checked(rc, [g.callback], residual_norms=res.copy())
    nxt = LowRankIterate(n, r, v_next, lam, eps_next, warm_block=ritz[:, : out.ritz_cols],
                         warm_orth_err=out.ritz_orth_err, _gram_err=out.gram_err)
    cert = CertificateRecord(iteration=None, lhs_cheap=out.lhs_cheap, holds_cheap=bool(out.holds_cheap),
                             threshold=out.threshold)
    return LowRankStepResult(
        iterate=nxt,
        cert=cert,
        lambda_r_plus_1=out.lambda_r_plus_1,
        b_r_plus_1=out.b_r_plus_1,
        shift=out.shift,
        top_eigenvalues=y,
        mu=mu,
        residual_norms=res,
        passes=int(out.passes),
        restarts=int(out.restarts),
        svd_tol_effective=tol_eff,
        svd_subspace_effective=sub_eff,
    )


def warm_start_wrap(V0, lam0, eps0: float) -> LowRankIterate:
    """(1-eps0) V0 diag(lam0) V0^T + (eps0/n) I in canonical structured form (meg.py:392-411)."""
    if not 0 < eps0 <= 0.75:
        raise ParameterError(f"eps0 must lie in (0, 3/4], got {eps0}")
    lam0 = np.asarray(lam0, dtype=float).ravel()
    n, r = tuple(V0.shape)
    if abs(lam0.sum() - 1.0) > 1e-10 or not np.all(lam0 > 0):
        raise ParameterError("lam0 must be strictly positive and sum to 1")
    order = np.argsort(-lam0, kind="stable")
    lam0 = lam0[order]
    if isinstance(V0, torch.Tensor):
        V0 = V0[:, torch.as_tensor(order, device=V0.device)]
    else:
        V0 = np.asarray(V0, dtype=float)[:, order]
    eps_p = eps0 * (n - r) / n
    lam = ((1.0 - eps0) * lam0 + eps0 / n) / (1.0 - eps_p)
    return LowRankIterate(n=n, r=r, V=V0, lam=lam / lam.sum(), eps=eps_p)


@dataclass(frozen=True)
class HostStepResult:
    """Result of `lowrank_meg_step_host`: the next factor in host memory plus the
    step's scalars (same meaning as LowRankStepResult's fields)."""

    V: object  # host array / pinned tensor, n x r
    lam: np.ndarray
    eps: float
    cert: CertificateRecord
    lambda_r_plus_1: float
    b_r_plus_1: float
    shift: float
    top_eigenvalues: np.ndarray
    residual_norms: np.ndarray
    passes: int
    warm_block: object  # device Ritz block for the next step
    warm_orth_err: float


def lowrank_meg_step_host(
    V,
    lam,
    eps: float,
    objective,
    eta: float,
    eps_next: float,
    svd_tol: float = 1e-10,
    svd_seed: int = 0,
    svd_subspace: int | None = None,
    *,
    t: int = 0,
    block: int | None = None,
    warm=None,
    warm_orth_err: float = 1.0,
    out=None,
) -> HostStepResult:
    """One MEG step for a caller that keeps the iterate factor V (n x r) in host
    memory: one native call uploads V, validates it like LowRankIterate
    (meg.py:62-77; ParameterError before the step), runs the step and writes
    V_next to `out` (a host array or pinned CPU tensor; allocated if None).

    `objective` is a device objective (its gradient is taken at the uploaded
    iterate) or a gradient descriptor; `warm` is the device Ritz block returned
    by the previous call (optional)."""
    if not 0 < eps_next <= 0.75:
        raise ParameterError(f"eps_next must lie in (0, 3/4], got {eps_next}")
    if not 0 < eps <= 0.75:
        raise ParameterError(f"eps must lie in (0, 3/4], got {eps}")
    n, r = int(V.shape[0]), int(V.shape[1])
    lam = np.ascontiguousarray(np.asarray(lam, dtype=np.float64).ravel())
    if lam.shape != (r,):
        raise ParameterError(f"lam must have {r} entries")
    if abs(lam.sum() - 1.0) > 1e-10:
        raise ParameterError(f"lam must sum to 1, got {lam.sum()!r}")
    if np.any(np.diff(lam) > 0) or not lam[-1] > 0:
        raise ParameterError("lam must be sorted non-increasing and strictly positive")
    g = objective.grad_operator(None, t) if hasattr(objective, "grad_operator") else objective
    if not isinstance(g, GradientOperator):
        raise TypeError("objective must be a device objective or gradient descriptor")
    s = g.solver()
    hold: list = []
    gs = g.struct(hold)
    it = _lib.Iterate()
    it.n, it.r, it.eps = n, r, float(eps)
    it.lam = _lib.dptr(lam)
    if isinstance(V, torch.Tensor):
        if V.is_cuda or V.dtype != torch.float64 or not V.is_contiguous():
            raise ParameterError("V must be a contiguous float64 host tensor")
        it.V, it.ldv = V.data_ptr(), V.stride(0)
    else:
        V = np.ascontiguousarray(V, dtype=np.float64)
        it.V, it.ldv = V.ctypes.data, V.strides[0] // 8
    if out is None:
        out = np.empty((n, r))
    out_ptr = out.data_ptr() if isinstance(out, torch.Tensor) else out.ctypes.data
    ld_out = out.stride(0) if isinstance(out, torch.Tensor) else out.strides[0] // 8
    warm_t = warm if isinstance(warm, torch.Tensor) and warm.shape[0] == n else None
    tol_eff, sub_eff = effective_settings(svd_tol, svd_subspace, g)
    opts = _eig_opts(tol_eff, None, svd_seed, sub_eff, 12, block, None, warm_t,
                     warm_orthonormal=warm_t is not None and warm_orth_err <= 1e-13)
    ritz = torch.empty((n, runtime.MAX_BLOCK), dtype=torch.float64, device=runtime.device())
    lam_next, y, mu, res = np.zeros(r), np.zeros(r + 1), np.zeros(r + 1), np.zeros(r + 1)
    o = _lib.StepResult()
    o.lam_next, o.y, o.mu, o.residual_norms = _lib.dptr(lam_next), _lib.dptr(y), _lib.dptr(mu), _lib.dptr(res)
    o.ritz_block = ritz.data_ptr()
    o.ld_ritz = ritz.stride(0)
    rc = s.lib.megb200_lowrank_meg_step_host(s.handle, C.byref(it), C.byref(gs), float(eta), float(eps_next),
                                             C.byref(opts), C.c_void_p(out_ptr), int(ld_out), C.byref(o))
    checked(rc, [getattr(g, "callback", None)], residual_norms=res.copy())
    cert = CertificateRecord(iteration=None, lhs_cheap=o.lhs_cheap, holds_cheap=bool(o.holds_cheap),
                             threshold=o.threshold)
    return HostStepResult(V=out, lam=lam_next, eps=float(eps_next), cert=cert, lambda_r_plus_1=o.lambda_r_plus_1,
                          b_r_plus_1=o.b_r_plus_1, shift=o.shift, top_eigenvalues=y, residual_norms=res,
                          passes=int(o.passes), warm_block=ritz[:, : o.ritz_cols], warm_orth_err=o.ritz_orth_err)


class HostStepper:
    """Repeated host-buffer MEG steps on one objective: the per-call part of
    `lowrank_meg_step_host` without its per-call setup.  The native structs, the result
    arrays and two alternating device Ritz-block buffers are made once; `step` validates
    lam/eps like LowRankIterate (meg.py:62-77; V is validated by the native call), fills the
    changing fields and makes the one native call.

    The returned `warm_block` stays valid until the step after next (double buffered), and the
    returned arrays are fresh copies.  For objectives whose gradient depends on the step index
    (the stochastic Frobenius objective) use `lowrank_meg_step_host`."""

    def __init__(self, objective, n: int, r: int, *, svd_tol: float = 1e-10, svd_subspace: int | None = None,
                 block: int | None = None):
        from .objectives import StochasticFrobeniusObjective

        if isinstance(objective, StochasticFrobeniusObjective):
            raise ParameterError("HostStepper needs a step-independent gradient; use lowrank_meg_step_host")
        g = objective.grad_operator(None, 0) if hasattr(objective, "grad_operator") else objective
        if not isinstance(g, GradientOperator):
            raise TypeError("objective must be a device objective or gradient descriptor")
        self.n, self.r = int(n), int(r)
        self.s = g.solver()
        self._hold: list = [g]
        self.gs = g.struct(self._hold)
        self.tol, self.subspace = effective_settings(svd_tol, svd_subspace, g)
        self.block = block
        dev = runtime.device()
        self.ritz = [torch.empty((self.n, runtime.MAX_BLOCK), dtype=torch.float64, device=dev) for _ in range(2)]
        self.k = 0
        self.buf = np.zeros(4 * self.r + 3)
        self.lam_next = self.buf[: self.r]
        self.y = self.buf[self.r: 2 * self.r + 1]
        self.mu = self.buf[2 * self.r + 1: 3 * self.r + 2]
        self.res = self.buf[3 * self.r + 2:]
        self.it = _lib.Iterate()
        self.it.n, self.it.r = self.n, self.r
        self.lam_in = np.zeros(self.r)
        self.it.lam = _lib.dptr(self.lam_in)
        self.o = _lib.StepResult()
        self.o.lam_next, self.o.y, self.o.mu = _lib.dptr(self.lam_next), _lib.dptr(self.y), _lib.dptr(self.mu)
        self.o.residual_norms = _lib.dptr(self.res)
        self.fn = self.s.lib.megb200_lowrank_meg_step_host
        self.opts = _eig_opts(self.tol, None, 0, self.subspace, 12, self.block)
        self._views: dict = {}  # (buffer, cols) -> warm-block view (the width is fixed per solve shape)

    def step(self, V, lam, eps: float, eta: float, eps_next: float, svd_seed: int = 0, *, warm=None,
             warm_orth_err: float = 1.0, out=None) -> HostStepResult:
        if not 0 < eps_next <= 0.75:
            raise ParameterError(f"eps_next must lie in (0, 3/4], got {eps_next}")
        if not 0 < eps <= 0.75:
            raise ParameterError(f"eps must lie in (0, 3/4], got {eps}")
        lam_in = self.lam_in
        try:
            lam_in[:] = lam
        except ValueError as e:
            raise ParameterError(f"lam must have {self.r} entries") from e
        ssum = 0.0
        prev = math.inf
        for v in lam_in.tolist():  # LowRankIterate's lam rules (meg.py:72-77), without array temporaries
            if not (0.0 < v <= prev):
                raise ParameterError("lam must be sorted non-increasing and strictly positive")
            prev = v
            ssum += v
        if abs(ssum - 1.0) > 1e-10:
            raise ParameterError(f"lam must sum to 1, got {ssum!r}")
        it = self.it
        it.eps = float(eps)
        if not (isinstance(V, torch.Tensor) and not V.is_cuda and V.dtype == torch.float64 and V.is_contiguous()
                and tuple(V.shape) == (self.n, self.r)):
            raise ParameterError("V must be a contiguous float64 host tensor of shape (n, r)")
        it.V, it.ldv = V.data_ptr(), self.r
        if out is None:
            out = torch.empty((self.n, self.r), dtype=torch.float64).pin_memory()
        opts = self.opts
        opts.seed = int(svd_seed) & 0xFFFFFFFFFFFFFFFF
        if isinstance(warm, torch.Tensor) and warm.shape[0] == self.n:
            opts.warm, opts.warm_cols, opts.ld_warm = warm.data_ptr(), warm.shape[1], warm.stride(0)
            opts.warm_orthonormal = 1 if warm_orth_err <= 1e-13 else 0
        else:
            opts.warm, opts.warm_cols, opts.ld_warm, opts.warm_orthonormal = 0, 0, 0, 0
        kb = self.k
        ritz = self.ritz[kb]
        self.k ^= 1
        o = self.o
        o.ritz_block, o.ld_ritz = ritz.data_ptr(), ritz.stride(0)
        rc = self.fn(self.s.handle, C.byref(it), C.byref(self.gs), float(eta), float(eps_next), C.byref(opts),
                     C.c_void_p(out.data_ptr()), self.r, C.byref(o))
        if rc:
            checked(rc, [getattr(self._hold[0], "callback", None)], residual_norms=self.res.copy())
        cert = CertificateRecord(iteration=None, lhs_cheap=o.lhs_cheap, holds_cheap=bool(o.holds_cheap),
                                 threshold=o.threshold)
        return HostStepResult(V=out, lam=self.lam_next.copy(), eps=float(eps_next), cert=cert,
                              lambda_r_plus_1=o.lambda_r_plus_1, b_r_plus_1=o.b_r_plus_1, shift=o.shift,
                              top_eigenvalues=self.y.copy(), residual_norms=self.res.copy(), passes=int(o.passes),
                              warm_block=self._view(kb, ritz, o.ritz_cols), warm_orth_err=o.ritz_orth_err)

    def _view(self, kb: int, ritz, cols: int):
        v = self._views.get((kb, cols))
        if v is None:
            v = self._views[(kb, cols)] = ritz[:, :cols]
        return v
