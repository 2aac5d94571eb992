"""Dense-shadow diagnostics on the device: exact MEG, the shadow low-rank step, Bregman distances.

The reference's lockstep / dense-shadow mode:
`exact_meg_step` (meg.py:269-284), `shadow_lowrank_step` (meg.py:367-385), `certificate_full`
(meg.py:240-260, in meg.py here), the von Neumann Bregman distance `bregman` (entropy.py:76-96)
and its structured form `bregman_structured` (entropy.py:99-142).  They need full
eigendecompositions -- O(n^3), allowed only for small n (the reference's dense_cap, 400) --
and are diagnostics off the per-iteration hot path.

Full eigendecompositions: n <= 112 through the native small symmetric solver of the block Krylov
method (megb200_sym_eigh: tridiagonalisation + multisection + twisted factorisation, verified,
Jacobi fallback); larger n (the shadow cap) through torch.linalg.eigh, i.e. cuSOLVER, like a
library GEMM -- nothing on the MEG step path uses it.  Inputs may be numpy or torch; results are
torch float64 CUDA tensors (scalars as floats).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import runtime
from .errors import EighError, ParameterError

EIG_CLAMP = 1e-300  # entropy.py:21
_MASS_TOL = 1e-14  # entropy.py:22
SHADOW_NATIVE_MAX = runtime.MAX_BASIS


class NotPSDError(ValueError):
    """Argument has a significantly negative eigenvalue (entropy.py:25-26)."""


@dataclass(frozen=True)
class BregmanValue:
    """Bregman distance value with degeneracy flags (entropy.py:29-43)."""

    value: float
    finite: bool = True
    clamped: bool = False

    def __float__(self) -> float:
        return self.value


def _dev(a) -> torch.Tensor:
    return runtime.as_device_f64(a)


def _sym(a: torch.Tensor) -> torch.Tensor:
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ParameterError(f"expected a square matrix, got shape {tuple(a.shape)}")
    return 0.5 * (a + a.T)


def full_eigh(a) -> tuple[torch.Tensor, torch.Tensor]:
    """Eigenvalues (non-increasing) and eigenvectors (columns) of sym(a) (linalg.py:106-119)."""
    a = _sym(_dev(a)).contiguous()
    n = a.shape[0]
    if n <= SHADOW_NATIVE_MAX:
        s = runtime.solver_for(max(n, 2) if n > 1 else 2)
        w = torch.empty(n, dtype=torch.float64, device=a.device)
        v = torch.empty((n, n), dtype=torch.float64, device=a.device)
        runtime.check(s.lib.megb200_sym_eigh(s.handle, a.data_ptr(), a.stride(0), n, w.data_ptr(), v.data_ptr()))
        return w, v
    try:
        w, v = torch.linalg.eigh(a)
    except RuntimeError as exc:  # pragma: no cover - cuSOLVER failure
        raise EighError(f"eigendecomposition of a {n}x{n} matrix did not converge: {exc}") from exc
    return torch.flip(w, (0,)), torch.flip(v, (1,))


def _log_matrix(w: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    return (v * torch.log(w)) @ v.T


def exact_meg_step(z, grad, eta: float) -> torch.Tensor:
    """exp(log Z - eta grad) / trace, Z symmetric positive definite with unit trace (meg.py:269-284)."""
    w, v = full_eigh(z)
    if float(w[-1]) <= 0:
        raise ParameterError(f"iterate must be positive definite, min eigenvalue {float(w[-1]):.3e}")
    exponent = _sym(_log_matrix(w, v) - float(eta) * _dev(grad))
    ew, ev = full_eigh(exponent)
    y = torch.exp(ew - ew[0])
    y = y / y.sum()
    return _sym((ev * y) @ ev.T)


def shadow_lowrank_step(x_dense, grad_dense, eta: float, eps_next: float, r: int):
    """Dense recomputation of the low-rank update (meg.py:367-385): (low-rank updated matrix,
    exact updated matrix, shifted spectrum y = exp(mu - mu_1) of the exponential)."""
    x = _dev(x_dense)
    n = x.shape[0]
    w, v = full_eigh(x)
    log_x = (v * torch.log(torch.clamp(w, min=1e-300))) @ v.T
    ew, ev = full_eigh(_sym(log_x - float(eta) * _dev(grad_dense)))
    y = torch.exp(ew - ew[0])
    exact = _sym((ev * (y / y.sum())) @ ev.T)
    kept = ev[:, :r]
    low = (1.0 - eps_next) * (kept * (y[:r] / y[:r].sum())) @ kept.T
    low = low + eps_next / (n - r) * (torch.eye(n, dtype=torch.float64, device=x.device) - kept @ kept.T)
    return _sym(low), exact, y


def _psd_spectrum(x: torch.Tensor, name: str = "X") -> torch.Tensor:
    w, _ = full_eigh(x)
    top = max(1e-30, float(torch.abs(w).max()))
    if float(w.min()) < -1e-8 * top:
        raise NotPSDError(f"{name} has eigenvalue {float(w.min()):.3e} < -1e-8 * ||{name}||_2")
    return w


def _entropy_sum(w: torch.Tensor) -> float:
    """sum lambda log lambda with 0 log 0 = 0 (entropy.py:54-58)."""
    w = torch.clamp(w, min=0.0)
    w = w[w > EIG_CLAMP]
    return float(torch.sum(w * torch.log(w)))


def von_neumann_entropy(x) -> float:
    """Tr(X log X - X) for PSD X (entropy.py:61-64)."""
    w = _psd_spectrum(_dev(x))
    return _entropy_sum(w) - float(torch.sum(torch.clamp(w, min=0.0)))


def _check_unit_trace(x: torch.Tensor, name: str) -> None:
    tr = float(torch.trace(x))
    if abs(tr - 1.0) > 1e-8:
        raise ValueError(f"{name} must have unit trace, got {tr!r}")


def bregman(x, y) -> BregmanValue:
    """Tr(X log X - X log Y) for trace-1 PSD X and (near) PD Y, diagonalised separately
    (entropy.py:76-96)."""
    x = _sym(_dev(x))
    y = _sym(_dev(y))
    _check_unit_trace(x, "X")
    _check_unit_trace(y, "Y")
    wx = _psd_spectrum(x, "X")
    wy, vy = full_eigh(y)
    mass = torch.einsum("ij,ji->i", vy.T @ x, vy)
    heavy = mass > _MASS_TOL
    if bool(torch.any(heavy & (wy <= 0.0))):
        return BregmanValue(value=math.inf, finite=False, clamped=True)
    clamped = bool(torch.any(heavy & (wy <= EIG_CLAMP)))
    cross = float(torch.sum(mass * torch.log(torch.clamp(wy, min=EIG_CLAMP))))
    return BregmanValue(value=_entropy_sum(wx) - cross, finite=True, clamped=clamped)


def structured_entropy_sum(lam, eps: float, n: int) -> float:
    """Tr(X log X) of a structured iterate (entropy.py:99-105)."""
    lam = np.asarray(lam, dtype=float)
    kept = (1.0 - eps) * lam
    tail = eps / (n - lam.size)
    k = kept[kept > EIG_CLAMP]
    return float(np.sum(k * np.log(k))) + eps * math.log(tail)


def structured_log_trace(x, y) -> float:
    """Tr(X log Y) with Y a structured iterate (entropy.py:108-125): X dense (needs X V_y, one
    n x r product) or structured (V_x^T V_y, r_x x r_y)."""
    log_kept = np.log((1.0 - y.eps) * np.asarray(y.lam))
    log_tail = math.log(y.eps / (y.n - y.r))
    vy = y.V_device
    if isinstance(x, (np.ndarray, torch.Tensor)):
        xd = _dev(x)
        mass = torch.einsum("ij,ij->j", vy, xd @ vy).cpu().numpy()
        trace_x = float(torch.trace(xd))
    else:
        cross = (x.V_device.T @ vy).cpu().numpy()
        sq = cross**2
        mass = (1.0 - x.eps) * (np.asarray(x.lam) @ sq) + (x.eps / (x.n - x.r)) * (1.0 - sq.sum(axis=0))
        trace_x = 1.0
    return float(np.sum(mass * (log_kept - log_tail))) + log_tail * trace_x


def bregman_structured(x, y) -> BregmanValue:
    """Tr(X log X - X log Y) with Y structured (entropy.py:128-142): O(r n^2) for dense X,
    O(r^2 n) for structured X."""
    if not y.eps > 0:
        raise ValueError("structured second argument must have eps > 0")
    if isinstance(x, (np.ndarray, torch.Tensor)):
        xd = _sym(_dev(x))
        _check_unit_trace(xd, "X")
        own = _entropy_sum(_psd_spectrum(xd, "X"))
        x = xd
    else:
        own = structured_entropy_sum(x.lam, x.eps, x.n)
    return BregmanValue(value=own - structured_log_trace(x, y), finite=True)
