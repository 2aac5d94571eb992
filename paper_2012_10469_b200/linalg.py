"""Device linear algebra mirroring `specmeg.linalg` (linalg.py:1-283) for the hot path.

`SymmetricOperator` (linalg.py:81-103) becomes a *device operator
descriptor*: A u = scale * Op u + L diag(d) L^T u + alpha u, with Op a dense
symmetric matrix or a CSR matrix resident in HBM.  `lanczos_top_r`
(linalg.py:130-241) keeps its signature and result type but runs the block
thick-restart Lanczos solver of csrc/megb200_runtime.cu: one streamed pass of
the operand per block of `block` vectors, CholQR2 orthonormalisation,
Jacobi Rayleigh-Ritz, same convergence rule (every residual <= tol *
max(1, max|theta|), linalg.py:214-215) and the same failure contract
(LanczosError carrying the best residuals).

Operators built from device data (`from_dense`, `from_csr`, or the descriptors
in `meg` / `objectives`) stream from HBM inside the pass kernels.  The
reference's form `SymmetricOperator(dim, apply_fn)` with a Python callable is
accepted too: the native solver calls it once per block pass through the C
ABI's callback operator (callbacks.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, runtime
from .callbacks import checked
from .errors import EighError, LanczosError, ParameterError, RankDeficiencyError  # noqa: F401  (re-export)


def symmetrize(a):
    """(A + A^T)/2 in float64 (linalg.py:55-60); numpy in -> numpy out, torch in -> torch out."""
    if isinstance(a, torch.Tensor):
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ParameterError(f"expected a square matrix, got shape {tuple(a.shape)}")
        a = a.to(torch.float64)
        return 0.5 * (a + a.T)
    a = np.asarray(a, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ParameterError(f"expected a square matrix, got shape {a.shape}")
    return 0.5 * (a + a.T)


@dataclass(frozen=True)
class TopREigen:
    """The r algebraically largest eigenpairs (linalg.py:71-78) plus solver telemetry."""

    r: int
    eigenvalues: np.ndarray  # (r,) non-increasing
    eigenvectors: object  # (n, r) orthonormal columns: numpy (default) or torch CUDA tensor
    residual_norms: np.ndarray  # (r,)
    passes: int = 0
    restarts: int = 0
    subspace_effective: int | None = None  # basis bound as applied (<= runtime.MAX_BASIS)


class SymmetricOperator:
    """Device symmetric operator  u -> scale * Op u + L diag(d) L^T u + alpha u."""

    def __init__(self, dim: int, apply_fn=None, *, dense=None, csr=None, scale: float = 1.0, L=None, d=None,
                 alpha: float = 0.0, qm=None):
        """`SymmetricOperator(dim, apply_fn)` is the reference's form (linalg.py:89-94): apply_fn
        takes a numpy (n, k) block (or torch CUDA tensors when marked with
        callbacks.device_callable) and is called once per block pass through the C ABI's callback
        operator.  Device data (dense / csr / low-rank) is the fast path."""
        from .callbacks import ApplyCallback

        self.dim = int(dim)
        self.callback = ApplyCallback(apply_fn, self.dim) if apply_fn is not None else None
        self.dense = dense  # torch (n, n) f64/f32 contiguous, symmetric
        self.csr = csr  # (rowptr int32, col int32, val f64) torch tensors
        self.qm = qm  # objectives.QuadMeasOperand: matrix-free measurement gradient (OP_QUADMEAS)
        self.scale = float(scale)
        self.L = L  # torch (n, l) f64 or None
        self.d = None if d is None else runtime.host_f64(d)
        self.alpha = float(alpha)

    @classmethod
    def from_dense(cls, a, dtype: str = "f64") -> "SymmetricOperator":
        """Upload a dense matrix, symmetrised as in linalg.py:96-99."""
        t = runtime.as_device_operand(a, "f64")
        t = (0.5 * (t + t.T)).contiguous()
        if dtype == "f32":
            t = t.to(torch.float32).contiguous()
        return cls(t.shape[0], dense=t)

    @classmethod
    def from_csr(cls, n: int, rowptr, col, val, scale: float = 1.0) -> "SymmetricOperator":
        dev = runtime.device()
        rp = torch.as_tensor(np.asarray(rowptr, dtype=np.int32)).to(dev)
        cl = torch.as_tensor(np.asarray(col, dtype=np.int32)).to(dev)
        vl = runtime.as_device_f64(val)
        return cls(n, csr=(rp, cl, vl), scale=scale)

    def _struct(self, keep: list) -> _lib.Operator:
        op = _lib.Operator()
        op.n = self.dim
        op.scale = self.scale
        op.alpha = self.alpha
        if self.dense is not None:
            op.kind = _lib.OP_DENSE
            op.dtype = runtime.dtype_code(self.dense)
            op.dense = self.dense.data_ptr()
            op.ld = self.dense.stride(0)
        elif self.csr is not None:
            rp, cl, vl = self.csr
            op.kind = _lib.OP_CSR
            op.rowptr, op.col, op.val = rp.data_ptr(), cl.data_ptr(), vl.data_ptr()
            op.nnz = cl.numel()
        elif self.qm is not None:
            op.kind = _lib.OP_QUADMEAS
            op.apply_ctx = self.qm.ctx(keep)
        elif self.callback is not None:
            op.kind = _lib.OP_CALLBACK
            op.apply = self.callback.c_fn
        else:
            op.kind = _lib.OP_NONE
        if self.L is not None and self.L.shape[1] > 0:
            op.L = self.L.data_ptr()
            op.l = self.L.shape[1]
            op.ldl = self.L.stride(0)
            keep.append(self.d)
            op.d = _lib.dptr(self.d)
        return op

    def _solver(self):
        nnz = self.csr[1].numel() if self.csr is not None else 0
        lw = self.L.shape[1] if self.L is not None else 0
        return runtime.solver_for(self.dim, max_nnz=nnz, max_lowrank=max(runtime.MAX_LOWRANK, lw))

    def apply(self, u):
        """A u for u of shape (n,) or (n, k) (linalg.py:93-94); numpy in -> numpy out."""
        is_np = not isinstance(u, torch.Tensor)
        vec = (u.ndim == 1)
        ut = runtime.as_device_f64(u)
        if vec:
            ut = ut.reshape(-1, 1).contiguous()
        if ut.shape[0] != self.dim:
            raise ParameterError(f"expected {self.dim} rows, got {ut.shape[0]}")
        k = ut.shape[1]
        w = torch.empty_like(ut)
        s = self._solver()
        keep: list = []
        op = self._struct(keep)
        checked(s.lib.megb200_operator_apply(s.handle, C.byref(op), ut.data_ptr(), ut.stride(0), k,
                                             w.data_ptr(), w.stride(0)), [self.callback])
        if vec:
            w = w.reshape(-1)
        return w.cpu().numpy() if is_np else w

    def to_dense(self) -> np.ndarray:
        """Materialise by applying to the identity (test/shadow use only, linalg.py:101-103)."""
        return symmetrize(self.apply(np.eye(self.dim)))


def _eig_opts(tol, max_iter, seed, subspace, restarts, block=None, keep=None, warm=None,
              warm_orthonormal=False) -> _lib.EigOpts:
    o = _lib.EigOpts()
    o.tol = float(tol)
    o.max_passes = int(max_iter) if max_iter is not None else 0
    o.restarts = int(restarts)
    o.block = int(block) if block else 0
    o.basis = int(subspace) if subspace is not None else 0
    o.keep = int(keep) if keep else 0
    o.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    if warm is not None:
        o.warm = warm.data_ptr()
        o.warm_cols = warm.shape[1]
        o.ld_warm = warm.stride(0)
        o.warm_orthonormal = 1 if warm_orthonormal else 0
    return o


def lanczos_top_r(
    op: SymmetricOperator,
    r: int,
    tol: float = 1e-10,
    max_iter: int | None = None,
    seed: int = 0,
    subspace: int | None = None,
    restarts: int = 12,
    *,
    block: int | None = None,
    return_device: bool = False,
) -> TopREigen:
    """Algebraically largest r eigenpairs of a device operator (linalg.py:130-241).

    `subspace` is the Krylov basis size, `max_iter` the budget in block passes
    (default restarts * basis), `block` the block width (default r + 7).
    Raises ParameterError for r outside [1, n) and LanczosError carrying the
    best residual norms when the tolerance is not reached.
    """
    if not isinstance(op, SymmetricOperator):
        if hasattr(op, "dim") and hasattr(op, "apply"):  # any object with the reference's operator interface
            op = SymmetricOperator(op.dim, op.apply)
        else:
            raise TypeError("lanczos_top_r needs a SymmetricOperator (or an object with .dim and .apply)")
    n = op.dim
    if not 1 <= r < n:
        raise ParameterError(f"need 1 <= r < n, got r={r}, n={n}")
    s = op._solver()
    keep: list = []
    ops = op._struct(keep)
    if subspace is not None and subspace > runtime.MAX_BASIS:
        import warnings

        from .meg import SolverSettingWarning

        warnings.warn(f"subspace={subspace} bounded by the device Rayleigh-Ritz limit {runtime.MAX_BASIS}",
                      SolverSettingWarning, stacklevel=2)
        subspace = runtime.MAX_BASIS
    opts = _eig_opts(tol, max_iter, seed, subspace, restarts, block)
    vals = np.zeros(r)
    res = np.zeros(r)
    vecs = torch.empty((n, r), dtype=torch.float64, device=runtime.device())
    out = _lib.EigResult()
    out.eigenvalues = _lib.dptr(vals)
    out.residual_norms = _lib.dptr(res)
    out.eigenvectors = vecs.data_ptr()
    out.ld_vec = r
    rc = s.lib.megb200_top_r(s.handle, C.byref(ops), int(r), C.byref(opts), C.byref(out))
    checked(rc, [op.callback], residual_norms=res.copy())
    return TopREigen(
        r=r,
        eigenvalues=vals,
        eigenvectors=vecs if return_device else vecs.cpu().numpy(),
        residual_norms=res,
        passes=int(out.passes),
        restarts=int(out.restarts),
        subspace_effective=subspace,
    )


def project_simplex(z, tau: float = 1.0) -> np.ndarray:
    """Euclidean projection onto {w >= 0, sum w = tau} (linalg.py:244-261).

    Host arithmetic on the r initial weights (run once per trajectory, never
    per iteration), exactly as in the reference.
    """
    z = np.asarray(z, dtype=float).ravel()
    if z.size < 1:
        raise ParameterError("need at least one coordinate")
    if not tau > 0:
        raise ParameterError(f"tau must be positive, got {tau}")
    srt = np.sort(z)[::-1]
    csum = np.cumsum(srt)
    k = int(np.flatnonzero(srt - (csum - tau) / np.arange(1, z.size + 1) > 0).max()) + 1
    return np.maximum(z - (csum[k - 1] - tau) / k, 0.0)
