"""Device gradient descriptors: the B200 form of the reference's `grad_apply` boundary.

The reference step takes any callable u -> grad f(X) u (meg.py:327-335; the
test objective `frobenius_objective`, test_meg.py:28-35, is used as
`lambda u: g @ u` at :153).  The device solver cannot call Python per
application, so gradients are descriptors whose data live in HBM:

    DenseGradient(G)                  grad u = G u           (a fixed dense gradient)
    FrobeniusObjective(M)             f = 1/2 ||X - M||_F^2,  grad u = X u - M u
    SampledObjective(Omega, Mobs)     f = 1/2 sum_Omega (X_ij - Mobs_ij)^2, grad = P_Omega(X - Mobs)
    StochasticFrobeniusObjective(M)   grad estimate X - M + sigma((1/b) A_t A_t^T - I/n)
    ZeroGradient(n)

`objective.grad_operator(x)` binds the gradient to an iterate X (factors
stay on device; X u is evaluated from them, never densified).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib, runtime
from .errors import ParameterError

# residual-rule floor for float32 operands: the fp32 product's rounding noise
# (~1e-8 relative to ||A||) sits above the fp64 default tol of 1e-10
F32_TOL_FLOOR = 1e-7


class GradientOperator:
    """A gradient evaluated at a bound iterate (device descriptor, see module doc)."""

    def __init__(self, kind: int, n: int, *, dense=None, csr=None, obs=None, x=None, A=None, sigma: float = 0.0,
                 owner=None, callback=None, qm=None):
        self.kind = kind
        self.callback = callback  # callbacks.ApplyCallback (GRAD_CALLBACK)
        self.qm = qm  # QuadMeasOperand (GRAD_QUADMEAS)
        self.n = int(n)
        self.dense = dense
        self.csr = csr
        self.obs = obs
        self.x = x
        self.A = A
        self.sigma = float(sigma)
        self.owner = owner

    @property
    def tol_floor(self) -> float:
        if self.dense is not None and self.dense.dtype == torch.float32:
            return F32_TOL_FLOOR
        return 0.0

    @property
    def nnz(self) -> int:
        return int(self.csr[1].numel()) if self.csr is not None else 0

    @property
    def lowrank_width(self) -> int:
        w = 0
        if self.x is not None:
            w += self.x.r
        if self.A is not None:
            w += self.A.shape[1]
        return w

    def struct(self, keep: list) -> _lib.Gradient:
        g = _lib.Gradient()
        g.kind = self.kind
        g.n = self.n
        if self.dense is not None:
            g.dtype = runtime.dtype_code(self.dense)
            g.dense = self.dense.data_ptr()
            g.ld = self.dense.stride(0)
        if self.csr is not None:
            rp, cl = self.csr
            g.rowptr, g.col = rp.data_ptr(), cl.data_ptr()
            g.nnz = cl.numel()
            g.obs = self.obs.data_ptr()
        if self.x is not None:
            lam = runtime.host_f64(self.x.lam)
            keep.append(lam)
            g.gV = self.x.V_device.data_ptr()
            g.g_r = self.x.r
            g.g_ldv = self.x.V_device.stride(0)
            g.g_lam = _lib.dptr(lam)
            g.g_eps = float(self.x.eps)
        if self.A is not None:
            g.A = self.A.data_ptr()
            g.bsz = self.A.shape[1]
            g.lda = self.A.stride(0)
            g.sigma = self.sigma
        if self.callback is not None:
            g.apply = self.callback.c_fn
        if self.qm is not None:
            g.apply_ctx = self.qm.ctx(keep)
        return g

    def solver(self):
        return runtime.solver_for(self.n, max_nnz=self.nnz,
                                  max_lowrank=max(runtime.MAX_LOWRANK, 2 * self.lowrank_width + 8))

    def __call__(self, u):
        """grad f(X_g) u, u of shape (n,) or (n, k): the descriptor is also the reference's
        `grad_apply` callable (meg.py:327-335), evaluated on the device (megb200_gradient_apply);
        numpy in -> numpy out, torch in -> torch out."""
        from .callbacks import checked

        is_np = not isinstance(u, torch.Tensor)
        vec = u.ndim == 1
        ut = runtime.as_device_f64(u)
        if vec:
            ut = ut.reshape(-1, 1).contiguous()
        if ut.shape[0] != self.n:
            raise ParameterError(f"expected {self.n} rows, got {ut.shape[0]}")
        w = torch.empty_like(ut)
        s = self.solver()
        keep: list = []
        gs = self.struct(keep)
        checked(s.lib.megb200_gradient_apply(s.handle, C.byref(gs), ut.data_ptr(), ut.stride(0), ut.shape[1],
                                             w.data_ptr(), w.stride(0)), [self.callback])
        if vec:
            w = w.reshape(-1)
        return w.cpu().numpy() if is_np else w


class CallbackGradient(GradientOperator):
    """grad u = fn(u) for a caller-supplied callable: the reference's `grad_apply` contract
    (meg.py:327-335; e.g. `lambda u: g @ u`, test_meg.py:153).  fn takes and returns numpy
    blocks (n, k) unless marked with callbacks.device_callable (torch CUDA tensors on the
    solver stream).  Called once per block pass by the native solver (callbacks.py)."""

    def __init__(self, n: int, fn, device: bool | None = None):
        from .callbacks import ApplyCallback

        super().__init__(_lib.GRAD_CALLBACK, n, callback=ApplyCallback(fn, n, device))


class ZeroGradient(GradientOperator):
    def __init__(self, n: int):
        super().__init__(_lib.GRAD_ZERO, n)


class DenseGradient(GradientOperator):
    """grad u = G u for a fixed dense symmetric G (symmetrised on upload, linalg.py:96-99)."""

    def __init__(self, g, dtype: str = "f64"):
        t = runtime.as_device_operand(g, "f64")
        t = 0.5 * (t + t.T)
        if dtype == "f32":
            t = t.to(torch.float32)
        super().__init__(_lib.GRAD_DENSE, t.shape[0], dense=t.contiguous())


class FrobeniusObjective:
    """f(X) = 1/2 ||X - M||_F^2 with M resident in HBM (f64 or f32)."""

    def __init__(self, m, dtype: str = "f64", symmetrize: bool = True):
        t = runtime.as_device_operand(m, "f64") if not (isinstance(m, torch.Tensor) and m.is_cuda) else m
        if symmetrize:
            t = 0.5 * (t.to(torch.float64) + t.to(torch.float64).T)
        t = t.to(torch.float64 if dtype == "f64" else torch.float32).contiguous()
        self.m = t
        self.n = t.shape[0]
        self.dtype = dtype
        s = runtime.solver_for(self.n)
        a, b = C.c_double(), C.c_double()
        runtime.check(s.lib.megb200_dense_stats(s.handle, t.data_ptr(), runtime.dtype_code(t), t.stride(0),
                                                C.byref(a), C.byref(b)))
        self.m_norm2 = a.value
        self.m_trace = b.value

    @classmethod
    def from_device(cls, m: torch.Tensor, dtype: str) -> "FrobeniusObjective":
        """Wrap a device matrix already symmetric (e.g. from the device generator) without copying."""
        obj = cls.__new__(cls)
        obj.m = m
        obj.n = m.shape[0]
        obj.dtype = dtype
        s = runtime.solver_for(obj.n)
        a, b = C.c_double(), C.c_double()
        runtime.check(s.lib.megb200_dense_stats(s.handle, m.data_ptr(), runtime.dtype_code(m), m.stride(0),
                                                C.byref(a), C.byref(b)))
        obj.m_norm2 = a.value
        obj.m_trace = b.value
        return obj

    def grad_operator(self, x, t: int = 0) -> GradientOperator:
        return GradientOperator(_lib.GRAD_FROBENIUS, self.n, dense=self.m, x=x, owner=self)

    def value(self, x) -> float:
        """1/2 ||X - M||_F^2 summed entry by entry over M with X_ij from the factors
        (megb200_objective_value_direct): no cancellation as X -> M, so it is exact to
        rounding RELATIVE to f itself.  One pass over M with r FMAs per entry."""
        g = self.grad_operator(x)
        s = g.solver()
        keep: list = []
        gs = g.struct(keep)
        v = C.c_double()
        runtime.check(s.lib.megb200_objective_value_direct(s.handle, C.byref(gs), C.byref(v)))
        return v.value

    def value_factored(self, x) -> float:
        """1/2 (||X||^2 - 2<X, M> + ||M||^2) from the factors: one pass M V.
        Cheaper (a block pass), but pure cancellation once X -> M (accurate to ~1e-16 ||M||^2)."""
        g = self.grad_operator(x)
        s = g.solver()
        keep: list = []
        gs = g.struct(keep)
        v = C.c_double()
        runtime.check(s.lib.megb200_objective_value(s.handle, C.byref(gs), self.m_norm2, self.m_trace, C.byref(v)))
        return v.value

    def dual_gap(self, x, tol: float = 1e-10, seed: int = 0, block: int | None = None,
                 subspace: int | None = None, warm: bool = True) -> tuple[float, float]:
        """Tr(X grad) - lambda_min(grad), grad = X - M (_dual_gap_core, objectives.py:332-335).

        Returns (gap, lambda_min).  lambda_min comes from the block solver on
        M - X (the top eigenpair of -grad, as the reference computes it).  With
        warm=True the solve starts from the Ritz block of this objective's previous
        certificate (the gradient moves little between certificates); the converged
        result obeys the same residual rule either way."""
        from .linalg import _eig_opts

        g = self.grad_operator(x)
        s = g.solver()
        keep: list = []
        gs = g.struct(keep)
        tol = max(tol, g.tol_floor)
        prev = getattr(self, "_gap_warm", None) if warm else None
        opts = _eig_opts(tol, None, seed, subspace, 12, block, None, prev, warm_orthonormal=False)
        gap, lmin = C.c_double(), C.c_double()
        out = torch.empty((self.n, runtime.MAX_BLOCK), dtype=torch.float64, device=runtime.device())
        cols = C.c_int32()
        runtime.check(s.lib.megb200_dual_gap_warm(s.handle, C.byref(gs), C.byref(opts), self.m_trace, C.byref(gap),
                                                  C.byref(lmin), out.data_ptr(), out.stride(0), C.byref(cols)),
                      residual_norms=[])
        self._gap_warm = out[:, : cols.value] if cols.value > 0 else None
        return gap.value, lmin.value


class SampledObjective:
    """f(X) = 1/2 sum_{(i,j) in Omega} (X_ij - Mobs_ij)^2 with a symmetric CSR pattern Omega."""

    def __init__(self, n: int, rowptr, col, obs):
        dev = runtime.device()
        self.n = int(n)

        def idx(a):
            if isinstance(a, torch.Tensor) and a.is_cuda:
                return a.to(torch.int32).contiguous()
            return torch.as_tensor(np.asarray(a, dtype=np.int32)).to(dev)

        self.rowptr, self.col = idx(rowptr), idx(col)
        self.obs = (obs.to(torch.float64).contiguous() if isinstance(obs, torch.Tensor) and obs.is_cuda
                    else runtime.as_device_f64(obs))
        if self.rowptr.numel() != self.n + 1 or self.col.numel() != self.obs.numel():
            raise ParameterError("inconsistent CSR arrays")

    def grad_operator(self, x, t: int = 0) -> GradientOperator:
        return GradientOperator(_lib.GRAD_SAMPLED, self.n, csr=(self.rowptr, self.col), obs=self.obs, x=x, owner=self)

    def value(self, x) -> float:
        g = self.grad_operator(x)
        s = g.solver()
        keep: list = []
        gs = g.struct(keep)
        v = C.c_double()
        runtime.check(s.lib.megb200_objective_value(s.handle, C.byref(gs), math.nan, math.nan, C.byref(v)))
        return v.value


class StochasticFrobeniusObjective(FrobeniusObjective):
    """grad estimate = X - M + sigma((1/b) A_t A_t^T - I/n), A_t ~ N(0, I/n)^{n x b}.

    A_t is generated on device by the counter-based generator (stream 5,
    counter (t n + i) b + j), the twin of oracle/inputs.minibatch, so no
    per-iteration upload is needed.
    """

    def __init__(self, m, batch: int = 64, sigma: float = 0.05, seed: int = 0, dtype: str = "f32"):
        super().__init__(m, dtype=dtype)
        self._init_stochastic(batch, sigma, seed)

    def _init_stochastic(self, batch, sigma, seed):
        self.batch = int(batch)
        self.sigma = float(sigma)
        self.seed = int(seed)
        self._a = torch.empty((self.n, self.batch), dtype=torch.float64, device=runtime.device())
        self._a_t = None

    @classmethod
    def from_device(cls, m: torch.Tensor, dtype: str, batch: int = 64, sigma: float = 0.05, seed: int = 0):
        obj = FrobeniusObjective.from_device.__func__(cls, m, dtype)
        obj._init_stochastic(batch, sigma, seed)
        return obj

    def minibatch(self, t: int) -> torch.Tensor:
        if self._a_t != t:
            s = runtime.solver_for(self.n)
            runtime.check(s.lib.megb200_gen_gaussian(
                s.handle, self.seed, 5, int(t) * self.n * self.batch, self.n, self.batch, 1.0 / math.sqrt(self.n),
                1 if self.dtype == "f32" else 0, self._a.data_ptr(), self._a.stride(0)))
            self._a_t = t
        return self._a

    def grad_operator(self, x, t: int = 0) -> GradientOperator:
        return GradientOperator(_lib.GRAD_STOCHASTIC, self.n, dense=self.m, x=x, A=self.minibatch(t),
                                sigma=self.sigma, owner=self)


class QuadMeasOperand:
    """Device arrays of the matrix-free measurement gradient weight * sym(a^T diag(res) b) (the C
    ABI's megb200_qm_data): a, b, the residuals it is evaluated at and the pass scratch."""

    def __init__(self, objective: "QuadMeasObjective", res: torch.Tensor, weight: float, idx: torch.Tensor | None = None):
        self.objective = objective
        self.res = res
        self.weight = float(weight)
        self.idx = idx  # device int64 mini-batch indices, or None for every measurement

    def ctx(self, keep: list) -> int:
        o = self.objective
        scratch = o._apply_scratch()
        d = _lib.QmData(a=o.a.data_ptr(), b=o.b.data_ptr(), res=self.res.data_ptr(),
                        m=o.m if self.idx is None else int(self.idx.numel()),
                        idx=None if self.idx is None else self.idx.data_ptr(), weight=self.weight,
                        scratch=scratch.data_ptr(), scratch_len=scratch.numel())
        keep.append(d)
        keep.append(self)
        return C.addressof(d)


class QuadMeasObjective:
    """The paper's recovery experiment (reference RecoveryObjective,
    objectives.py:174-228): g(X) = f(tau X) on the unit-trace cone,
    f(Z) = 1/2 sum_i (a_i^T Z b_i - y_i)^2 over m measurement pairs (a_i, b_i).

    a, b (m x n, unit rows) and y are uploaded once.  `grad_operator(x)` evaluates the
    residuals of x from its factors on the device (k_qm_residuals, the structured
    measurement of objectives.py:111-118) and materialises tau * grad f(tau X) =
    tau * sym(a^T diag(res) b) (k_qm_grad_part / k_qm_grad_reduce; the reference's own dense
    path, objectives.py:211-216), which the step consumes as its dense gradient.  Above `dense_cap`
    (default 1024, the reference's) the gradient is never formed: the operator is matrix-free,
    two streaming passes over a and b per block application (k_qm_fwd / k_qm_bwd; the reference's
    _apply_measurement_gradient, objectives.py:152-158 and :218-221)."""

    def __init__(self, a, b, y, tau: float, dense_cap: int = 1024):
        self.dense_cap = int(dense_cap)
        self._scratch = None
        self.a = runtime.as_device_f64(a).contiguous()
        self.b = runtime.as_device_f64(b).contiguous()
        self.y = runtime.as_device_f64(np.asarray(y, dtype=np.float64).ravel() if not isinstance(y, torch.Tensor)
                                       else y).reshape(-1).contiguous()
        if self.a.dim() != 2 or self.a.shape != self.b.shape or self.y.numel() != self.a.shape[0]:
            raise ParameterError("a, b must be m x n and y of length m")
        self.m, self.n = int(self.a.shape[0]), int(self.a.shape[1])
        self.dim = self.n
        self.tau = float(tau)

    @classmethod
    def from_instance(cls, inst) -> "QuadMeasObjective":
        """From a reference-style instance (fields a, b, y, tau; e.g. specmeg.objectives.generate_instance)."""
        return cls(inst.a, inst.b, inst.y, inst.tau)

    @classmethod
    def from_container(cls, path: str) -> "QuadMeasObjective":
        """From a "SPECMEG-QMI v1" file (the reference's save_instance format)."""
        from .inputs import load_quad_meas

        d = load_quad_meas(path)
        return cls(d["a"], d["b"], d["y"], d["tau"])

    @staticmethod
    def preset_beta(n: int, r: int) -> float:
        """Smoothness preset 0.4 sqrt(r n) (objectives.py:194-197); the experiment's eta = 1/beta."""
        return 0.4 * math.sqrt(r * n)

    def _solver(self):
        return runtime.solver_for(self.n)

    @property
    def matrix_free(self) -> bool:
        return self.n > self.dense_cap

    def _apply_scratch(self) -> torch.Tensor:
        if self._scratch is None:
            s = self._solver()
            need = int(s.lib.megb200_qm_apply_scratch(s.handle, self.m, 32))
            self._scratch = torch.empty(need, dtype=torch.float64, device=runtime.device())
        return self._scratch

    def _operator(self, res: torch.Tensor, weight: float, scale: float = 1.0):
        """weight * sym(a^T diag(res) b) as a device operator (_operator_from_residuals,
        objectives.py:214-221): materialised up to dense_cap, matrix-free above it."""
        from .linalg import SymmetricOperator

        if self.matrix_free:
            return SymmetricOperator(self.n, qm=QuadMeasOperand(self, res, weight), scale=scale)
        return SymmetricOperator(self.n, dense=self.gradient_matrix(res, weight=weight), scale=scale)

    def apply_gradient(self, res: torch.Tensor, u, weight: float | None = None) -> torch.Tensor:
        """weight / 2 (a^T (res * (b u)) + b^T (res * (a u))) for a device block u (n x k, k <= 32)
        without forming the gradient (_apply_measurement_gradient, objectives.py:152-158)."""
        s = self._solver()
        ut = runtime.as_device_f64(u)
        vec = ut.dim() == 1
        if vec:
            ut = ut.reshape(-1, 1)
        ut = ut.contiguous()
        w = torch.empty_like(ut)
        keep: list = []
        q = QuadMeasOperand(self, res, self.tau if weight is None else weight)
        runtime.check(s.lib.megb200_qm_apply(s.handle, q.ctx(keep), ut.data_ptr(), ut.stride(0), int(ut.shape[1]),
                                             w.data_ptr(), w.stride(0)))
        return w.reshape(-1) if vec else w

    def residuals(self, x) -> torch.Tensor:
        """a_i^T (tau X) b_i - y_i for a factored iterate (device tensor of length m)."""
        if x.n != self.n:
            raise ParameterError("iterate dimension does not match the objective")
        return self._residuals(x.V_device, x.lam, float(x.eps))

    def _residuals(self, V, lam, eps: float) -> torch.Tensor:
        s = self._solver()
        V = runtime.as_device_f64(V).contiguous()
        lam = runtime.host_f64(lam)
        res = torch.empty(self.m, dtype=torch.float64, device=runtime.device())
        runtime.check(s.lib.megb200_qm_residuals(s.handle, self.a.data_ptr(), self.b.data_ptr(), self.y.data_ptr(),
                                                 self.m, V.data_ptr(), V.stride(0), int(V.shape[1]), _lib.dptr(lam),
                                                 float(eps), self.tau, res.data_ptr()))
        return res

    def spectral_init(self, r: int, seed: int = 0, tol: float = 1e-10):
        """Start factor (reference spectral_init, objectives.py:293-316): a Gaussian probe u (n x r,
        unit Frobenius norm, host default_rng(seed)), the residuals of tau u u^T on the device, the
        top-r eigenpairs of -grad f(tau u u^T) by the block solver, and the simplex-projected
        negated eigenvalues (init_weights_from_top_eigs, :319-323).  Returns (V, weights)."""
        from .linalg import SymmetricOperator, lanczos_top_r, project_simplex

        if not 1 <= r < self.n:
            raise ParameterError(f"need 1 <= r < n, got r={r}, n={self.n}")
        rng = np.random.default_rng(seed)
        u = rng.standard_normal((self.n, r))
        u /= np.linalg.norm(u)
        res = self._residuals(u, np.ones(r), 0.0)
        top = lanczos_top_r(self._operator(res, 1.0, scale=-1.0), r, tol=tol, seed=seed)
        w = project_simplex(-np.asarray(top.eigenvalues, dtype=float), self.tau)
        w = w / w.sum()
        w = np.maximum(w, 1e-12)
        return top.eigenvectors, w / w.sum()

    def dual_gap(self, x, seed: int = 0, tol: float = 1e-10) -> float:
        """Linear-optimisation gap of tau X (reference dual_gap / _dual_gap_core,
        objectives.py:326-341): Tr(tau X grad) - tau v^T grad v, v the bottom eigenvector of grad f(tau X)
        (top of its negation, block solver on the device), Tr(tau X grad) = res . (res + y)."""
        from .linalg import SymmetricOperator, lanczos_top_r

        res = self.residuals(x)
        top = lanczos_top_r(self._operator(res, 1.0, scale=-1.0), 1, tol=tol, seed=seed)
        r_h = res.cpu().numpy()
        trace_term = float(r_h @ (r_h + self.y.cpu().numpy()))
        return trace_term + self.tau * float(top.eigenvalues[0])

    def value(self, x) -> float:
        """f(tau X) = 1/2 ||res||^2 (qm_value, objectives.py:133-136)."""
        res = self.residuals(x)
        s = self._solver()
        out = C.c_double()
        runtime.check(s.lib.megb200_qm_value(s.handle, res.data_ptr(), self.m, C.byref(out)))
        return float(out.value)

    def gradient_matrix(self, res: torch.Tensor, weight: float | None = None) -> torch.Tensor:
        """weight * sym(a^T diag(res) b) (n x n device tensor; weight defaults to tau)."""
        s = self._solver()
        G = torch.empty((self.n, self.n), dtype=torch.float64, device=runtime.device())
        w = self.tau if weight is None else float(weight)
        runtime.check(s.lib.megb200_qm_gradient(s.handle, self.a.data_ptr(), self.b.data_ptr(), res.data_ptr(),
                                                self.m, w, G.data_ptr(), G.stride(0)))
        return G

    def gradient_dense(self, X) -> torch.Tensor:
        """tau * grad f(tau X) at a DENSE trace-1 matrix X (the dense-shadow / exact-MEG mode,
        SPEC.md:320 grad_dense): residuals a_i^T (tau X) b_i - y_i by a dense product (cuBLAS --
        a diagnostic off the step path), then the device gradient kernel."""
        Xd = runtime.as_device_f64(X)
        res = self.tau * torch.sum((self.a @ Xd) * self.b, dim=1) - self.y
        return self.gradient_matrix(res.contiguous())

    def grad_operator(self, x, t: int = 0) -> GradientOperator:
        """tau * grad f(tau X) at x (RecoveryObjective.grad_operator, objectives.py:211-221):
        materialised on the device up to dense_cap, matrix-free above it."""
        res = self.residuals(x)
        if self.matrix_free:
            return GradientOperator(_lib.GRAD_QUADMEAS, self.n, qm=QuadMeasOperand(self, res, self.tau), owner=self)
        G = self.gradient_matrix(res)
        return GradientOperator(_lib.GRAD_DENSE, self.n, dense=G, owner=self)


class QuadMeasStochasticOracle:
    """Mini-batch gradient estimator over the measurements (reference StochasticOracle,
    objectives.py:235-273): batches of L indices drawn uniformly with replacement by the host
    generator numpy default_rng(seed) (the reference's draws, in the same order), uploaded, and
    reduced on the device as tau (m / L) sym(a[B]^T diag(res[B]) b[B]); L == m uses every index
    once (the deterministic gradient)."""

    def __init__(self, objective: QuadMeasObjective, L: int, seed: int = 0):
        if L < 1:
            raise ParameterError(f"mini-batch size must be >= 1, got {L}")
        self.objective = objective
        self.L = int(L)
        self.rng = np.random.default_rng(seed)

    def sample_batch(self) -> np.ndarray:
        if self.L == self.objective.m:
            return np.arange(self.objective.m)
        return self.rng.integers(0, self.objective.m, size=self.L)

    def grad_operator(self, x, batch) -> GradientOperator:
        obj = self.objective
        res = obj.residuals(x)
        idx = torch.as_tensor(np.ascontiguousarray(np.asarray(batch, dtype=np.int64))).to(runtime.device())
        if idx.numel() < 1:
            raise ParameterError("batch must contain at least one index")
        s = obj._solver()
        w = obj.tau * obj.m / idx.numel()
        if obj.matrix_free and idx.numel() <= obj.m:  # objectives.py:266-269 (the scratch is sized for m rows)
            return GradientOperator(_lib.GRAD_QUADMEAS, obj.n, qm=QuadMeasOperand(obj, res, w, idx), owner=(obj, idx))
        G = torch.empty((obj.n, obj.n), dtype=torch.float64, device=runtime.device())
        runtime.check(s.lib.megb200_qm_gradient_batch(s.handle, obj.a.data_ptr(), obj.b.data_ptr(), res.data_ptr(),
                                                      idx.data_ptr(), idx.numel(), w, G.data_ptr(), G.stride(0)))
        return GradientOperator(_lib.GRAD_DENSE, obj.n, dense=G, owner=(obj, idx))
