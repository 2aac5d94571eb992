"""Device generator for the synthetic BASELINE inputs (twin of oracle/inputs.py).

The counter-based Gaussian (splitmix64 finaliser + Box-Muller, csrc
megb200_internal.h) is evaluated on the device, so an n = 32768 target is
produced in HBM without host generation or upload.  The planted factor's QR
runs once on the host (n x r, setup only), like the oracle.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib, runtime
from .configs import Workload


def planted_factor(w: Workload) -> np.ndarray:
    """Orthonormal n x r: QR of the stream-1 Gaussian block (counter i*r + j)."""
    s = runtime.solver_for(w.n)
    g = torch.empty((w.n, w.r), dtype=torch.float64, device=runtime.device())
    runtime.check(s.lib.megb200_gen_gaussian(s.handle, w.seed, 1, 0, w.n, w.r, 1.0, 0, g.data_ptr(), g.stride(0)))
    q, _ = np.linalg.qr(g.cpu().numpy())
    return np.ascontiguousarray(q)


def dense_target(w: Workload, U: np.ndarray | None = None) -> torch.Tensor:
    """M = U diag(Lambda) U^T + sigma sym(G) generated in HBM (f64, or rounded to f32)."""
    U = planted_factor(w) if U is None else U
    s = runtime.solver_for(w.n)
    ud = runtime.as_device_f64(U)
    lam = np.ascontiguousarray(np.asarray(w.spectrum, dtype=np.float64))
    tdt = torch.float64 if w.dtype == "f64" else torch.float32
    m = torch.empty((w.n, w.n), dtype=tdt, device=runtime.device())
    runtime.check(s.lib.megb200_gen_dense_target(s.handle, ud.data_ptr(), w.r, _lib.dptr(lam), float(w.noise),
                                                 w.seed, 2, m.data_ptr(), runtime.dtype_code(m), m.stride(0)))
    return m


def sampled_instance(w: Workload, U: np.ndarray | None = None):
    """Config 3 in HBM (twin of oracle/inputs.sampled_instance): the symmetric Bernoulli(p)
    pattern over i <= j (stream 3, canonical counter min(i,j) n + max(i,j)), mirrored, and the
    observed values (U Lambda U^T)_ij + obs_noise N(0,1) (stream 4).  Returns device tensors
    (rowptr int32 (n+1), col int32 (nnz) sorted per row, obs f64 (nnz))."""
    U = planted_factor(w) if U is None else U
    s = runtime.solver_for(w.n)
    dev = runtime.device()
    rowptr = torch.empty(w.n + 1, dtype=torch.int32, device=dev)
    nnz = C.c_int64()
    runtime.check(s.lib.megb200_gen_sampled_pattern(s.handle, w.seed, float(w.sample_p), rowptr.data_ptr(),
                                                    C.byref(nnz)))
    col = torch.empty(nnz.value, dtype=torch.int32, device=dev)
    obs = torch.empty(nnz.value, dtype=torch.float64, device=dev)
    ud = runtime.as_device_f64(U)
    lam = np.ascontiguousarray(np.asarray(w.spectrum, dtype=np.float64))
    runtime.check(s.lib.megb200_gen_sampled_values(s.handle, w.seed, float(w.sample_p), ud.data_ptr(), w.r,
                                                   _lib.dptr(lam), float(w.obs_noise), rowptr.data_ptr(),
                                                   col.data_ptr(), obs.data_ptr()))
    return rowptr, col, obs


def initial_iterate(w: Workload, op_dense: torch.Tensor | None = None, tol: float = 1e-10, csr=None):
    """Warm start of SURVEY.md 8d step 4: top-r eigenpairs of M (device solver, basis 64) -- or of
    (1/p) P_Omega(Mobs) for the sampled config (csr = (rowptr, col, obs)) -- simplex-projected
    weights floored at 1e-12, warm_start_wrap with eps0 = schedule(0)."""
    from .linalg import SymmetricOperator, lanczos_top_r, project_simplex
    from .meg import warm_start_wrap

    if csr is not None:
        op = SymmetricOperator(w.n, csr=tuple(csr), scale=1.0 / w.sample_p)
    else:
        op = SymmetricOperator(w.n, dense=op_dense)
    top = lanczos_top_r(op, w.r, tol=tol, seed=w.seed, subspace=64, return_device=True)
    lam = project_simplex(top.eigenvalues, 1.0)
    lam = lam / lam.sum()
    lam = np.maximum(lam, 1e-12)
    lam = lam / lam.sum()
    return warm_start_wrap(top.eigenvectors, lam, w.eps(0))


def quad_meas_instance(n: int, r_true: int, kappa: float = 0.5, tau_fraction: float = 0.5, seed: int = 0,
                       m: int | None = None):
    """The paper's recovery instance (reference generate_instance, objectives.py:67-105; same
    numpy draws in the same order): unit-Frobenius Gaussian factor v, m = 20 n r spherical
    pairs (a_i, b_i), y0_i = n (a_i.v)(v.b_i), noise of relative size kappa, tau = tau_fraction n.
    Returns (a, b, y, tau) as host arrays (setup only)."""
    rng = np.random.default_rng(seed)
    m = 20 * n * r_true if m is None else m
    v = rng.standard_normal((n, r_true))
    v /= np.linalg.norm(v)
    a = rng.standard_normal((m, n))
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    b = rng.standard_normal((m, n))
    b /= np.linalg.norm(b, axis=1, keepdims=True)
    y0 = n * np.einsum("ij,ij->i", a @ v, b @ v)
    if kappa == 0.0:
        y = y0.copy()
    else:
        d = rng.standard_normal(m)
        d /= np.linalg.norm(d)
        y = y0 + kappa * np.linalg.norm(y0) * d
    return a, b, y, tau_fraction * n


# ---------------------------------------------------------------------------
# "SPECMEG-QMI v1" instance container (reference objectives.py:371-417):
# magic line, sorted-key JSON header line, then raw little-endian float64 arrays
# V_factor (n x r_true), a (m x n), b (m x n), y0 (m), y (m).  Byte-compatible with the
# reference's save_instance / load_instance, so device runs ingest reference instances exactly.

QMI_MAGIC = b"SPECMEG-QMI v1\n"


def save_quad_meas(path: str, *, n: int, r_true: int, m: int, kappa: float, tau: float, seed: int, V_factor, a, b,
                   y0, y) -> None:
    import json

    header = {"n": int(n), "r_true": int(r_true), "m": int(m), "kappa": kappa, "tau": tau, "seed": seed}
    with open(path, "wb") as fh:
        fh.write(QMI_MAGIC)
        fh.write((json.dumps(header, sort_keys=True) + "\n").encode("ascii"))
        for arr in (V_factor, a, b, y0, y):
            fh.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def load_quad_meas(path: str) -> dict:
    """Read a container: dict with n, r_true, m, kappa, tau, seed, V_factor, a, b, y0, y.
    ValueError on a wrong magic line or a truncated payload (the reference's checks)."""
    import json

    with open(path, "rb") as fh:
        magic = fh.readline()
        if magic != QMI_MAGIC:
            raise ValueError(f"{path}: not a SPECMEG-QMI v1 container (magic {magic!r})")
        header = json.loads(fh.readline().decode("ascii"))
        blob = fh.read()
    n, r_true, m = header["n"], header["r_true"], header["m"]
    sizes = [n * r_true, m * n, m * n, m, m]
    if len(blob) != 8 * sum(sizes):
        raise ValueError(f"{path}: truncated container ({len(blob)} payload bytes)")
    parts, off = [], 0
    for size in sizes:
        parts.append(np.frombuffer(blob, dtype="<f8", count=size, offset=8 * off).copy())
        off += size
    v, a, b, y0, y = parts
    return dict(n=n, r_true=r_true, m=m, kappa=header["kappa"], tau=header["tau"], seed=header["seed"],
                V_factor=v.reshape(n, r_true), a=a.reshape(m, n), b=b.reshape(m, n), y0=y0, y=y)
