"""Sign- and rotation-invariant comparators shared by the parity tests."""

from __future__ import annotations

import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# Tolerances from BASELINE north_star: 1e-9 relative (fp64), 1e-4 relative (fp32).
TOL = {"f64": 1e-9, "f32": 1e-4}


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def normwise(a, b) -> float:
    """max |a - b| / max |b| (the X-entry metric of SURVEY.md 8c)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def x_norms(ref: dict, iters: int) -> np.ndarray:
    """||X_{t+1}||_F from the recorded lam / eps: sum((1 - eps) lam)^2 + tail^2 (n - r)."""
    lam, eps, n = np.asarray(ref["lam"][:iters]), np.asarray(ref["eps"][:iters]), int(ref["n"])
    r = lam.shape[1]
    tail = eps / (n - r)
    return np.sqrt(np.sum(((1.0 - eps)[:, None] * lam) ** 2, axis=1) + tail**2 * (n - r))


def f_rel_err(a, b, ref: dict, iters: int) -> float:
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    scale = np.maximum(np.abs(b), x_norms(ref, iters) * np.sqrt(2.0 * np.abs(b)))
    return float(np.max(np.abs(a - b) / scale))


def lhs_err(a, b) -> float:
    """|a - b| / max(1, |b|): the certificate lhs can cross zero."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    fin = np.isfinite(b)
    assert np.array_equal(fin, np.isfinite(a))
    return float(np.max(np.abs(a[fin] - b[fin]) / np.maximum(1.0, np.abs(b[fin])))) if fin.any() else 0.0


def compare_trajectory(got: dict, ref: dict, tol: float, iters: int | None = None, f_scale: float = 0.0,
                       f_direct_tol: float | None = None) -> dict:
    """Per-quantity worst errors; asserts each within tol.

    f is compared normwise against f_scale (the magnitude of the summands
    1/2 ||M||_F^2 of the factored evaluation 1/2(||X||^2 - 2<X,M> + ||M||^2)):
    when X -> M the value itself is pure cancellation (config 4 reaches f/F ~ 1e-7).
    Where both sides carry f_direct (1/2 sum_ij (X_ij - M_ij)^2 summed entry by entry), that
    value is compared RELATIVELY at the same tolerance.
    """
    iters = iters if iters is not None else len(ref["shift"])
    errs = {
        "shift": rel_err(got["shift"][:iters], ref["shift"][:iters]),
        "y": rel_err(got["y"][:iters], ref["y"][:iters]),
        "lam": rel_err(got["lam"][:iters], ref["lam"][:iters]),
        "lhs": lhs_err(got["lhs"][:iters], ref["lhs"][:iters]),
        "f": float(np.max(np.abs(np.asarray(got["f"][:iters]) - ref["f"][:iters]))
        / max(float(np.max(np.abs(ref["f"][:iters]))), f_scale)),
    }
    if "f_direct" in got and "f_direct" in ref:
        # entry-by-entry sums on both sides: f compares relatively to max(f, ||X|| ||X - M||), the
        # first-order sensitivity of f = 1/2||X - M||^2 to a relative change of X (|df| <= ||X - M|| ||dX||).
        # Equal to ~2f where noise dominates (cfg1/2/5); where X -> M (noise-free cfg4, f/F ~ 1e-7) a
        # plain relative error of f amplifies the iterate's by ||X|| / ||X - M|| ~ 3e3
        errs["f_direct"] = f_rel_err(got["f_direct"][:iters], ref["f_direct"][:iters], ref, iters)
    for k, v in ref.items():
        if k.startswith("probe_") and k in got and int(k.split("_")[1]) < iters:
            errs[k] = normwise(got[k], v)
    bad = {k: v for k, v in errs.items() if not v <= (f_direct_tol or tol if k == "f_direct" else tol)}
    assert not bad, f"parity failures (tol {tol:g}): {bad}; all: {errs}"
    return errs
