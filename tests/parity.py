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


def lhs_err(a, b) -> float:
    """|a - b| / max(1, |b|): the certificate lhs can cross zero."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    fin = np.isfinite(b)
    assert np.array_equal(fin, np.isfinite(a))
    return float(np.max(np.abs(a[fin] - b[fin]) / np.maximum(1.0, np.abs(b[fin])))) if fin.any() else 0.0


def compare_trajectory(got: dict, ref: dict, tol: float, iters: int | None = None, f_scale: float = 0.0) -> dict:
    """Per-quantity worst errors; asserts each within tol.

    f is compared normwise against f_scale (the magnitude of the summands
    1/2 ||M||_F^2 of the factored evaluation 1/2(||X||^2 - 2<X,M> + ||M||^2)):
    when X -> M the value itself is pure cancellation (config 4 reaches f/F ~ 1e-7).
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
    for k, v in ref.items():
        if k.startswith("probe_") and k in got and int(k.split("_")[1]) < iters:
            errs[k] = normwise(got[k], v)
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"parity failures (tol {tol:g}): {bad}; all: {errs}"
    return errs
