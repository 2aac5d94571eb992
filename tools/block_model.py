"""Numpy model of the device block eigensolver (design tool, not shipped, not the oracle).

Mirrors the control flow of paper_2012_10469_b200/csrc/megb200_solver.cu so the
algorithm (block thick-restart Lanczos with CholQR2, warm start from the
previous step's Ritz block) can be checked for pass counts and parity on the
CPU before the kernels exist.
"""

from __future__ import annotations

import math
import sys

import numpy as np


def orth_block(q, w, rng, scale):
    """CGS2 against q, CholQR2 with breakdown replacement.  Returns (Q_new, R)."""
    b = w.shape[1]
    for _ in range(2):
        if q.shape[1]:
            w = w - q @ (q.T @ w)
    g = w.T @ w
    r1 = np.zeros((b, b))
    bad = []
    # pivot-safe Cholesky
    for j in range(b):
        s = g[j, j] - r1[:j, j] @ r1[:j, j]
        if s <= (1e-13 * scale) ** 2:
            bad.append(j)
            continue
        r1[j, j] = math.sqrt(s)
        for k in range(j + 1, b):
            r1[j, k] = (g[j, k] - r1[:j, j] @ r1[:j, k]) / r1[j, j]
    for j in bad:
        r1[j, j] = 1.0  # placeholder; column replaced below, relation row zeroed
    w = np.linalg.solve(r1.T, w.T).T
    for j in bad:
        r1[j, :] = 0.0
        v = rng.standard_normal(w.shape[0])
        for _ in range(2):
            if q.shape[1]:
                v = v - q @ (q.T @ v)
            good = [k for k in range(b) if k not in bad or k < j]
            if good:
                wg = w[:, good]
                v = v - wg @ (wg.T @ v)  # not exactly orthonormal yet; CholQR below fixes
        w[:, j] = v / np.linalg.norm(v)
    if q.shape[1]:
        w = w - q @ (q.T @ w)
    g2 = w.T @ w
    r2 = np.linalg.cholesky(g2).T
    w = np.linalg.solve(r2.T, w.T).T
    return w, r2 @ r1


def block_top(apply, n, nreq, b, m, tol, seed, warm=None, max_passes=200, keep=None):
    rng = np.random.default_rng(seed)
    cap = m + b
    Q = np.zeros((n, cap))
    AQ = np.zeros((n, cap))
    H = np.zeros((cap, cap))
    start = rng.standard_normal((n, b))
    if warm is not None:
        start[:, : warm.shape[1]] = warm
    Q[:, :b], _ = orth_block(Q[:, :0], start, rng, 1.0)
    cols = 0
    passes = 0
    scale = 1.0
    keep = keep if keep is not None else m - b
    while passes < max_passes:
        AQ[:, cols : cols + b] = apply(Q[:, cols : cols + b])
        passes += 1
        c = Q[:, : cols + b].T @ AQ[:, cols : cols + b]
        H[: cols + b, cols : cols + b] = c
        cols += b
        Hs = np.triu(H[:cols, :cols])
        Hs = Hs + np.triu(Hs, 1).T
        th, S = np.linalg.eigh(Hs)
        order = np.argsort(-th)
        th, S = th[order], S[:, order]
        scale = max(1.0, np.abs(th).max())
        Q[:, cols : cols + b], R = orth_block(Q[:, :cols], AQ[:, cols - b : cols] - Q[:, :cols] @ c, rng, scale)
        est = np.linalg.norm(R @ S[cols - b : cols, :nreq], axis=0)
        if np.all(est <= tol * scale):
            X = Q[:, :cols] @ S[:, :nreq]
            AX = AQ[:, :cols] @ S[:, :nreq]
            res = np.linalg.norm(AX - X * th[:nreq], axis=0)
            if np.all(res <= tol * scale):
                ritz = Q[:, :cols] @ S[:, :b]
                return th[:nreq], X, res, passes, ritz
        if cols + b > m:
            k = keep
            Xk = Q[:, :cols] @ S[:, :k]
            AXk = AQ[:, :cols] @ S[:, :k]
            nxt = Q[:, cols : cols + b].copy()
            Q[:, :k] = Xk
            AQ[:, :k] = AXk
            H[:] = 0
            H[np.arange(k), np.arange(k)] = th[:k]
            Q[:, k : k + b] = nxt
            cols = k
    raise RuntimeError(f"no convergence in {passes} passes; est {est}")


def meg_step_block(x, grad_apply, eta, eps_next, b, m, tol, seed, warm):
    from oracle import cpu_meg as om

    op = om.logmap_operator(x, grad_apply, eta)
    th, X, res, passes, ritz = block_top(op.apply, x.n, x.r + 1, b, m, tol, seed, warm)
    shift = th[0]
    y = np.exp(th - shift)
    lam = y[: x.r] / y[: x.r].sum()
    lam = lam / lam.sum()
    nxt = om.LowRankIterate(n=x.n, r=x.r, V=X[:, : x.r], lam=lam, eps=eps_next)
    cert = om.certificate_cheap(float(y[x.r]), float(y.sum()), eps_next, x.n, x.r)
    return nxt, y, shift, cert, passes, ritz


def main(name="cfg2_n1024", cfg_name="cfg2", n=1024, b=18, m=72, warm_on=True):
    sys.path.insert(0, ".")
    from oracle import cpu_meg as om, inputs, objectives
    from tests.parity import load_golden

    ref = load_golden(name)
    iters = int(ref["iters"])
    cfg = inputs.CONFIGS[cfg_name]
    if n is not None:
        cfg = cfg.scaled(n, iters)
    obj = objectives.make_objective(cfg)
    x = objectives.initial_iterate(om, cfg, obj)
    warm = None
    plist = []
    errs = []
    for t in range(iters):
        x, y, shift, cert, passes, ritz = meg_step_block(
            x, obj.grad_apply(x, t), cfg.eta(t), cfg.eps(t + 1), b, m, 1e-10, t, warm
        )
        if warm_on:
            warm = ritz
        plist.append(passes)
        errs.append(max(abs(shift - ref["shift"][t]) / abs(ref["shift"][t]),
                        np.max(np.abs(y - ref["y"][t]) / ref["y"][t]),
                        abs(cert.lhs_cheap - ref["lhs"][t]) / max(1, abs(ref["lhs"][t]))))
    print(name, "passes", plist, "max err", max(errs))


if __name__ == "__main__":
    import ast

    kw = {}
    for a in sys.argv[1:]:
        k, v = a.split("=")
        try:
            kw[k] = ast.literal_eval(v)
        except Exception:
            kw[k] = v
    main(**kw)
