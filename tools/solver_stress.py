"""Stress the multi-pass block solver (dev tool): random symmetric operators with separated, clustered,
low-rank and semicircle spectra, dense and CSR, several (n, r, block, subspace); every result is checked
against torch.linalg.eigh (eigenvalues, residuals, orthonormality).

    python tools/solver_stress.py
"""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import runtime  # noqa: E402

dev = runtime.device()
bad = 0
cases = 0


def spectrum(kind, n, rng):
    if kind == "separated":
        return np.concatenate([5.0 - 0.3 * np.arange(12), rng.uniform(-1, 1, n - 12)])
    if kind == "clustered":
        return np.concatenate([3.0 + 1e-6 * np.arange(4), 2.0 + 1e-3 * np.arange(6), rng.uniform(-1, 1.5, n - 10)])
    if kind == "lowrank":
        return np.concatenate([np.linspace(4, 1, 20), 1e-9 * rng.standard_normal(n - 20)])
    return None  # semicircle: plain GOE


for n, kind in itertools.product([160, 700, 2500], ["separated", "clustered", "lowrank", "goe"]):
    rng = np.random.default_rng(n + len(kind))
    if kind == "goe":
        g = torch.randn((n, n), dtype=torch.float64, generator=torch.Generator().manual_seed(n)).to(dev)
        a = (g + g.T) / (2 * np.sqrt(n))
    else:
        ev = torch.tensor(spectrum(kind, n, rng), dtype=torch.float64, device=dev)
        q, _ = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, generator=torch.Generator().manual_seed(n + 1)).to(dev))
        a = (q * ev) @ q.T
        a = (a + a.T) / 2
    a = a.contiguous()
    w = torch.linalg.eigvalsh(a).flip(0).cpu().numpy()
    op = pb.SymmetricOperator(n, dense=a)
    for r, block, sub in [(3, None, None), (10, 14, 98), (10, 18, 64), (8, 16, 64), (20, 32, None), (5, 12, 40)]:
        if r + 1 >= n:
            continue
        tol = 1e-10 if kind != "goe" else 1e-6  # the semicircle edge has no gap: looser, fewer passes
        cases += 1
        try:
            top = pb.lanczos_top_r(op, r, tol=tol, seed=cases, subspace=sub, block=block, max_iter=3000,
                                   return_device=True)
            v = top.eigenvectors
            th = torch.tensor(top.eigenvalues, device=dev)
            res = float((a @ v - v * th).norm(dim=0).max())
            orth = float((v.T @ v - torch.eye(r, dtype=torch.float64, device=dev)).abs().max())
            everr = float(np.abs(top.eigenvalues - w[:r]).max())
            scale = max(1.0, float(np.abs(w).max()))
            ok = res <= 20 * tol * scale and orth <= 1e-9 and everr <= max(1e-8, 100 * tol) * scale
            if not ok:
                bad += 1
            print(f"{'ok ' if ok else 'BAD'} n={n} {kind:9s} r={r} block={block} sub={sub}: passes {top.passes} restarts "
                  f"{top.restarts} res {res:.1e} orth {orth:.1e} ev_err {everr:.1e}", flush=True)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print(f"ERR n={n} {kind} r={r} block={block} sub={sub}: {type(e).__name__}: {str(e)[:160]}", flush=True)
print(f"{cases} cases, {bad} bad")
sys.exit(1 if bad else 0)
