"""Golden lockstep (dense-shadow) run of the UNMODIFIED reference.

    python tests/golden/make_golden_shadow.py

Frobenius objective f(X) = 1/2 ||X - D||^2 of the reference's test_meg.py:28-35, the random
structured start of test_entropy.py:28-35, then T steps of: low-rank MEG (meg.py:327-364 with
the dense `lambda u: g @ u` of test_meg.py:153), the dense shadow of the same update
(shadow_lowrank_step, meg.py:367-385) and its full certificate (certificate_full), the exact
MEG sequence W_{t+1} = exact_meg_step(W_t, grad(W_t), eta) from the same start (meg.py:269-284),
and the Bregman distances B(W_{t+1}, X_{t+1}) dense (entropy.py:76-96) and structured
(entropy.py:128-142) -- the Fig. 1-2 lockstep curve.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.environ.get("SPECMEG_SRC", "/root/reference/pkg/src"))

from specmeg import entropy as ref_ent  # noqa: E402
from specmeg import meg as ref_meg  # noqa: E402
from specmeg.linalg import symmetrize  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def random_lowrank_iterate(n, r, rng, eps):
    """test_entropy.py:28-35 draws."""
    q, _ = np.linalg.qr(rng.standard_normal((n, r)))
    lam = np.sort(rng.dirichlet(np.ones(r) * 3))[::-1]
    lam = np.maximum(lam, 1e-6)
    lam /= lam.sum()
    lam = np.sort(lam)[::-1]
    return ref_meg.LowRankIterate(n=n, r=r, V=q, lam=lam, eps=eps)


def make(n=40, r=3, T=20, eta=0.1, seed=8):
    rng = np.random.default_rng(seed)
    d = symmetrize(rng.standard_normal((n, n))) * 0.3
    x = random_lowrank_iterate(n, r, rng, eps=0.3)
    rec = {"D": d, "V0": x.V, "lam0": x.lam, "eps0": np.float64(x.eps), "n": np.int64(n), "r": np.int64(r),
           "eta": np.float64(eta)}
    w = x.densify()
    keys = ("lhs_cheap", "lhs_full", "holds_full", "bregman", "bregman_structured", "shadow_err")
    out = {k: [] for k in keys}
    ys = []
    for t in range(T):
        eps_next = 0.6 / (t + 11) ** 2
        g = symmetrize(x.densify() - d)
        res = ref_meg.lowrank_meg_step(x, lambda u, g=g: g @ u, eta=eta, eps_next=eps_next, svd_seed=t)
        low, _, y = ref_meg.shadow_lowrank_step(x.densify(), g, eta, eps_next, r)
        cert = ref_meg.certificate_full(y, eps_next, n, r, iteration=t)
        w = ref_meg.exact_meg_step(w, symmetrize(w - d), eta)
        x = res.iterate
        out["lhs_cheap"].append(res.cert.lhs_cheap)
        out["lhs_full"].append(cert.lhs_full)
        out["holds_full"].append(cert.holds_full)
        out["bregman"].append(ref_ent.bregman(w, x.densify()).value)
        out["bregman_structured"].append(ref_ent.bregman_structured(w, x).value)
        out["shadow_err"].append(np.max(np.abs(low - x.densify())))
        ys.append(y)
    rec.update({k: np.asarray(v) for k, v in out.items()})
    rec["y"] = np.asarray(ys)
    rec["W_final"] = w
    rec["X_final"] = x.densify()
    path = os.path.join(OUT, f"shadow_n{n}_r{r}.npz")
    np.savez_compressed(path, **rec)
    print(path, "B(W_T, X_T) =", rec["bregman"][-1])


if __name__ == "__main__":
    make()
