"""Golden fixtures for the quadratic-measurement objective, from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_qm.py

For each case: the reference's `specmeg.objectives.generate_instance` (checksums of a, b, y
are stored so the oracle's restatement can be pinned without the reference), and a MEG
trajectory of `specmeg.meg.lowrank_meg_step` driven by `RecoveryObjective.grad_operator`
(tau * grad f(tau X), materialised densely by the reference for n <= 1024), eta = 1/beta with
the reference preset beta = 0.4 sqrt(r n), eps_t = EpsilonSchedule.experiment(10), svd_seed = t,
from the seeded start of oracle/qm.py.start_iterate.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("SPECMEG_SRC", "/root/reference/pkg/src"))

from specmeg import meg as ref_meg  # noqa: E402
from specmeg import objectives as ref_obj  # noqa: E402

from oracle import qm as oq  # noqa: E402  (start iterate only)

CASES = {"qm_n100_r1": (100, 1, 0), "qm_n60_r3": (60, 3, 1), "qm_n100_r5": (100, 5, 2)}
# mini-batch runs (StochasticOracle, objectives.py:235-273): name -> (n, r, seed, L, oracle seed)
STOCH = {"qms_n100_r5_L1000": (100, 5, 3, 1000, 7), "qms_n60_r3_L3600": (60, 3, 4, 3600, 8)}
T = 15


def checksums(a: np.ndarray) -> np.ndarray:
    return np.array([a.sum(), (a * a).sum(), a.ravel()[0], a.ravel()[-1], a.ravel()[a.size // 3]])


def main():
    out_dir = os.path.dirname(os.path.abspath(__file__))
    sched = ref_meg.EpsilonSchedule.experiment(10.0)
    for name, (n, r, seed) in CASES.items():
        inst = ref_obj.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
        beta = ref_obj.RecoveryObjective.preset_beta(n, r)
        obj = ref_obj.RecoveryObjective(inst, smoothness_hint=beta)
        eta = 1.0 / beta
        x0o = oq.start_iterate(n, r, seed, sched.eval(0))
        x = ref_meg.LowRankIterate(n=n, r=r, V=x0o.V, lam=x0o.lam, eps=x0o.eps)
        rec = {k: [] for k in ("shift", "y", "lam", "eps", "lhs", "f", "V")}
        for t in range(T):
            op = obj.grad_operator(x)
            res = ref_meg.lowrank_meg_step(x, op.apply, eta, sched.eval(t + 1), svd_seed=t)
            x = res.iterate
            rec["shift"].append(res.shift)
            rec["y"].append(res.top_eigenvalues)
            rec["lam"].append(x.lam)
            rec["eps"].append(x.eps)
            rec["lhs"].append(res.cert.lhs_cheap)
            rec["f"].append(obj.value(x))
            rec["V"].append(x.V)
        V_si, w_si = ref_obj.spectral_init(inst, r, seed=seed)
        gap = ref_obj.dual_gap(inst, x, seed=seed)
        np.savez_compressed(
            os.path.join(out_dir, name + ".npz"), n=n, r=r, seed=seed, eta=eta, tau=inst.tau, m=inst.m,
            a_sum=checksums(inst.a), b_sum=checksums(inst.b), y_sum=checksums(inst.y),
            si_V=V_si, si_w=w_si, gap_final=gap,
            V0=x0o.V, lam0=x0o.lam, eps0=x0o.eps, **{k: np.array(v) for k, v in rec.items()})
        print(name, "m =", inst.m, "f:", rec["f"][0], "->", rec["f"][-1])
    for name, (n, r, seed, L, oseed) in STOCH.items():
        inst = ref_obj.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
        beta = ref_obj.RecoveryObjective.preset_beta(n, r)
        obj = ref_obj.RecoveryObjective(inst, smoothness_hint=beta)
        oracle = ref_obj.StochasticOracle(obj, L, seed=oseed)
        eta = 1.0 / beta
        x0o = oq.start_iterate(n, r, seed, sched.eval(0))
        x = ref_meg.LowRankIterate(n=n, r=r, V=x0o.V, lam=x0o.lam, eps=x0o.eps)
        rec = {k: [] for k in ("shift", "y", "lam", "eps", "lhs", "f", "V")}
        for t in range(T):
            batch = oracle.sample_batch()
            op = oracle.grad_operator(x, batch)
            res = ref_meg.lowrank_meg_step(x, op.apply, eta, sched.eval(t + 1), svd_seed=t)
            x = res.iterate
            rec["shift"].append(res.shift)
            rec["y"].append(res.top_eigenvalues)
            rec["lam"].append(x.lam)
            rec["eps"].append(x.eps)
            rec["lhs"].append(res.cert.lhs_cheap)
            rec["f"].append(obj.value(x))
            rec["V"].append(x.V)
        np.savez_compressed(
            os.path.join(out_dir, name + ".npz"), n=n, r=r, seed=seed, L=L, oracle_seed=oseed, eta=eta,
            tau=inst.tau, m=inst.m, V0=x0o.V, lam0=x0o.lam, eps0=x0o.eps,
            **{k: np.array(v) for k, v in rec.items()})
        print(name, "m =", inst.m, "L =", L, "f:", rec["f"][0], "->", rec["f"][-1])


def container_fixture():
    """A small container written by the reference's own save_instance (format pin)."""
    out_dir = os.path.dirname(os.path.abspath(__file__))
    inst = ref_obj.generate_instance(8, 1, kappa=0.5, tau_fraction=0.5, seed=11)
    ref_obj.save_instance(inst, os.path.join(out_dir, "qmi_n8_r1_seed11.bin"))


if __name__ == "__main__":
    main()
    container_fixture()
