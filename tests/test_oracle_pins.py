"""Pin the CPU oracle (oracle/cpu_meg.py) before trusting it.

1. Every known-answer / property test the reference suite holds for the hot
   path, restated against the oracle (reference test file:line cited).
2. The golden trajectories produced by the unmodified reference
   (tests/golden/make_golden.py) reproduced by the oracle on the same seeded
   inputs.
"""

import math

import numpy as np
import pytest

from oracle import cpu_meg as om
from oracle import inputs, objectives
from tests.parity import compare_trajectory, load_golden


def random_symmetric(n, rng, scale=1.0):
    return om.symmetrize(rng.standard_normal((n, n))) * scale


def random_lowrank_iterate(n, r, rng, eps=None):
    """test_entropy.py:28-35 fixture, restated."""
    q, _ = np.linalg.qr(rng.standard_normal((n, r)))
    lam = np.sort(rng.dirichlet(np.ones(r) * 3))[::-1]
    lam = np.maximum(lam, 1e-6)
    lam /= lam.sum()
    lam = np.sort(lam)[::-1]
    if eps is None:
        eps = float(rng.uniform(0.01, 0.5))
    return om.LowRankIterate(n=n, r=r, V=q, lam=lam, eps=eps)


# ---------------------------------------------------------------------------
# Lanczos known answers (test_linalg.py:61-140)


def test_lanczos_diagonal_top2():
    top = om.lanczos_top_r(om.SymmetricOperator.from_dense(np.diag([5.0, 4, 3, 2, 1])), r=2, seed=1)
    assert np.allclose(top.eigenvalues, [5.0, 4.0], atol=1e-10)
    assert np.allclose(np.abs(top.eigenvectors), np.eye(5)[:, :2], atol=1e-8)


def test_lanczos_algebraic_not_magnitude():
    op = om.SymmetricOperator.from_dense(-np.diag(np.arange(1.0, 13)))
    top = om.lanczos_top_r(op, r=1, seed=5)
    assert np.allclose(top.eigenvalues, [-1.0], atol=1e-10)


def test_lanczos_repeated_eigenvalues():
    top = om.lanczos_top_r(om.SymmetricOperator.from_dense(np.diag([2.0, 2, 2, 1, 0])), r=3, seed=11)
    assert np.allclose(top.eigenvalues, [2.0, 2.0, 2.0], atol=1e-9)


def test_lanczos_parameter_error_and_failure():
    with pytest.raises(om.ParameterError):
        om.lanczos_top_r(om.SymmetricOperator.from_dense(np.eye(4)), r=4)
    rng = np.random.default_rng(2)
    op = om.SymmetricOperator.from_dense(random_symmetric(60, rng))
    with pytest.raises(om.LanczosError) as err:
        om.lanczos_top_r(op, r=3, tol=1e-16, subspace=6, max_iter=8, restarts=1)
    assert err.value.residual_norms.shape == (3,)


@pytest.mark.parametrize("n,r,seed,aseed", [(100, 5, 3, 7), (200, 8, 2, 17)])
def test_lanczos_matches_dense(n, r, seed, aseed):
    a = random_symmetric(n, np.random.default_rng(aseed))
    w, v = om.full_eigh(a)
    top = om.lanczos_top_r(om.SymmetricOperator.from_dense(a), r=r, seed=seed)
    assert np.max(np.abs(top.eigenvalues - w[:r])) <= 1e-8 * max(1.0, np.abs(w).max())
    ov = v[:, :r].T @ top.eigenvectors
    assert np.max(np.arccos(np.clip(np.linalg.svd(ov, compute_uv=False), -1, 1))) <= 1e-6


def test_lanczos_deterministic():
    op = om.SymmetricOperator.from_dense(random_symmetric(40, np.random.default_rng(4)))
    t1, t2 = om.lanczos_top_r(op, r=3, seed=9), om.lanczos_top_r(op, r=3, seed=9)
    assert np.array_equal(t1.eigenvectors, t2.eigenvectors)


# ---------------------------------------------------------------------------
# step / operator / certificate known answers (test_meg.py)


def test_step_diagonal_oracle():
    """test_meg.py:127-131."""
    x = om.LowRankIterate(n=3, r=1, V=np.eye(3)[:, :1], lam=np.array([1.0]), eps=0.5)
    res = om.lowrank_meg_step(x, lambda u: np.zeros_like(u), eta=1.0, eps_next=0.1, svd_seed=0)
    assert np.allclose(res.iterate.densify(), np.diag([0.9, 0.05, 0.05]), atol=1e-10)


def test_logmap_matches_dense_log():
    """test_meg.py:98-108."""
    rng = np.random.default_rng(4)
    x = random_lowrank_iterate(40, 3, rng)
    g = om.symmetrize(rng.standard_normal((40, 40)))
    op = om.logmap_operator(x, lambda u: g @ u, eta=0.3)
    w, v = np.linalg.eigh(x.densify())
    assert np.max(np.abs(op.to_dense() - ((v * np.log(w)) @ v.T - 0.3 * g))) <= 1e-8


def test_dense_shadow_equivalence_fifty_steps():
    """test_meg.py:144-156: 50 low-rank steps vs the dense shadow, 1e-7."""
    rng = np.random.default_rng(8)
    n, r = 60, 5
    d = om.symmetrize(rng.standard_normal((n, n))) * 0.3
    x = random_lowrank_iterate(n, r, rng, eps=0.3)
    for t in range(50):
        eps_next = 0.6 / (t + 11) ** 2
        g = om.symmetrize(x.densify() - d)
        res = om.lowrank_meg_step(x, lambda u, g=g: g @ u, eta=0.5, eps_next=eps_next, svd_seed=t)
        shadow, _, _ = om.shadow_lowrank_step(x.densify(), g, 0.5, eps_next, r)
        assert np.max(np.abs(res.iterate.densify() - shadow)) <= 1e-7
        x = res.iterate


def test_certificate_arithmetic():
    """test_meg.py:190-217."""
    rec = om.certificate_cheap(0.3, 0.8, 0.5, 3, 1)
    assert rec.lhs_cheap == pytest.approx(math.log(1.5), abs=1e-12) and rec.holds_cheap and rec.threshold == 1.0
    assert om.certificate_cheap(0.0, 0.5, 0.1, 5, 1).lhs_cheap == -math.inf
    full = om.certificate_full(np.array([0.5, 0.3, 0.2]), 0.5, 3, 1)
    assert full.lhs_full == pytest.approx(math.log(1.2), abs=1e-12)
    for n in (2, 5, 50):
        assert om.certificate_full(np.full(n, 1.0 / n), 0.5, n, 1).lhs_full == pytest.approx(
            math.log(2 * (n - 1) / n), abs=1e-12
        )
    with pytest.raises(om.ParameterError):
        om.certificate_cheap(0.1, 0.0, 0.1, 5, 1)


def test_warm_start_and_schedules():
    """test_meg.py:263-289, 341-377."""
    x1 = om.warm_start_wrap(np.eye(2)[:, :1], np.array([1.0]), eps0=0.1)
    assert np.allclose(x1.densify(), np.diag([0.95, 0.05]), atol=1e-14)
    assert om.EpsilonSchedule.experiment(10.0).eval(0) == pytest.approx(0.6 / 121.0, rel=1e-12)
    assert om.EpsilonSchedule.cubic_det(100.0, 0.5, 0.0).eval(0) == 0.75
    assert inputs.CONFIGS["cfg2"].eps(0) == pytest.approx(0.6 / 121.0, rel=1e-15)


def test_project_simplex():
    """test_linalg.py:158-187."""
    assert np.allclose(om.project_simplex(np.array([0.2, 0.3])), [0.45, 0.55], atol=1e-12)
    assert np.allclose(om.project_simplex(np.array([2.0, -1.0])), [1.0, 0.0], atol=1e-12)


# ---------------------------------------------------------------------------
# golden trajectories from the reference itself


def f_scale(obj):
    if hasattr(obj, "m_norm2"):
        return 0.5 * obj.m_norm2
    return 0.5 * float(obj.inst.obs @ obj.inst.obs)


GOLDEN_SMALL = [
    ("cfg1_full", "cfg1", None),
    ("cfg2_n1024", "cfg2", 1024),
    ("cfg3_n2048", "cfg3", 2048),
    ("cfg4_n2048", "cfg4", 2048),
    ("cfg5_n2048", "cfg5", 2048),
]


@pytest.mark.parametrize("name,cfg_name,n", GOLDEN_SMALL)
def test_oracle_reproduces_reference_trajectory(name, cfg_name, n):
    ref = load_golden(name)
    iters = int(ref["iters"])
    cfg = inputs.CONFIGS[cfg_name]
    if n is not None:
        cfg = cfg.scaled(n, iters)
    obj = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, obj)
    z = objectives.probes(cfg.n)
    assert np.max(np.abs(objectives.x_apply(x0, z) - ref["x0_probe"])) <= 1e-12
    probe_at = [int(k.split("_")[1]) for k in ref if k.startswith("probe_")]
    got, _ = objectives.run_trajectory(om, cfg, obj, x0, iters, probe_at=probe_at)
    # converged-quantity parity between two valid solvers: <= ~1e-11.  f itself (entry
    # sums) amplifies iterate differences by ~||X|| / ||X - M|| (3e3 on cfg4, where X -> M)
    compare_trajectory(got, ref, tol=1e-10, f_scale=f_scale(obj), f_direct_tol=1e-9)


def test_generator_is_counter_based():
    """Same counters -> same draws regardless of the chunking used to request them."""
    key = inputs.stream_key(0, 2)
    a = inputs.gaussian(key, np.arange(1000, dtype=np.uint64))
    b = np.concatenate([inputs.gaussian(key, np.arange(i, i + 100, dtype=np.uint64)) for i in range(0, 1000, 100)])
    assert np.array_equal(a, b)
    assert abs(a.mean()) < 0.1 and abs(a.std() - 1.0) < 0.1
    cfg = inputs.CONFIGS["cfg2"].scaled(64)
    m = inputs.dense_target(cfg)
    assert np.array_equal(m, m.T)


# ---------------------------------------------------------------------------
# quadratic-measurement objective: oracle/qm.py pinned to the
# reference's instance generator and trajectories (tests/golden/make_golden_qm.py)

QM_CASES = ["qm_n100_r1", "qm_n60_r3", "qm_n100_r5"]


def _qm_checksums(a):
    a = np.asarray(a)
    return np.array([a.sum(), (a * a).sum(), a.ravel()[0], a.ravel()[-1], a.ravel()[a.size // 3]])


def _qm_eps(t):
    return min(0.6 / (t + 11.0) ** 2, 0.75)  # EpsilonSchedule.experiment(10) (meg.py:182-190)


def qm_projector_err(V, lam, eps, Vg, lamg, epsg):
    """normwise difference of the two iterates' dense forms (sign/rotation invariant)."""
    n, r = V.shape
    X = (1 - eps) * (V * lam) @ V.T + eps / (n - r) * (np.eye(n) - V @ V.T)
    Xg = (1 - epsg) * (Vg * lamg) @ Vg.T + epsg / (n - r) * (np.eye(n) - Vg @ Vg.T)
    return float(np.max(np.abs(X - Xg)) / np.max(np.abs(Xg)))


@pytest.mark.parametrize("name", QM_CASES)
def test_qm_oracle_matches_reference_golden(name):
    from oracle import qm as oq

    g = load_golden(name)
    n, r, seed = int(g["n"]), int(g["r"]), int(g["seed"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    for key, arr in (("a_sum", inst.a), ("b_sum", inst.b), ("y_sum", inst.y)):
        np.testing.assert_allclose(_qm_checksums(arr), g[key], rtol=1e-13, atol=0)
    assert inst.tau == float(g["tau"]) and inst.m == int(g["m"])
    x = om.LowRankIterate(n=n, r=r, V=g["V0"], lam=g["lam0"], eps=float(g["eps0"]))
    eta = float(g["eta"])
    got = {k: [] for k in ("shift", "y", "lam", "lhs", "f")}
    for t in range(len(g["shift"])):
        G = oq.dense_gradient(inst, oq.residuals(inst, x), inst.tau)
        res = om.lowrank_meg_step(x, lambda u, G=G: G @ u, eta, _qm_eps(t + 1), svd_seed=t)
        x = res.iterate
        got["shift"].append(res.shift)
        got["y"].append(res.top_eigenvalues)
        got["lam"].append(x.lam)
        got["lhs"].append(res.cert.lhs_cheap)
        got["f"].append(oq.value(inst, x))
        assert qm_projector_err(x.V, x.lam, x.eps, g["V"][t], g["lam"][t], float(g["eps"][t])) <= 1e-10
    compare_trajectory({k: np.array(v) for k, v in got.items()}, g, 1e-10)


@pytest.mark.parametrize("name", ["qms_n100_r5_L1000", "qms_n60_r3_L3600"])
def test_qm_stochastic_oracle_matches_reference_golden(name):
    """Mini-batch runs (StochasticOracle, objectives.py:235-273): the oracle's batches and
    estimates reproduce the reference trajectory."""
    from oracle import qm as oq

    g = load_golden(name)
    n, r, seed, L = int(g["n"]), int(g["r"]), int(g["seed"]), int(g["L"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    sto = oq.StochasticOracle(inst, L, seed=int(g["oracle_seed"]))
    x = om.LowRankIterate(n=n, r=r, V=g["V0"], lam=g["lam0"], eps=float(g["eps0"]))
    got = {k: [] for k in ("shift", "y", "lam", "lhs", "f")}
    for t in range(len(g["shift"])):
        G = sto.gradient(x, sto.sample_batch())
        res = om.lowrank_meg_step(x, lambda u, G=G: G @ u, float(g["eta"]), _qm_eps(t + 1), svd_seed=t)
        x = res.iterate
        for k, v in (("shift", res.shift), ("y", res.top_eigenvalues), ("lam", x.lam), ("lhs", res.cert.lhs_cheap),
                     ("f", oq.value(inst, x))):
            got[k].append(v)
        assert qm_projector_err(x.V, x.lam, x.eps, g["V"][t], g["lam"][t], float(g["eps"][t])) <= 1e-10
    compare_trajectory({k: np.array(v) for k, v in got.items()}, g, 1e-10)


@pytest.mark.parametrize("name", QM_CASES)
def test_qm_spectral_init_and_dual_gap_oracle(name):
    """spectral_init (objectives.py:293-323) and dual_gap (:326-341) restated, against the reference."""
    from oracle import qm as oq

    g = load_golden(name)
    n, r, seed = int(g["n"]), int(g["r"]), int(g["seed"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    V, w = oq.spectral_init(inst, r, seed=seed)
    P, Pg = (V * w) @ V.T, (g["si_V"] * g["si_w"]) @ g["si_V"].T
    assert np.max(np.abs(P - Pg)) <= 1e-10 * np.max(np.abs(Pg))
    assert np.max(np.abs(w - g["si_w"])) <= 1e-10
    x = om.LowRankIterate(n=n, r=r, V=g["V"][-1], lam=g["lam"][-1], eps=float(g["eps"][-1]))
    assert abs(oq.dual_gap(inst, x, seed=seed) - float(g["gap_final"])) <= 1e-9 * abs(float(g["gap_final"]))


def test_oracle_shadow_lockstep_matches_reference():
    """Dense-shadow diagnostics of the oracle (exact_meg_step, shadow_lowrank_step,
    certificate_full, bregman, bregman_structured) reproduce the unmodified reference's lockstep
    run (tests/golden/make_golden_shadow.py)."""
    g0 = load_golden("shadow_n40_r3")
    n, r, eta = int(g0["n"]), int(g0["r"]), float(g0["eta"])
    d = g0["D"]
    x = om.LowRankIterate(n=n, r=r, V=g0["V0"], lam=g0["lam0"], eps=float(g0["eps0"]))
    w = x.densify()
    for t in range(len(g0["bregman"])):
        eps_next = 0.6 / (t + 11) ** 2
        g = om.symmetrize(x.densify() - d)
        res = om.lowrank_meg_step(x, lambda u, g=g: g @ u, eta, eps_next, svd_seed=t)
        low, _, y = om.shadow_lowrank_step(x.densify(), g, eta, eps_next, r)
        assert np.max(np.abs(y - g0["y"][t]) / np.abs(g0["y"][t]).max()) <= 1e-11
        cert = om.certificate_full(y, eps_next, n, r)
        assert abs(cert.lhs_full - g0["lhs_full"][t]) <= 1e-10 * max(1.0, abs(g0["lhs_full"][t]))
        w = om.exact_meg_step(w, om.symmetrize(w - d), eta)
        x = res.iterate
        assert np.max(np.abs(low - x.densify())) <= 1e-7
        assert abs(om.bregman(w, x.densify())[0] - g0["bregman"][t]) <= 1e-9 * abs(g0["bregman"][t])
        assert abs(om.bregman_structured(w, x) - g0["bregman_structured"][t]) <= 1e-9 * abs(g0["bregman"][t])
    assert np.max(np.abs(w - g0["W_final"])) <= 1e-10


def test_qm_matrix_free_apply_oracle():
    """oracle.qm.apply_measurement_gradient (objectives.py:152-158) equals the materialised
    gradient's product (objectives.py:155-156) -- the identity the reference's dense_cap switch
    relies on (objectives.py:214-221) -- for a vector and for a block."""
    from oracle import qm as oq

    inst = oq.generate_instance(40, 2, kappa=0.5, tau_fraction=0.5, seed=4)
    rng = np.random.default_rng(0)
    res = rng.standard_normal(inst.m)
    G = oq.dense_gradient(inst, res, 1.0)
    for u in (rng.standard_normal(40), rng.standard_normal((40, 6))):
        got = oq.apply_measurement_gradient(inst.a, inst.b, res, u)
        assert np.max(np.abs(got - G @ u)) <= 1e-13 * np.max(np.abs(G @ u))
