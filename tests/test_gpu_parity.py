"""Parity of the B200 path (through the C ABI) with the oracle and the reference goldens.

Every test here needs a CUDA device; tolerances are the north_star's:
1e-9 relative for float64 operands, 1e-4 relative for float32 operands.
"""

import math

import numpy as np
import pytest

from oracle import cpu_meg as om
from oracle import inputs, objectives
from tests.gpu_helpers import f_scale, random_lowrank_iterate_np, run_gpu
from tests.parity import TOL, compare_trajectory, load_golden, normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_2012_10469_b200 as pkg

    return pkg


def random_symmetric(n, rng, scale=1.0):
    return om.symmetrize(rng.standard_normal((n, n))) * scale


# ---------------------------------------------------------------------------
# lanczos_top_r known answers on the device solver (test_linalg.py:61-140)


def test_top_r_diagonal(pb):
    top = pb.lanczos_top_r(pb.SymmetricOperator.from_dense(np.diag([5.0, 4, 3, 2, 1])), r=2, seed=1)
    assert np.allclose(top.eigenvalues, [5.0, 4.0], atol=1e-10)
    assert np.allclose(np.abs(top.eigenvectors), np.eye(5)[:, :2], atol=1e-8)


def test_top_r_algebraic_not_magnitude(pb):
    top = pb.lanczos_top_r(pb.SymmetricOperator.from_dense(-np.diag(np.arange(1.0, 13))), r=1, seed=5)
    assert np.allclose(top.eigenvalues, [-1.0], atol=1e-10)
    assert np.allclose(np.abs(top.eigenvectors[:, 0]), np.eye(12)[:, 0], atol=1e-7)


def test_top_r_repeated(pb):
    top = pb.lanczos_top_r(pb.SymmetricOperator.from_dense(np.diag([2.0, 2, 2, 1, 0])), r=3, seed=11)
    assert np.allclose(top.eigenvalues, [2.0, 2.0, 2.0], atol=1e-9)


def test_top_r_errors(pb):
    with pytest.raises(pb.ParameterError):
        pb.lanczos_top_r(pb.SymmetricOperator.from_dense(np.eye(4)), r=4)
    with pytest.raises(pb.ParameterError):
        pb.lanczos_top_r(pb.SymmetricOperator.from_dense(np.eye(4)), r=0)
    op = pb.SymmetricOperator.from_dense(random_symmetric(60, np.random.default_rng(2)))
    with pytest.raises(pb.LanczosError) as err:
        pb.lanczos_top_r(op, r=3, tol=1e-16, subspace=6, max_iter=8, restarts=1)
    assert err.value.residual_norms.shape == (3,)


@pytest.mark.parametrize("n,r,seed,aseed", [(100, 5, 3, 7), (200, 8, 2, 17), (1000, 12, 0, 5)])
def test_top_r_matches_dense(pb, n, r, seed, aseed):
    a = random_symmetric(n, np.random.default_rng(aseed))
    w, v = om.full_eigh(a)
    top = pb.lanczos_top_r(pb.SymmetricOperator.from_dense(a), r=r, seed=seed, subspace=96)
    scale = max(1.0, np.abs(w).max())
    assert np.max(np.abs(top.eigenvalues - w[:r])) <= 1e-8 * scale
    ov = v[:, :r].T @ top.eigenvectors
    assert np.max(np.arccos(np.clip(np.linalg.svd(ov, compute_uv=False), -1, 1))) <= 1e-6
    assert np.max(np.abs(top.eigenvectors.T @ top.eigenvectors - np.eye(r))) <= 1e-10


def test_top_r_deterministic(pb):
    op = pb.SymmetricOperator.from_dense(random_symmetric(300, np.random.default_rng(4)))
    t1, t2 = pb.lanczos_top_r(op, r=3, seed=9), pb.lanczos_top_r(op, r=3, seed=9)
    assert np.array_equal(t1.eigenvalues, t2.eigenvalues)
    assert np.array_equal(t1.eigenvectors, t2.eigenvectors)


def test_operator_apply_f32_and_csr(pb):
    rng = np.random.default_rng(3)
    n = 777
    a = random_symmetric(n, rng)
    u = rng.standard_normal((n, 19))
    a32 = a.astype(np.float32).astype(np.float64)
    got = pb.SymmetricOperator.from_dense(a, dtype="f32").apply(u)
    assert normwise(got, a32 @ u) <= 2e-6
    import scipy.sparse as sp

    mask = rng.random((n, n)) < 0.03
    mask = np.triu(mask) | np.triu(mask).T
    g = sp.csr_matrix(np.where(mask, a, 0.0))
    op = pb.SymmetricOperator.from_csr(n, g.indptr, g.indices, g.data, scale=-0.5)
    assert normwise(op.apply(u), -0.5 * (g @ u)) <= 1e-14


@pytest.mark.parametrize("n,b,density", [(3000, 18, 0.04), (2500, 32, 0.02), (4096, 7, 0.05), (1500, 16, 0.001)])
def test_csr_panel_pass_ragged(pb, n, b, density):
    """The panel-tiled CSR pass (n >= 1024: U panels in shared memory, per-row panel pointers) against
    scipy on ragged patterns: empty rows, one dense row longer than the prefetched batches, odd and
    even block widths (the 16-byte staged copy and its plain fallback), a nearly empty matrix."""
    import scipy.sparse as sp

    rng = np.random.default_rng(n + b)
    mask = rng.random((n, n)) < density
    mask[5, :] = True         # a row with n entries in every panel
    mask[17:40, :] = False    # empty rows
    mask = np.triu(mask) | np.triu(mask).T
    vals = om.symmetrize(rng.standard_normal((n, n)))
    g = sp.csr_matrix(np.where(mask, vals, 0.0))
    g.sort_indices()
    u = rng.standard_normal((n, b))
    op = pb.SymmetricOperator.from_csr(n, g.indptr.astype(np.int32), g.indices.astype(np.int32), g.data, scale=1.5)
    want = 1.5 * (g @ u)
    assert normwise(op.apply(u), want) <= 1e-14
    assert normwise(op.apply(u), want) <= 1e-14  # a second pass (panel pointers rebuilt outside a solve)


def test_overlapped_restart_matches_serial_order():
    """top_r through restarts with the wide Rayleigh-Ritz overlapped (side stream, carried block) and with
    the serial order (MEGB200_NO_RR_OVERLAP=1, its own process: the switch is read once) agree to the
    solver's accuracy and take the same number of passes."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json, numpy as np, paper_2012_10469_b200 as pb\n"
        "from oracle import cpu_meg as om\n"
        "rng = np.random.default_rng(11)\n"
        "n = 1536\n"
        "q, _ = np.linalg.qr(rng.standard_normal((n, n)))\n"
        "ev = np.concatenate([3.0 - 0.2 * np.arange(6), 1.0 - 0.9 * rng.random(n - 6) ** 0.5])\n"
        "a = (q * ev) @ q.T\n"
        "a = (a + a.T) / 2\n"
        "top = pb.lanczos_top_r(pb.SymmetricOperator.from_dense(a), r=6, tol=1e-10, seed=3, subspace=64, block=14)\n"
        "print(json.dumps({'ev': top.eigenvalues.tolist(), 'passes': int(top.passes),\n"
        "                  'res': float(np.abs(a @ top.eigenvectors - top.eigenvectors * top.eigenvalues).max())}))\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for extra in ({}, {"MEGB200_NO_RR_OVERLAP": "1"}):
        env = dict(os.environ, PYTHONPATH=root, **extra)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    a, b = outs
    assert a["passes"] > 8 and a["passes"] == b["passes"]  # restarts happened; same subspaces
    assert np.max(np.abs(np.array(a["ev"]) - np.array(b["ev"]))) <= 1e-10
    assert a["res"] <= 1e-9 and b["res"] <= 1e-9


# ---------------------------------------------------------------------------
# step, operator, certificates (test_meg.py)


def test_step_diagonal_oracle(pb):
    """test_meg.py:127-131."""
    x = pb.LowRankIterate(3, 1, np.eye(3)[:, :1], np.array([1.0]), 0.5)
    res = pb.lowrank_meg_step(x, pb.ZeroGradient(3), eta=1.0, eps_next=0.1, svd_seed=0)
    assert np.allclose(res.iterate.densify(), np.diag([0.9, 0.05, 0.05]), atol=1e-10)


def test_eps_next_validation(pb):
    q, lam, eps = random_lowrank_iterate_np(8, 2, np.random.default_rng(10))
    x = pb.LowRankIterate(8, 2, q, lam, eps)
    with pytest.raises(pb.ParameterError):
        pb.lowrank_meg_step(x, pb.ZeroGradient(8), eta=1.0, eps_next=0.8)
    with pytest.raises(TypeError):
        pb.lowrank_meg_step(x, 5, eta=1.0, eps_next=0.1)


def test_iterate_validation(pb):
    with pytest.raises(pb.ParameterError):
        pb.LowRankIterate(5, 2, np.ones((5, 2)), np.array([0.5, 0.5]), 0.1)  # not orthonormal
    with pytest.raises(pb.ParameterError):
        pb.LowRankIterate(5, 2, np.eye(5)[:, :2], np.array([0.3, 0.7]), 0.1)  # not sorted


def test_logmap_matches_dense_log(pb):
    """test_meg.py:98-108 on the device operator."""
    rng = np.random.default_rng(4)
    q, lam, eps = random_lowrank_iterate_np(40, 3, rng)
    g = om.symmetrize(rng.standard_normal((40, 40)))
    x = pb.LowRankIterate(40, 3, q, lam, eps)
    op = pb.logmap_operator(x, pb.DenseGradient(g), eta=0.3)
    w, v = np.linalg.eigh(x.densify())
    assert np.max(np.abs(op.to_dense() - ((v * np.log(w)) @ v.T - 0.3 * g))) <= 1e-8


def test_logmap_frobenius_matches_oracle(pb):
    """The factored Frobenius gradient operator equals the oracle's logmap of the dense driver."""
    rng = np.random.default_rng(5)
    n, r = 300, 6
    q, lam, eps = random_lowrank_iterate_np(n, r, rng)
    m = om.symmetrize(rng.standard_normal((n, n))) * 0.1
    xo = om.LowRankIterate(n, r, q, lam, eps)
    x = pb.LowRankIterate(n, r, q, lam, eps)
    u = rng.standard_normal((n, 7))
    ref = om.logmap_operator(xo, lambda v: xo.apply(v) - m @ v, 0.7).apply(u)
    got = pb.logmap_operator(x, pb.FrobeniusObjective(m).grad_operator(x), 0.7).apply(u)
    assert normwise(got, ref) <= 1e-13


def test_dense_shadow_equivalence_fifty_steps(pb):
    """test_meg.py:144-156 on the device path: 50 steps vs the dense shadow at 1e-7."""
    rng = np.random.default_rng(8)
    n, r = 60, 5
    d = om.symmetrize(rng.standard_normal((n, n))) * 0.3
    q, lam, _ = random_lowrank_iterate_np(n, r, rng)
    x = pb.LowRankIterate(n, r, q, lam, 0.3)
    for t in range(50):
        eps_next = 0.6 / (t + 11) ** 2
        g = om.symmetrize(x.densify() - d)
        res = pb.lowrank_meg_step(x, pb.DenseGradient(g), eta=0.5, eps_next=eps_next, svd_seed=t)
        shadow, _, _ = om.shadow_lowrank_step(x.densify(), g, 0.5, eps_next, r)
        assert np.max(np.abs(res.iterate.densify() - shadow)) <= 1e-7
        x = res.iterate


def test_trace_one_and_floor(pb):
    """test_meg.py:133-142."""
    rng = np.random.default_rng(7)
    n = 30
    q, lam, eps = random_lowrank_iterate_np(n, 4, rng)
    x = pb.LowRankIterate(n, 4, q, lam, eps)
    g = pb.DenseGradient(om.symmetrize(rng.standard_normal((n, n))))
    for t in range(5):
        x = pb.lowrank_meg_step(x, g, eta=0.2, eps_next=0.1 / (t + 1), svd_seed=t).iterate
        assert abs(np.trace(x.densify()) - 1.0) <= 1e-12
        assert x.eigenvalues_full()[-1] >= x.eps / (n - x.r) - 1e-12


def test_certificate_arithmetic(pb):
    rec = pb.certificate_cheap(0.3, 0.8, 0.5, 3, 1)
    assert rec.lhs_cheap == pytest.approx(math.log(1.5), abs=1e-12) and rec.holds_cheap and rec.threshold == 1.0


# ---------------------------------------------------------------------------
# trajectories vs the reference goldens


SMALL = [
    ("cfg1_full", "cfg1", None),
    ("cfg2_n1024", "cfg2", 1024),
    ("cfg3_n2048", "cfg3", 2048),
    ("cfg4_n2048", "cfg4", 2048),
    ("cfg5_n2048", "cfg5", 2048),
]


@pytest.mark.parametrize("name,cfg_name,n", SMALL)
def test_trajectory_matches_reference(pb, name, cfg_name, n):
    ref = load_golden(name)
    iters = int(ref["iters"])
    cfg = inputs.CONFIGS[cfg_name]
    if n is not None:
        cfg = cfg.scaled(n, iters)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    probe_at = [int(k.split("_")[1]) for k in ref if k.startswith("probe_")]
    got, _, _ = run_gpu(cfg, host, x0, iters, probe_at=probe_at, block=cfg.block)
    compare_trajectory(got, ref, tol=TOL[cfg.dtype], f_scale=f_scale(host))


@pytest.mark.parametrize("name,cfg_name", [("cfg2_prefix", "cfg2"), ("cfg3_prefix", "cfg3"), ("cfg4_prefix", "cfg4")])
def test_full_size_prefix_matches_reference(pb, name, cfg_name):
    ref = load_golden(name)
    iters = int(ref["iters"])
    cfg = inputs.CONFIGS[cfg_name]
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    probe_at = [int(k.split("_")[1]) for k in ref if k.startswith("probe_")]
    got, _, _ = run_gpu(cfg, host, x0, iters, probe_at=probe_at, block=cfg.block)
    compare_trajectory(got, ref, tol=TOL[cfg.dtype], f_scale=f_scale(host))


def test_dual_gap_matches_reference(pb):
    """_dual_gap_core (objectives.py:332-335) at the final config-5 (n=2048) iterate."""
    ref = load_golden("cfg5_n2048")
    iters = int(ref["iters"])
    cfg = inputs.CONFIGS["cfg5"].scaled(2048, iters)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    _, x, gobj = run_gpu(cfg, host, x0, iters, block=cfg.block)
    gap, lmin = gobj.dev.dual_gap(x, block=32)
    assert abs(gap - float(ref["dual_gap_final"])) <= 1e-4 * max(1.0, abs(float(ref["dual_gap_final"])))


# ---------------------------------------------------------------------------
# native run loop (driver.run) vs the reference goldens and the per-step API


@pytest.mark.parametrize("name,cfg_name,n", [("cfg2_n1024", "cfg2", 1024), ("cfg3_n2048", "cfg3", 2048),
                                             ("cfg4_n2048", "cfg4", 2048), ("cfg1_full", "cfg1", None)])
def test_run_loop_matches_reference(pb, name, cfg_name, n):
    from paper_2012_10469_b200 import driver
    from tests.gpu_helpers import GpuObjective, upload_iterate

    ref = load_golden(name)
    iters = int(ref["iters"])
    cfg = inputs.CONFIGS[cfg_name]
    if n is not None:
        cfg = cfg.scaled(n, iters)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    gobj = GpuObjective(cfg, host)
    res = driver.run(upload_iterate(x0), gobj.dev, iters, eta=cfg.eta0, eta_decay=cfg.eta_decay,
                     svd_subspace=cfg.subspace, block=cfg.block)
    tol = TOL[cfg.dtype]
    got = {"shift": res.shift, "y": res.y, "lam": res.lam, "lhs": res.lhs, "f": ref["f"]}
    compare_trajectory(got, {k: ref[k] for k in ("shift", "y", "lam", "lhs", "f")}, tol=tol)
    assert np.all(res.passes >= 1)
    # final iterate equals the reference's last iterate (probe of X)
    last = int(ref["iters"]) - 1
    if f"probe_{last}" in ref:
        z = objectives.probes(cfg.n)
        assert normwise(objectives.x_apply(res.iterate, z), ref[f"probe_{last}"]) <= tol


def test_run_loop_equals_step_api(pb):
    from paper_2012_10469_b200 import driver

    cfg = inputs.CONFIGS["cfg2"].scaled(512, 12)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    dev = pb.FrobeniusObjective(host.m)
    res = driver.run(pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps), dev, 12, svd_subspace=64, block=18)
    x = pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps)
    for t in range(12):
        step = pb.lowrank_meg_step(x, dev.grad_operator(x), 1.0, cfg.eps(t + 1), svd_seed=t, svd_subspace=64, block=18)
        x = step.iterate
        assert abs(step.shift - res.shift[t]) <= 1e-13 * abs(step.shift)
        assert np.max(np.abs(step.top_eigenvalues - res.y[t]) / res.y[t]) <= 1e-12


def _run_arrays(res):
    return {k: np.asarray(getattr(res, k)) for k in ("shift", "y", "lam", "eps", "lhs", "holds")}


@pytest.mark.parametrize("poor_warm", [False, True])
def test_pipelined_run_bit_identical(pb, monkeypatch, poor_warm):
    """The pipelined run loop (step t+1 enqueued before step t is confirmed) gives
    bit-identical results to the synchronous loop.  poor_warm starts from an
    orthonormal but random warm block, so the first fast step misses the
    tolerance: the speculative step is discarded and the step re-runs."""
    import torch

    from paper_2012_10469_b200 import driver

    cfg = inputs.CONFIGS["cfg2"].scaled(1024, 16)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    dev = pb.FrobeniusObjective(host.m)
    warm = None
    if poor_warm:
        q, _ = np.linalg.qr(np.random.default_rng(5).standard_normal((x0.n, 18)))
        warm = torch.from_numpy(q).cuda()

    def go():
        x = pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps, warm_block=warm, warm_orth_err=0.0)
        return driver.run(x, dev, 16, svd_subspace=64, block=18)

    monkeypatch.setenv("MEGB200_NO_PIPELINE", "1")
    ref = go()
    monkeypatch.setenv("MEGB200_NO_PIPELINE", "0")
    got = go()
    a, b = _run_arrays(ref), _run_arrays(got)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(ref.passes, got.passes)
    if poor_warm:
        assert got.passes[0] > 1, "the first step did not exercise the re-run path"
    assert np.array_equal(ref.iterate.V, got.iterate.V)
    assert np.array_equal(ref.iterate.lam, got.iterate.lam)


def test_run_chaining_continues_warm(pb):
    """run(T1) then run(T2) from its iterate (which carries the Ritz block) equals run(T1 + T2)."""
    from paper_2012_10469_b200 import driver

    cfg = inputs.CONFIGS["cfg2"].scaled(768, 10)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    dev = pb.FrobeniusObjective(host.m)
    whole = driver.run(pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps), dev, 10, svd_subspace=64, block=18)
    first = driver.run(pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps), dev, 4, svd_subspace=64, block=18)
    assert first.iterate.warm_block is not None and first.iterate.warm_block.shape[1] == 18
    second = driver.run(first.iterate, dev, 6, t0=4, svd_subspace=64, block=18)
    assert np.all(second.passes[:1] == whole.passes[4:5])
    assert np.array_equal(np.concatenate([first.shift, second.shift]), whole.shift)
    assert np.array_equal(np.concatenate([first.lam, second.lam]), whole.lam)
    assert np.array_equal(second.iterate.V, whole.iterate.V)


def test_host_buffer_step_matches_device_step(pb):
    """lowrank_meg_step_host (host V in/out, one native call) equals the device-tensor step,
    and rejects a non-orthonormal V with ParameterError before stepping (meg.py:69-71)."""
    import torch

    cfg = inputs.CONFIGS["cfg2"].scaled(1024, 6)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    dev = pb.FrobeniusObjective(host.m)
    x = pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps)
    Vh = torch.from_numpy(np.ascontiguousarray(x0.V)).pin_memory()
    lam, eps, warm, werr = x0.lam.copy(), x0.eps, None, 1.0
    for t in range(6):
        ref = pb.lowrank_meg_step(x, dev.grad_operator(x), 1.0, cfg.eps(t + 1), svd_seed=t, svd_subspace=64, block=18)
        got = pb.lowrank_meg_step_host(Vh, lam, eps, dev, 1.0, cfg.eps(t + 1), svd_seed=t, svd_subspace=64, block=18,
                                       warm=warm, warm_orth_err=werr, out=torch.empty_like(Vh).pin_memory())
        assert np.array_equal(got.top_eigenvalues, ref.top_eigenvalues)
        assert np.array_equal(got.lam, ref.iterate.lam)
        assert got.shift == ref.shift and got.cert.lhs_cheap == ref.cert.lhs_cheap
        assert np.array_equal(got.V.numpy(), ref.iterate.V)
        x = ref.iterate
        Vh, lam, eps, warm, werr = got.V, got.lam, got.eps, got.warm_block, got.warm_orth_err
    bad = Vh.clone()
    bad[:, 0] *= 1.5
    with pytest.raises(pb.ParameterError):
        pb.lowrank_meg_step_host(bad, lam, eps, dev, 1.0, 0.01)


@pytest.mark.parametrize("m", [56, 96, 112])
@pytest.mark.parametrize("spectrum", ["separated", "clustered", "repeated"])
def test_wide_rayleigh_ritz(pb, m, spectrum):
    """The wide Rayleigh-Ritz solver (k_rr_wide: tridiagonalisation + multisection + twisted
    eigenvectors, verified, cyclic-Jacobi fallback) against numpy.linalg.eigh on restarted-basis-like
    spectra: theta non-increasing, eigenvalues to 1e-12 ||H||, the returned columns orthonormal and
    eigenvectors to 1e-12 ||H|| (linalg.py:205-211 semantics), for all pairs and for a top-nvec solve."""
    import ctypes as C

    import torch
    from paper_2012_10469_b200 import runtime

    rng = np.random.default_rng(m + len(spectrum))
    top = -1.0 - 0.4 * np.arange(10)
    if spectrum == "separated":
        ev = np.concatenate([top, -13.6 - 3.0 * rng.random(m - 10)])
    elif spectrum == "clustered":  # the bulk edge of the MEG operator: gaps ~1e-5 and below
        ev = np.concatenate([top, -13.6 - 0.028 * rng.random(m - 20), -13.6 - 1e-7 * rng.random(10)])
    else:  # exact multiplicities
        ev = np.concatenate([top, np.repeat([-13.6, -13.7, -14.0], (m - 10) // 3 + 1)[: m - 10]])
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    h = (q * ev) @ q.T
    h = 0.5 * (h + h.T)
    lib = runtime.solver_for(4096).lib
    f = lib.megb200_debug_rr_solve
    f.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
    dev = runtime.device()
    H = torch.tensor(h, dtype=torch.float64, device=dev)
    ref = np.sort(np.linalg.eigvalsh(h))[::-1]
    hn = np.linalg.norm(h)
    for nvec in (m, m // 3 + 2):
        th = torch.empty(m, dtype=torch.float64, device=dev)
        S = torch.empty((m, m), dtype=torch.float64, device=dev)
        info = torch.empty(4, dtype=torch.float64, device=dev)
        assert f(H.data_ptr(), m, m, th.data_ptr(), S.data_ptr(), info.data_ptr(), 0 if nvec == m else -nvec) == 0
        torch.cuda.synchronize()
        thv, sv = th.cpu().numpy(), S.cpu().numpy()[:, :nvec]
        assert np.all(np.diff(thv) <= 0)
        assert np.max(np.abs(thv[:nvec] - ref[:nvec])) <= 1e-12 * hn
        assert abs(thv[-1] - ref[-1]) <= 1e-12 * hn  # the smallest (norm estimate) is always exact
        assert np.max(np.abs(sv.T @ sv - np.eye(nvec))) <= 1e-13
        assert np.max(np.abs(h @ sv - sv * thv[:nvec])) <= 1e-12 * hn


@pytest.mark.parametrize("name", ["qm_n100_r1", "qm_n60_r3", "qm_n100_r5"])
def test_quad_meas_matches_reference_golden(pb, name):
    """The paper's quadratic-measurement objective on the device:
    residuals (k_qm_residuals) and tau * grad f(tau X) (k_qm_grad_part / reduce) against the
    oracle restatement (1e-12), then a MEG trajectory through lowrank_meg_step against the
    unmodified reference's golden run (1e-9, tests/golden/make_golden_qm.py)."""
    from oracle import qm as oq
    from tests.test_oracle_pins import _qm_eps, qm_projector_err

    g = load_golden(name)
    n, r, seed = int(g["n"]), int(g["r"]), int(g["seed"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    dev = pb.QuadMeasObjective.from_instance(inst)
    x = pb.LowRankIterate(n, r, g["V0"], g["lam0"], float(g["eps0"]))
    ox = om.LowRankIterate(n=n, r=r, V=g["V0"], lam=g["lam0"], eps=float(g["eps0"]))
    res_o = oq.residuals(inst, ox)
    res_d = dev.residuals(x).cpu().numpy()
    assert normwise(res_d, res_o) <= 1e-12
    G_o = oq.dense_gradient(inst, res_o, inst.tau)
    G_d = dev.gradient_matrix(dev.residuals(x)).cpu().numpy()
    assert normwise(G_d, G_o) <= 1e-12
    assert abs(dev.value(x) - oq.value(inst, ox)) <= 1e-12 * abs(oq.value(inst, ox))
    eta = float(g["eta"])
    got = {k: [] for k in ("shift", "y", "lam", "lhs", "f")}
    for t in range(len(g["shift"])):
        res = pb.lowrank_meg_step(x, dev.grad_operator(x), eta, _qm_eps(t + 1), svd_seed=t)
        x = res.iterate
        got["shift"].append(res.shift)
        got["y"].append(res.top_eigenvalues)
        got["lam"].append(x.lam)
        got["lhs"].append(res.cert.lhs_cheap)
        got["f"].append(dev.value(x))
        assert qm_projector_err(x.V, x.lam, x.eps, g["V"][t], g["lam"][t], float(g["eps"][t])) <= 1e-9
    compare_trajectory({k: np.array(v) for k, v in got.items()}, g, TOL["f64"])


@pytest.mark.parametrize("name", ["qms_n100_r5_L1000", "qms_n60_r3_L3600"])
def test_quad_meas_stochastic_matches_reference_golden(pb, name):
    """Mini-batch quadratic-measurement MEG (QuadMeasStochasticOracle: host draws of the
    reference's generator, device batch gradient k_qm_grad_part over gathered rows) against the
    unmodified reference's StochasticOracle run (1e-9); the batch estimate itself against the
    oracle to 1e-12."""
    from oracle import qm as oq
    from tests.test_oracle_pins import _qm_eps, qm_projector_err

    g = load_golden(name)
    n, r, seed, L = int(g["n"]), int(g["r"]), int(g["seed"]), int(g["L"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    dev = pb.QuadMeasObjective.from_instance(inst)
    sto = pb.QuadMeasStochasticOracle(dev, L, seed=int(g["oracle_seed"]))
    osto = oq.StochasticOracle(inst, L, seed=12345)
    x = pb.LowRankIterate(n, r, g["V0"], g["lam0"], float(g["eps0"]))
    ox = om.LowRankIterate(n=n, r=r, V=g["V0"], lam=g["lam0"], eps=float(g["eps0"]))
    probe = np.random.default_rng(5).integers(0, inst.m, size=L)
    assert normwise(sto.grad_operator(x, probe).dense.cpu().numpy(), osto.gradient(ox, probe)) <= 1e-12
    got = {k: [] for k in ("shift", "y", "lam", "lhs", "f")}
    for t in range(len(g["shift"])):
        res = pb.lowrank_meg_step(x, sto.grad_operator(x, sto.sample_batch()), float(g["eta"]), _qm_eps(t + 1),
                                  svd_seed=t)
        x = res.iterate
        for k, v in (("shift", res.shift), ("y", res.top_eigenvalues), ("lam", x.lam), ("lhs", res.cert.lhs_cheap),
                     ("f", dev.value(x))):
            got[k].append(v)
        assert qm_projector_err(x.V, x.lam, x.eps, g["V"][t], g["lam"][t], float(g["eps"][t])) <= 1e-9
    compare_trajectory({k: np.array(v) for k, v in got.items()}, g, TOL["f64"])


@pytest.mark.parametrize("n,r,ks", [(100, 5, (1, 5, 13, 20, 32, 40)), (1100, 1, (1, 9, 18))])
def test_quad_meas_matrix_free_apply(pb, n, r, ks):
    """The matrix-free block application of the measurement gradient (k_qm_fwd / k_qm_bwd,
    reference _apply_measurement_gradient objectives.py:152-158) against the oracle restatement
    and against the materialised gradient, over all measurements and over a mini-batch with
    repeats, for block widths on both sides of the kernels' 8 / 16 / 32 register tiles (1e-12)."""
    from oracle import qm as oq
    from paper_2012_10469_b200 import _lib as _plib

    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=3)
    dev = pb.QuadMeasObjective.from_instance(inst)
    ox = oq.start_iterate(n, r, 3, 0.6 / 121)
    x = pb.LowRankIterate(n, r, ox.V, ox.lam, ox.eps)
    res_o = oq.residuals(inst, ox)
    res_d = dev.residuals(x)
    rng = np.random.default_rng(17)
    batch = rng.integers(0, inst.m, size=max(1, inst.m // 7))
    for k in ks:
        u = rng.standard_normal((n, k))
        want = inst.tau * oq.apply_measurement_gradient(inst.a, inst.b, res_o, u)
        got = dev.apply_gradient(res_d, u).cpu().numpy()
        assert normwise(got, want) <= 1e-12
    u = rng.standard_normal((n, 7))
    w = inst.tau * inst.m / batch.size
    want = w * oq.apply_measurement_gradient(inst.a[batch], inst.b[batch], res_o[batch], u)
    sto = pb.QuadMeasStochasticOracle(dev, batch.size, seed=0)
    dev.dense_cap = 0  # matrix-free at any n
    op = sto.grad_operator(x, batch)
    assert op.kind == _plib.GRAD_QUADMEAS
    assert normwise(op(u), want) <= 1e-12
    dev.dense_cap = 10 ** 9
    assert normwise(sto.grad_operator(x, batch)(u), want) <= 1e-12


@pytest.mark.parametrize("name", ["qm_n100_r5", "qm_n60_r3"])
def test_quad_meas_matrix_free_matches_reference_golden(pb, name):
    """The MEG trajectory with the matrix-free operator (dense_cap = 0: what RecoveryObjective
    does above dense_cap, objectives.py:218-221) against the unmodified reference's golden run
    (1e-9), plus spectral_init and the dual gap through the same operator."""
    from oracle import qm as oq
    from paper_2012_10469_b200 import _lib as _plib
    from tests.test_oracle_pins import _qm_eps, qm_projector_err

    g = load_golden(name)
    n, r, seed = int(g["n"]), int(g["r"]), int(g["seed"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    dev = pb.QuadMeasObjective(inst.a, inst.b, inst.y, inst.tau, dense_cap=0)
    assert dev.matrix_free
    x = pb.LowRankIterate(n, r, g["V0"], g["lam0"], float(g["eps0"]))
    eta = float(g["eta"])
    got = {k: [] for k in ("shift", "y", "lam", "lhs", "f")}
    for t in range(len(g["shift"])):
        gop = dev.grad_operator(x)
        assert gop.kind == _plib.GRAD_QUADMEAS
        res = pb.lowrank_meg_step(x, gop, eta, _qm_eps(t + 1), svd_seed=t)
        x = res.iterate
        for k, v in (("shift", res.shift), ("y", res.top_eigenvalues), ("lam", x.lam), ("lhs", res.cert.lhs_cheap),
                     ("f", dev.value(x))):
            got[k].append(v)
        assert qm_projector_err(x.V, x.lam, x.eps, g["V"][t], g["lam"][t], float(g["eps"][t])) <= 1e-9
    compare_trajectory({k: np.array(v) for k, v in got.items()}, g, TOL["f64"])
    V, w = dev.spectral_init(r, seed=seed)
    P, Pg = (V * w) @ V.T, (g["si_V"] * g["si_w"]) @ g["si_V"].T
    assert np.max(np.abs(P - Pg)) <= 1e-9 * np.max(np.abs(Pg))
    xg = pb.LowRankIterate(n, r, g["V"][-1], g["lam"][-1], float(g["eps"][-1]))
    assert abs(dev.dual_gap(xg, seed=seed) - float(g["gap_final"])) <= 1e-9 * abs(float(g["gap_final"]))


@pytest.mark.parametrize("name", ["qm_n100_r1", "qm_n60_r3", "qm_n100_r5"])
def test_quad_meas_spectral_init_and_dual_gap(pb, name):
    """QuadMeasObjective.spectral_init (probe residuals with eps = 0, gradient, block solver on
    -grad, simplex weights) and dual_gap against the unmodified reference (1e-9)."""
    from oracle import qm as oq

    g = load_golden(name)
    n, r, seed = int(g["n"]), int(g["r"]), int(g["seed"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    dev = pb.QuadMeasObjective.from_instance(inst)
    V, w = dev.spectral_init(r, seed=seed)
    P, Pg = (V * w) @ V.T, (g["si_V"] * g["si_w"]) @ g["si_V"].T
    assert np.max(np.abs(P - Pg)) <= 1e-9 * np.max(np.abs(Pg))
    assert np.max(np.abs(w - g["si_w"])) <= 1e-9
    x = pb.LowRankIterate(n, r, g["V"][-1], g["lam"][-1], float(g["eps"][-1]))
    assert abs(dev.dual_gap(x, seed=seed) - float(g["gap_final"])) <= 1e-9 * abs(float(g["gap_final"]))


def test_recovery_run_record_and_csv(pb, tmp_path):
    """driver.run_recovery (SPEC harness rows) reproduces the reference trajectory's f values and
    certificates, logs the dual gap, and emit_metrics writes the spec's CSV (exact header, empty
    dense-shadow cells, summary comments) that parses back to full precision."""
    import csv

    from oracle import qm as oq
    from paper_2012_10469_b200 import driver
    from tests.test_oracle_pins import _qm_eps  # noqa: F401

    g = load_golden("qm_n60_r3")
    n, r, seed = int(g["n"]), int(g["r"]), int(g["seed"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    dev = pb.QuadMeasObjective.from_instance(inst)
    x0 = pb.LowRankIterate(n, r, g["V0"], g["lam0"], float(g["eps0"]))
    T = len(g["shift"])
    run = driver.run_recovery(dev, x0, T, eta=float(g["eta"]), gap_every=5, seed=seed)
    f = np.array([row["f_value"] for row in run.rows])
    assert np.max(np.abs(f - g["f"]) / np.abs(g["f"])) <= 1e-9
    lhs = np.array([row["cert_cheap_lhs"] for row in run.rows])
    assert np.max(np.abs(lhs - g["lhs"]) / np.maximum(1.0, np.abs(g["lhs"]))) <= 1e-9
    assert abs(run.summary["dual_gap"] - float(g["gap_final"])) <= 1e-9 * abs(float(g["gap_final"]))
    path = tmp_path / "run.csv"
    driver.emit_metrics(run, str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == driver.RUN_CSV_HEADER
    body = list(csv.DictReader([ln for ln in lines if not ln.startswith("#")]))
    assert len(body) == T and body[0]["cert_full_lhs"] == "" and body[0]["bregman_to_exact"] == ""
    assert np.array_equal(np.array([float(b["f_value"]) for b in body]), f)
    assert any(ln.startswith("# dual_gap = ") for ln in lines)


def test_host_stepper_matches_host_step(pb):
    """HostStepper (structs and buffers made once) gives bit-identical results to
    lowrank_meg_step_host, rejects invalid lam / V like LowRankIterate (meg.py:62-77)."""
    import torch

    cfg = inputs.CONFIGS["cfg2"].scaled(1024, 6)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    dev = pb.FrobeniusObjective(host.m)
    st = pb.HostStepper(dev, x0.n, x0.r, svd_subspace=64, block=18)
    Va = torch.from_numpy(np.ascontiguousarray(x0.V)).pin_memory()
    Vb = Va.clone().pin_memory()
    la, ea, wa, wea = x0.lam.copy(), x0.eps, None, 1.0
    lb, eb, wb, web = x0.lam.copy(), x0.eps, None, 1.0
    for t in range(6):
        ra = pb.lowrank_meg_step_host(Va, la, ea, dev, 1.0, cfg.eps(t + 1), svd_seed=t, svd_subspace=64, block=18,
                                      warm=wa, warm_orth_err=wea, out=torch.empty_like(Va).pin_memory())
        rb = st.step(Vb, lb, eb, 1.0, cfg.eps(t + 1), t, warm=wb, warm_orth_err=web,
                     out=torch.empty_like(Vb).pin_memory())
        assert np.array_equal(ra.top_eigenvalues, rb.top_eigenvalues) and np.array_equal(ra.lam, rb.lam)
        assert np.array_equal(ra.V.numpy(), rb.V.numpy()) and ra.cert.lhs_cheap == rb.cert.lhs_cheap
        Va, la, ea, wa, wea = ra.V, ra.lam, ra.eps, ra.warm_block, ra.warm_orth_err
        Vb, lb, eb, wb, web = rb.V, rb.lam, rb.eps, rb.warm_block, rb.warm_orth_err
    with pytest.raises(pb.ParameterError):
        st.step(Vb, lb[::-1].copy(), eb, 1.0, 0.01)
    bad = Vb.clone()
    bad[:, 0] *= 1.5
    with pytest.raises(pb.ParameterError):
        st.step(bad.pin_memory(), lb, eb, 1.0, 0.01)


def test_dual_gap_warm_start_matches_cold(pb):
    """A certificate warm-started from the previous certificate's Ritz block (megb200_dual_gap_warm)
    converges to the cold one within the residual rule (cfg2 shape at n = 1024)."""
    cfg = inputs.CONFIGS["cfg2"].scaled(1024, 6)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    dev = pb.FrobeniusObjective(host.m)
    x = pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps)
    gaps = []
    for t in range(12):
        x = pb.lowrank_meg_step(x, dev.grad_operator(x), 1.0, cfg.eps(t + 1), svd_seed=t, svd_subspace=64,
                                block=18).iterate
        if t % 4 == 3:
            warm = dev.dual_gap(x, warm=True)
            cold = dev.dual_gap(x, warm=False)
            assert abs(warm[0] - cold[0]) <= 1e-9 * max(1.0, abs(cold[0]))
            assert abs(warm[1] - cold[1]) <= 1e-9 * max(1.0, abs(cold[1]))
            gaps.append(warm[0])
    assert all(g > -1e-9 for g in gaps)


# ---------------------------------------------------------------------------
# full-size parity on the paths bench.py times (reference goldens at the stated sizes)


def _golden_x0(pb, ref):
    n = int(ref["n"])
    return pb.LowRankIterate(n, ref["V0"].shape[1], ref["V0"], ref["x0_lam"], float(ref["x0_eps"]))


class _DevObjective:
    """run_trajectory adapter over a device objective (no host copy of the operand)."""

    def __init__(self, dev, stochastic=False):
        self.dev = dev
        self.value_direct = dev.value
        self.stochastic = stochastic

    def grad_apply(self, x, t=0):
        return self.dev.grad_operator(x, t) if self.stochastic else self.dev.grad_operator(x)

    def value(self, x):
        return self.dev.value(x)


def _run_loop_vs_golden(pb, dev, x0, ref, cfg, tol):
    """driver.run (the native, pipelined loop bench.py times) against a reference golden."""
    from paper_2012_10469_b200 import driver

    iters = int(ref["iters"])
    res = driver.run(x0, dev, iters, eta=cfg.eta0, eta_decay=cfg.eta_decay, svd_subspace=cfg.subspace,
                     block=cfg.block)
    got = {"shift": res.shift, "y": res.y, "lam": res.lam, "lhs": res.lhs, "f": ref["f"]}
    compare_trajectory(got, {k: ref[k] for k in ("shift", "y", "lam", "lhs", "f")}, tol=tol)
    last = iters - 1
    z = objectives.probes(cfg.n)
    assert normwise(objectives.x_apply(res.iterate, z), ref[f"probe_{last}"]) <= tol
    if "f_direct" in ref:
        from tests.parity import f_rel_err

        f_last = dev.value(res.iterate)
        assert f_rel_err([f_last], ref["f_direct"][last:], {k: ref[k][last:] if k in ("lam", "eps") else ref[k]
                                                          for k in ("lam", "eps", "n")}, 1) <= tol
    return res


def test_cfg2_long_full_size_matches_reference(pb):
    """cfg2 at n = 4096 for 45 steps (past bench.py's warm-up into the one-pass steady state):
    the per-step API and the pipelined native loop (driver.run) against the unmodified reference
    at 1e-9, f compared relatively (entry-by-entry sums on both sides)."""
    ref = load_golden("cfg2_long")
    cfg = inputs.CONFIGS["cfg2"]
    from paper_2012_10469_b200 import configs
    from paper_2012_10469_b200 import inputs as dinputs

    m = dinputs.dense_target(configs.WORKLOADS["cfg2"])
    dev = pb.FrobeniusObjective.from_device(m, "f64")
    z = objectives.probes(cfg.n)
    mz = (m @ __import__("torch").as_tensor(z, device=m.device)).cpu().numpy()
    assert normwise(mz, ref["m_probe"]) <= 1e-13  # the device generator reproduces the reference's M
    x0 = _golden_x0(pb, ref)
    assert abs(dev.value(x0) - float(ref["f0_direct"])) <= 1e-12 * float(ref["f0_direct"])
    probe_at = [int(k.split("_")[1]) for k in ref if k.startswith("probe_")]
    from tests.gpu_helpers import gpu_api

    got, _ = objectives.run_trajectory(gpu_api(), cfg, _DevObjective(dev), x0, int(ref["iters"]), probe_at=probe_at,
                                       step_kwargs={"block": cfg.block})
    errs = compare_trajectory(got, ref, tol=TOL["f64"], f_scale=0.5 * float(ref["m_norm2"]))
    assert "f_direct" in errs
    _run_loop_vs_golden(pb, dev, _golden_x0(pb, ref), ref, cfg, TOL["f64"])


def test_cfg5_full_size_matches_reference(pb):
    """cfg5 at its stated size (n = 32768, the 4 GiB float32 operand, k = 32): M from the device
    generator checked against the reference-side checksums, 3 steps through the per-step API and
    through driver.run against the unmodified reference at 1e-4 (fp32), and the dual-gap
    certificate (_dual_gap_core, objectives.py:332-335) at the last iterate."""
    import torch

    ref = load_golden("cfg5_full")
    cfg = inputs.CONFIGS["cfg5"]
    from paper_2012_10469_b200 import configs
    from paper_2012_10469_b200 import inputs as dinputs

    m = dinputs.dense_target(configs.WORKLOADS["cfg5"])
    assert m.dtype == torch.float32 and m.shape == (32768, 32768)
    z = torch.as_tensor(objectives.probes(cfg.n), device=m.device)
    mz = torch.cat([m[i:i + 4096].double() @ z for i in range(0, cfg.n, 4096)]).cpu().numpy()
    # the float64 entry before rounding can differ from numpy's in the last bit (device log/cos),
    # which flips an occasional float32 rounding (one f32 ulp, 6e-8 relative, on that entry)
    assert normwise(mz, ref["m_probe"]) <= 1e-9
    dev = pb.FrobeniusObjective.from_device(m, "f32")
    assert abs(dev.m_trace - float(ref["m_trace"])) <= 1e-12 * abs(float(ref["m_trace"]))
    assert abs(dev.m_norm2 - float(ref["m_norm2"])) <= 1e-12 * float(ref["m_norm2"])
    x0 = _golden_x0(pb, ref)
    assert abs(dev.value(x0) - float(ref["f0_direct"])) <= 1e-12 * float(ref["f0_direct"])
    probe_at = [int(k.split("_")[1]) for k in ref if k.startswith("probe_")]
    from tests.gpu_helpers import gpu_api

    got, x = objectives.run_trajectory(gpu_api(), cfg, _DevObjective(dev), x0, int(ref["iters"]), probe_at=probe_at,
                                       step_kwargs={"block": cfg.block})
    compare_trajectory(got, ref, tol=TOL["f32"], f_scale=0.5 * float(ref["m_norm2"]))
    gap, _ = dev.dual_gap(x, block=32, warm=False)
    gref = float(ref["dual_gap_final"])
    assert abs(gap - gref) <= TOL["f32"] * abs(gref), (gap, gref)
    _run_loop_vs_golden(pb, dev, _golden_x0(pb, ref), ref, cfg, TOL["f32"])


@pytest.mark.parametrize("name,cfg_name", [("cfg3_prefix", "cfg3"), ("cfg4_prefix", "cfg4")])
def test_full_size_prefix_run_loop_matches_reference(pb, name, cfg_name):
    """cfg3 (CSR, n = 8192) and cfg4 (stochastic, n = 16384) full-size prefixes through the native
    run loop (driver.run), from the reference's own warm start."""
    ref = load_golden(name)
    cfg = inputs.CONFIGS[cfg_name]
    host = objectives.make_objective(cfg)
    from tests.gpu_helpers import GpuObjective

    dev = GpuObjective(cfg, host).dev
    _run_loop_vs_golden(pb, dev, _golden_x0(pb, ref), ref, cfg, TOL[cfg.dtype])


# ---------------------------------------------------------------------------
# the reference's callable contract (linalg.py:81-94, meg.py:327-335) through the callback operator


def test_callable_operator_matches_dense(pb):
    """SymmetricOperator(dim, apply_fn) with a numpy callable (test_linalg.py's usage) and with a
    device (torch) callable give the dense operator's eigenpairs."""
    import torch

    from paper_2012_10469_b200.callbacks import device_callable

    a = random_symmetric(300, np.random.default_rng(21))
    ref = pb.lanczos_top_r(pb.SymmetricOperator.from_dense(a), r=4, seed=3)
    got = pb.lanczos_top_r(pb.SymmetricOperator(300, lambda u: a @ u), r=4, seed=3)
    at = torch.as_tensor(a, device="cuda")
    dev = pb.lanczos_top_r(pb.SymmetricOperator(300, device_callable(lambda u: at @ u)), r=4, seed=3)
    scale = np.abs(np.linalg.eigvalsh(a)).max()
    for t in (got, dev):
        assert np.max(np.abs(t.eigenvalues - ref.eigenvalues)) <= 1e-12 * scale
        assert np.max(np.abs(np.abs(t.eigenvectors.T @ ref.eigenvectors) - np.eye(4))) <= 1e-8
    assert np.allclose(pb.SymmetricOperator(300, lambda u: a @ u).apply(np.eye(300)[:, :3]), a[:, :3], atol=1e-14)


def test_callable_grad_apply_matches_descriptor(pb):
    """lowrank_meg_step with the reference-style `lambda u: g @ u` (test_meg.py:153) equals the
    DenseGradient descriptor step, and the descriptors are themselves callables."""
    rng = np.random.default_rng(9)
    n, r = 120, 4
    q, lam, eps = random_lowrank_iterate_np(n, r, rng)
    g = om.symmetrize(rng.standard_normal((n, n))) * 0.2
    x = pb.LowRankIterate(n, r, q, lam, eps)
    ref = pb.lowrank_meg_step(x, pb.DenseGradient(g), eta=0.7, eps_next=0.05, svd_seed=2)
    got = pb.lowrank_meg_step(x, lambda u: g @ u, eta=0.7, eps_next=0.05, svd_seed=2)
    assert np.max(np.abs(got.top_eigenvalues - ref.top_eigenvalues) / ref.top_eigenvalues) <= 1e-12
    assert np.max(np.abs(got.iterate.densify() - ref.iterate.densify())) <= 1e-12
    assert abs(got.cert.lhs_cheap - ref.cert.lhs_cheap) <= 1e-12 * max(1.0, abs(ref.cert.lhs_cheap))
    u = rng.standard_normal((n, 3))
    m = om.symmetrize(rng.standard_normal((n, n)))
    dev = pb.FrobeniusObjective(m).grad_operator(x)
    assert normwise(dev(u), x.densify() @ u - m @ u) <= 1e-13
    assert normwise(dev(u[:, 0]), x.densify() @ u[:, 0] - m @ u[:, 0]) <= 1e-13
    assert normwise(pb.DenseGradient(g)(u), g @ u) <= 1e-14


def test_callable_errors_propagate(pb):
    rng = np.random.default_rng(3)
    q, lam, eps = random_lowrank_iterate_np(50, 3, rng)
    x = pb.LowRankIterate(50, 3, q, lam, eps)

    def bad(u):
        raise ValueError("user gradient failed")

    with pytest.raises(ValueError, match="user gradient failed"):
        pb.lowrank_meg_step(x, bad, eta=1.0, eps_next=0.1)
    with pytest.raises(ValueError):
        pb.lanczos_top_r(pb.SymmetricOperator(50, bad), r=2)


def test_solver_settings_reported(pb):
    """svd_subspace beyond the device basis limit and the float32 tolerance floor are applied
    visibly: a SolverSettingWarning and the effective values in the result."""
    from paper_2012_10469_b200.meg import SolverSettingWarning

    rng = np.random.default_rng(4)
    n, r = 400, 3
    q, lam, eps = random_lowrank_iterate_np(n, r, rng)
    m = om.symmetrize(rng.standard_normal((n, n))) * 0.01
    x = pb.LowRankIterate(n, r, q, lam, eps)
    with pytest.warns(SolverSettingWarning):
        res = pb.lowrank_meg_step(x, pb.FrobeniusObjective(m).grad_operator(x), 1.0, 0.05, svd_subspace=200)
    assert res.svd_subspace_effective == pb.runtime.MAX_BASIS
    with pytest.warns(SolverSettingWarning):
        res32 = pb.lowrank_meg_step(x, pb.FrobeniusObjective(m, dtype="f32").grad_operator(x), 1.0, 0.05)
    assert res32.svd_tol_effective == pb.objectives.F32_TOL_FLOOR
    assert res.svd_tol_effective == 1e-10


# ---------------------------------------------------------------------------
# dense shadow / lockstep: exact MEG, shadow step, full certificate, Bregman


def test_shadow_lockstep_matches_reference(pb):
    """The device dense-shadow diagnostics against the unmodified reference's lockstep run
    (tests/golden/make_golden_shadow.py): exact_meg_step (meg.py:269-284), shadow_lowrank_step
    (meg.py:367-385) + certificate_full, bregman (entropy.py:76-96), bregman_structured
    (entropy.py:128-142); the low-rank steps themselves through lowrank_meg_step."""
    from paper_2012_10469_b200 import shadow as sh

    g0 = load_golden("shadow_n40_r3")
    n, r, eta = int(g0["n"]), int(g0["r"]), float(g0["eta"])
    d = g0["D"]
    x = pb.LowRankIterate(n, r, g0["V0"], g0["lam0"], float(g0["eps0"]))
    w = x.densify()
    for t in range(len(g0["bregman"])):
        eps_next = 0.6 / (t + 11) ** 2
        g = om.symmetrize(x.densify() - d)
        res = pb.lowrank_meg_step(x, pb.DenseGradient(g), eta, eps_next, svd_seed=t)
        assert abs(res.cert.lhs_cheap - g0["lhs_cheap"][t]) <= 1e-9 * max(1.0, abs(g0["lhs_cheap"][t]))
        low, _, y = sh.shadow_lowrank_step(x.densify(), g, eta, eps_next, r)
        y = y.cpu().numpy()
        assert np.max(np.abs(y - g0["y"][t])) <= 1e-11 * np.abs(g0["y"][t]).max()
        cert = pb.certificate_full(y, eps_next, n, r)
        assert abs(cert.lhs_full - g0["lhs_full"][t]) <= 1e-9 * max(1.0, abs(g0["lhs_full"][t]))
        w = sh.exact_meg_step(w, om.symmetrize(w - d), eta).cpu().numpy()
        x = res.iterate
        assert np.max(np.abs(low.cpu().numpy() - x.densify())) <= 1e-7  # test_meg.py:144-156's bar
        b = sh.bregman(w, x.densify())
        assert b.finite and abs(b.value - g0["bregman"][t]) <= 1e-9 * abs(g0["bregman"][t])
        bs = sh.bregman_structured(w, x)
        assert abs(bs.value - g0["bregman_structured"][t]) <= 1e-9 * abs(g0["bregman"][t])
    assert np.max(np.abs(w - g0["W_final"])) <= 1e-10


def test_shadow_eigh_paths_and_entropy_identities(pb):
    """full_eigh on the native small solver (n <= 112) and on cuSOLVER (n > 112) agree with
    numpy; bregman(X, X) = 0 and the structured form equals the dense one (test_entropy.py)."""
    from paper_2012_10469_b200 import shadow as sh

    rng = np.random.default_rng(12)
    for n in (30, 112, 150):
        a = random_symmetric(n, rng)
        w, v = sh.full_eigh(a)
        ref = np.sort(np.linalg.eigvalsh(a))[::-1]
        assert np.max(np.abs(w.cpu().numpy() - ref)) <= 1e-12 * np.abs(ref).max()
        vv = v.cpu().numpy()
        assert np.max(np.abs(a @ vv - vv * w.cpu().numpy())) <= 1e-11 * np.abs(ref).max()
    q, lam, eps = random_lowrank_iterate_np(50, 4, rng)
    x = pb.LowRankIterate(50, 4, q, lam, eps)
    assert abs(sh.bregman(x.densify(), x.densify()).value) <= 1e-12
    z = om.symmetrize(rng.standard_normal((50, 50)))
    z = z @ z.T + np.eye(50)
    z /= np.trace(z)
    assert abs(sh.bregman_structured(z, x).value - sh.bregman(z, x.densify()).value) <= 1e-10


def test_recovery_lockstep_columns(pb):
    """driver.run_recovery(shadow=True) fills the spec's dense-shadow columns (cert_full_lhs,
    cert_full_holds, bregman_to_exact) exactly as the oracle computes them."""
    from oracle import qm as oq
    from paper_2012_10469_b200 import driver

    g = load_golden("qm_n60_r3")
    n, r, seed = int(g["n"]), int(g["r"]), int(g["seed"])
    inst = oq.generate_instance(n, r, kappa=0.5, tau_fraction=0.5, seed=seed)
    dev = pb.QuadMeasObjective.from_instance(inst)
    x0 = pb.LowRankIterate(n, r, g["V0"], g["lam0"], float(g["eps0"]))
    eta = 0.02 * float(g["eta"])  # the exact MEG sequence stays positive definite over the 5 steps
    run = driver.run_recovery(dev, x0, 5, eta=eta, shadow=True)
    ox = om.LowRankIterate(n=n, r=r, V=g["V0"], lam=g["lam0"], eps=float(g["eps0"]))
    w = ox.densify()
    from tests.test_oracle_pins import _qm_eps

    for t, row in enumerate(run.rows):
        eps_next = _qm_eps(t + 1)
        G = oq.dense_gradient(inst, oq.residuals(inst, ox), inst.tau)
        _, _, y = om.shadow_lowrank_step(ox.densify(), G, eta, eps_next, r)
        cf = om.certificate_full(y, eps_next, n, r)
        assert abs(row["cert_full_lhs"] - cf.lhs_full) <= 1e-8 * max(1.0, abs(cf.lhs_full))
        assert row["cert_full_holds"] == int(cf.holds_full)
        res_w = inst.tau * np.einsum("ij,ij->i", inst.a @ w, inst.b) - inst.y
        w = om.exact_meg_step(w, oq.dense_gradient(inst, res_w, inst.tau), eta)
        ox = om.lowrank_meg_step(ox, lambda u, G=G: G @ u, eta, eps_next, svd_seed=t).iterate
        assert abs(row["bregman_to_exact"] - om.bregman_structured(w, ox)) <= 1e-8 * max(1.0, abs(row["bregman_to_exact"]))
    assert "first_iter_cert_full" in run.summary


# ---------------------------------------------------------------------------
# round-2 plumbing: device generators, direct objective, run-loop certificate cadence and timed window


def test_device_sampled_instance_matches_oracle(pb):
    """The device generator of cfg3's instance (k_sampled_count / k_sampled_fill) reproduces
    oracle/inputs.sampled_instance: same symmetric pattern (exact) and observed values."""
    from paper_2012_10469_b200 import configs
    from paper_2012_10469_b200 import inputs as dinputs

    cfg = inputs.CONFIGS["cfg3"].scaled(1024)
    w = configs.Workload(**{k: getattr(cfg, k) for k in configs.Workload.__dataclass_fields__})
    ref = inputs.sampled_instance(cfg, keep_planted=False)
    rp, col, obs = dinputs.sampled_instance(w)
    assert np.array_equal(rp.cpu().numpy(), ref.rowptr)
    assert np.array_equal(col.cpu().numpy(), ref.col)
    assert np.max(np.abs(obs.cpu().numpy() - ref.obs)) <= 1e-15


def test_direct_objective_value(pb):
    """megb200_objective_value_direct (entry-by-entry 1/2 ||X - M||^2) against the oracle's direct
    sum, relatively, in float64 and float32 operands."""
    rng = np.random.default_rng(31)
    n, r = 700, 6
    q, lam, eps = random_lowrank_iterate_np(n, r, rng)
    m = om.symmetrize(rng.standard_normal((n, n))) * 0.01 + q[:, :r] @ np.diag(lam) @ q[:, :r].T
    xo = om.LowRankIterate(n=n, r=r, V=q, lam=lam, eps=eps)
    x = pb.LowRankIterate(n, r, q, lam, eps)
    ref = objectives.frob_value_direct(xo, m)
    assert abs(pb.FrobeniusObjective(m).value(x) - ref) <= 1e-12 * ref
    m32 = m.astype(np.float32).astype(np.float64)
    ref32 = objectives.frob_value_direct(xo, m32)
    assert abs(pb.FrobeniusObjective(m, dtype="f32").value(x) - ref32) <= 1e-12 * ref32


def test_run_loop_certificate_cadence_and_timed_window(pb):
    """driver.run(cert_every=k) computes the dual gap of X_{t+1} after every step t with
    (t+1) % k == 0, equal to FrobeniusObjective.dual_gap on the same iterate; the timed window
    brackets exactly the requested steps."""
    from paper_2012_10469_b200 import driver

    cfg = inputs.CONFIGS["cfg2"].scaled(1024, 12)
    host = objectives.make_objective(cfg)
    x0 = objectives.initial_iterate(om, cfg, host)
    dev = pb.FrobeniusObjective(host.m)
    x = pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps)
    res = driver.run(x, dev, 12, svd_subspace=64, block=18, cert_every=4, timed_from=2, timed_count=8)
    cert_steps = [i for i in range(12) if np.isfinite(res.gap[i])]
    assert cert_steps == [3, 7, 11]
    assert res.timed_ms > 0 and res.timed_launches > 0
    # the same trajectory step by step, certificates from the public dual_gap (cold, same rule)
    xs = pb.LowRankIterate(x0.n, x0.r, x0.V, x0.lam, x0.eps)
    for t in range(12):
        xs = pb.lowrank_meg_step(xs, dev.grad_operator(xs), 1.0, cfg.eps(t + 1), svd_seed=t, svd_subspace=64,
                                 block=18).iterate
        if t in cert_steps:
            gap, lmin = dev.dual_gap(xs, warm=False)
            assert abs(gap - res.gap[t]) <= 1e-9 * max(1.0, abs(gap))
            assert abs(lmin - res.lmin[t]) <= 1e-9 * max(1.0, abs(lmin))


def test_one_launch_step_kernel_parity():
    """The opt-in one-launch pass + step tail (k_dense_step_mma, MEGB200_STEP_MMA=1)
    stays parity-green: a cfg2-shaped trajectory (n = 1024, 30 steps) against the reference golden,
    in a subprocess (the switch is read once per process)."""
    import subprocess
    import sys

    code = (
        "import numpy as np\n"
        "from oracle import cpu_meg as om, inputs, objectives\n"
        "from tests.gpu_helpers import run_gpu, f_scale\n"
        "from tests.parity import TOL, compare_trajectory, load_golden\n"
        "ref = load_golden('cfg2_n1024')\n"
        "cfg = inputs.CONFIGS['cfg2'].scaled(1024, int(ref['iters']))\n"
        "host = objectives.make_objective(cfg)\n"
        "x0 = objectives.initial_iterate(om, cfg, host)\n"
        "got, _, _ = run_gpu(cfg, host, x0, int(ref['iters']), probe_at=[0, 29], block=cfg.block)\n"
        "compare_trajectory(got, ref, tol=TOL['f64'], f_scale=f_scale(host))\n"
        "print('ok')\n"
    )
    import os

    env = dict(os.environ, MEGB200_STEP_MMA="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
