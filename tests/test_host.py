"""CPU-only tests: the C-ABI library loads and exports every declared symbol, host logic,
config-table agreement, and the multi-process (replica) aggregation of bench.py over gloo."""

import math
import os
import re
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "megb200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(megb200_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for required in ("megb200_lowrank_meg_step", "megb200_top_r", "megb200_logmap_apply", "megb200_operator_apply",
                     "megb200_certificate_cheap", "megb200_dual_gap", "megb200_objective_value"):
        assert required in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2012_10469_b200 import _lib

    lib = _lib.load()
    bound = {name for name, _, _ in _lib.SIGNATURES}
    for sym in declared_symbols():
        assert hasattr(lib, sym), f"{sym} not exported by libmegb200.so"
        assert sym in bound, f"{sym} declared in the header but not bound in _lib.SIGNATURES"
    assert lib.megb200_abi_version() == 1


def test_certificate_arithmetic_through_the_c_abi():
    """certificate_cheap is host arithmetic in the library (meg.py:222-239; test_meg.py:190-217)."""
    import paper_2012_10469_b200 as pb

    rec = pb.certificate_cheap(0.3, 0.8, 0.5, 3, 1)
    assert rec.lhs_cheap == pytest.approx(math.log(1.5), abs=1e-12) and rec.holds_cheap and rec.threshold == 1.0
    assert pb.certificate_cheap(0.0, 0.5, 0.1, 5, 1).lhs_cheap == -math.inf
    with pytest.raises(pb.ParameterError):
        pb.certificate_cheap(0.1, 0.0, 0.1, 5, 1)
    with pytest.raises(pb.ParameterError):
        pb.certificate_cheap(-0.1, 1.0, 0.1, 5, 1)
    full = pb.certificate_full(np.array([0.5, 0.3, 0.2]), 0.5, 3, 1)
    assert full.lhs_full == pytest.approx(math.log(1.2), abs=1e-12)
    assert full.lhs_cheap >= full.lhs_full


def test_no_device_raises_loudly():
    """Without a GPU the product path must fail, never fall back to the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_2012_10469_b200 as pb
    from paper_2012_10469_b200 import _lib

    with pytest.raises((_lib.NativeLibraryError, RuntimeError)):
        pb.LowRankIterate(4, 1, np.eye(4)[:, :1], np.array([1.0]), 0.5)


def test_schedules_and_step_rules():
    import paper_2012_10469_b200 as pb

    assert pb.EpsilonSchedule.experiment(10.0).eval(0) == pytest.approx(0.6 / 121.0, rel=1e-12)
    assert pb.EpsilonSchedule.cubic_det(100.0, 0.5, 0.0).eval(0) == 0.75
    assert pb.EpsilonSchedule.quadratic_stoch(1.0, 0.0).eval(1) == pytest.approx(9.0 / 32.0 / 4.0, rel=1e-12)
    assert pb.StepConfig.one_over_beta(2.0).eval(10) == 0.5
    assert pb.StepConfig.stochastic_fixed(1.0, 2.0, 400).eval(5) == pytest.approx(1.0 / 80.0, rel=1e-12)
    with pytest.raises(pb.ParameterError):
        pb.StepConfig.fixed(0.0)


def test_project_simplex_matches_oracle():
    import paper_2012_10469_b200 as pb
    from oracle import cpu_meg as om

    rng = np.random.default_rng(3)
    for _ in range(50):
        z = rng.standard_normal(7) * 3
        tau = float(rng.uniform(0.1, 5))
        assert np.array_equal(pb.project_simplex(z, tau), om.project_simplex(z, tau))


def test_product_config_table_matches_oracle():
    from oracle import inputs
    from paper_2012_10469_b200 import configs

    for name, w in configs.WORKLOADS.items():
        c = inputs.CONFIGS[name]
        for field in ("n", "r", "iters", "dtype", "block", "kind", "subspace", "eta0", "eta_decay", "sample_p",
                      "obs_noise", "batch", "sigma", "cert_every", "seed", "noise"):
            assert getattr(w, field) == getattr(c, field), (name, field)
        assert np.allclose(w.spectrum, c.spectrum, rtol=0, atol=0)
        assert w.eps(7) == c.eps(7) and w.eta(7) == c.eta(7)


def test_device_generator_constants_match_oracle():
    """The splitmix64 constants / stream ids in megb200_internal.h are the oracle's."""
    from oracle import inputs

    hdr = open(os.path.join(ROOT, "paper_2012_10469_b200", "csrc", "megb200_internal.h")).read()
    assert "0x9E3779B97F4A7C15" in hdr and "0xBF58476D1CE4E5B9" in hdr and "0x94D049BB133111EB" in hdr
    assert int(inputs.GOLDEN) == 0x9E3779B97F4A7C15


# ---------------------------------------------------------------------------
# replica aggregation (bench.py) over gloo, world size 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _replica_worker(rank, world, port, out):
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    per_rank_seconds = [2.0, 3.0][rank]  # rank 1 is the slow replica
    value, tmax = bench.aggregate(per_rank_seconds, steps=100, world=world)
    bench.barrier(world)
    out.put((rank, value, tmax))
    dist.destroy_process_group()


def test_replica_aggregation_max_over_ranks_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for _, value, tmax in res:
        assert tmax == 3.0  # the slowest rank defines the job time
        assert value == pytest.approx(2 * 100 / 3.0)  # whole-job iterations/s over both replicas


def test_qmi_container_matches_reference_bytes(tmp_path):
    """SPECMEG-QMI v1 (objectives.py:371-417): the product reader loads a container written by
    the reference's save_instance (tests/golden/qmi_n8_r1_seed11.bin) to exactly the instance the
    oracle regenerates, and the product writer reproduces the file byte for byte; a wrong magic
    or a truncated payload raises ValueError like the reference."""
    import os

    import numpy as np
    import pytest

    from oracle import qm as oq
    from paper_2012_10469_b200 import inputs as pin

    path = os.path.join(os.path.dirname(__file__), "golden", "qmi_n8_r1_seed11.bin")
    d = pin.load_quad_meas(path)
    inst = oq.generate_instance(8, 1, kappa=0.5, tau_fraction=0.5, seed=11)
    for k in ("a", "b", "y0", "y", "V_factor"):
        assert np.array_equal(d[k], getattr(inst, k)), k
    assert (d["n"], d["r_true"], d["m"], d["tau"], d["seed"]) == (8, 1, inst.m, inst.tau, 11)
    out = tmp_path / "copy.bin"
    pin.save_quad_meas(str(out), **d)
    assert out.read_bytes() == open(path, "rb").read()
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOT-QMI\n" + open(path, "rb").read()[15:])
    with pytest.raises(ValueError):
        pin.load_quad_meas(str(bad))
    cut = tmp_path / "cut.bin"
    cut.write_bytes(open(path, "rb").read()[:-8])
    with pytest.raises(ValueError):
        pin.load_quad_meas(str(cut))


def test_quad_meas_instance_generator_matches_oracle():
    """The product-side instance generator (inputs.quad_meas_instance) draws exactly the oracle's
    (= the reference's) instance: same numpy draws in the same order."""
    import numpy as np

    from oracle import qm as oq
    from paper_2012_10469_b200 import inputs as pin

    for n, r, seed in ((20, 1, 0), (30, 3, 5)):
        a, b, y, tau = pin.quad_meas_instance(n, r, seed=seed)
        inst = oq.generate_instance(n, r, seed=seed)
        assert np.array_equal(a, inst.a) and np.array_equal(b, inst.b) and np.array_equal(y, inst.y)
        assert tau == inst.tau


def test_emit_metrics_csv_format(tmp_path):
    """SPEC harness emit_metrics: exact header, empty cells for absent fields, 17-digit round trip,
    summary as trailing comments; an empty record gives header + summary only."""
    import csv

    import numpy as np

    from paper_2012_10469_b200 import driver

    rows = [{"t": 1, "f_value": 0.1 + 0.2, "eps_t": 1e-3 / 3, "eta_t": 0.5, "cert_cheap_lhs": -np.inf,
             "cert_cheap_holds": 1, "cert_full_lhs": None, "cert_full_holds": None, "bregman_to_exact": None,
             "lambda_rsp1": 2.0 / 3.0, "elapsed_ns": 12345}]
    run = driver.RecoveryRun(iterate=None, rows=rows, summary={"T": 1, "dual_gap": 1.0 / 7.0})
    path = tmp_path / "r.csv"
    driver.emit_metrics(run, str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == driver.RUN_CSV_HEADER
    row = next(csv.DictReader(lines[:2]))
    assert float(row["f_value"]) == 0.1 + 0.2 and float(row["eps_t"]) == 1e-3 / 3
    assert row["cert_cheap_lhs"] == "-inf" and row["cert_full_lhs"] == "" and row["elapsed_ns"] == "12345"
    assert lines[2:] == ["# T = 1", f"# dual_gap = {1.0 / 7.0!r}"]
    empty = tmp_path / "e.csv"
    driver.emit_metrics(driver.RecoveryRun(iterate=None, rows=[], summary={"T": 0}), str(empty))
    assert empty.read_text().splitlines() == [driver.RUN_CSV_HEADER, "# T = 0"]
