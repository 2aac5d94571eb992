#!/usr/bin/env python
"""Benchmark: low-rank MEG iterations/sec on B200 (BASELINE.json metric).

Headline (`--workload`, default cfg2 = BASELINE configs[1]): n = 4096, r = 10, float64,
block k = r + 8 = 18, dense 1/2||X - M||_F^2, eta = 1, eps_t = 0.6/(t+11)^2, one trajectory
from the warm start.  A *step* is one `lowrank_meg_step` (meg.py:327-364) continuing it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload cfg2] [--workloads cfg3,cfg4,cfg5|none]

Timing.  The native run loop (megb200_meg_run, pipelined) runs W + K steps in one call; CUDA
events recorded on the solver stream at the start of step W and at the end of step W + K - 1
bracket exactly the K timed steps (the first W steps, including the cold first solve, are the
warm-up), with barrier + synchronize around the call.  Inputs are resident in HBM.  L2 is not
flushed: the operands of every timed workload exceed the 126 MB L2 (cfg2 134 MB streamed
evict-first; cfg4 1.07 GB; cfg5 4.29 GB); cfg3's CSR (40 MB) is re-streamed every pass and
its gathers are what it is bound by -- see `config.l2` per workload.

`e2e`: the same metric through the reference-facing host-buffer entry point
(megb200_lowrank_meg_step_host / pb.HostStepper): every step uploads V from pinned host memory,
validates it, steps, and reads V_next back into pinned host memory.

`roofline`: the dominant kernel (the streamed operand pass): algorithmic bytes per pass
(operand as stored + 2 n k 8) / its mean duration, from CUDA events bracketing EVERY pass
kernel of a further K-step window of the same loop (the events cost the pass its programmatic-
launch overlap, so this is a slight under-estimate), against MEASURED_PEAKS.json.

`workloads`: the same device / e2e / roofline measurement for configs 3, 4 and 5 (cfg5 with its
dual-gap certificate every 10 iterations inside the timed steps), beside the headline.

N > 1: one independent replica per GPU (the path does not shard at this tier);
without torchrun in the environment, `--gpus N` re-launches itself under
torch.distributed.run.  Time = max over ranks; value = N * K / that time.
`--impl reference` times the CPU restatement of the reference (oracle/, "port") on the
host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "low-rank MEG iterations/sec at n=4096–32768, r=5–20; achieved HBM GB/s vs peak"
UNIT = "iterations/s"
KIND_DESC = {"dense": "deterministic low-rank MEG, dense 1/2||X-M||_F^2",
             "sampled": "sampled-entry low-rank MEG, 1/2 sum_Omega (X_ij-M_ij)^2, 5% symmetric CSR",
             "stochastic": "stochastic low-rank MEG, X-M + rank-64 minibatch noise (b=64, sigma=0.05)"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="cfg2", help="headline workload")
    ap.add_argument("--workloads", default="cfg3,cfg4,cfg5", help="extra workloads reported beside it, or 'none'")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU baseline sampling")
    ap.add_argument("--ref-budget", type=float, default=150.0, help="max seconds of reference-arm timed steps")
    ap.add_argument("--clock-ms", type=int, default=50, help="nvidia-smi clock sampling interval (ms)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (replicas only)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` without a torchrun environment: run N local replicas under torch.distributed.run."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def init_dist(world: int, backend: str):
    import torch.distributed as dist

    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank scalar (timing rule: the slowest rank defines the job)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def aggregate(per_rank_seconds: float, steps: int, world: int, device=None) -> tuple[float, float]:
    """(whole-job iterations/s, max seconds): every replica runs `steps` steps."""
    tmax = max_over_ranks(per_rank_seconds, world, device)
    return world * steps / tmax, tmax


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, interval_ms: int = 50):
        self.gpu = gpu_index
        self.interval = max(1, int(interval_ms))
        self.proc = None
        self.path = tempfile.mktemp(prefix="clocks_", suffix=".csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.interval)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for name, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


# ---------------------------------------------------------------------------
# workload descriptions (shared by both arms so the config dicts agree)


def workload_table():
    """The five BASELINE configs (paper_2012_10469_b200/configs.py; the oracle keeps a twin)."""
    from paper_2012_10469_b200 import configs

    return configs.WORKLOADS


def operand_bytes(w) -> int:
    if w.kind == "sampled":
        return 0  # data-dependent (nnz); reported by the device arm
    return w.n * w.n * (8 if w.dtype == "f64" else 4)


def l2_note(w) -> str:
    if w.kind == "sampled":
        return ("not flushed: the CSR operand (~40 MB) is smaller than the 126 MB L2 and is re-read by every one of "
                "the ~27 passes of a step, so it can stay L2-resident between passes; the panel pass is bound by "
                "shared-memory wavefronts, not by HBM (profiles/)")
    mb = operand_bytes(w) / 1e6
    return f"not flushed: operand {mb:.0f} MB > 126 MB L2, streamed evict-first every pass"


def config_dict(name: str, world: int) -> dict:
    w = workload_table()[name]
    d = {"workload": f"{name}: {KIND_DESC[w.kind]}, n={w.n}, r={w.r}, {w.dtype}, block k={w.block}, "
                     f"eta={'eta0/sqrt(t+1)' if w.eta_decay else w.eta0}, eps_t=0.6/(t+11)^2, warm start from the "
                     f"rank-{w.r} projection" + (f", dual-gap certificate every {w.cert_every} iterations"
                                                 if w.cert_every else ""),
         "n": w.n, "r": w.r, "block": w.block, "operand_dtype": w.dtype, "operand_bytes": operand_bytes(w),
         "l2": l2_note(w),
         "parallelism": f"replicas x{world}" if world > 1 else "single replica"}
    return d


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement of the reference step on the host cores


def cpu_reference_run(workload: str, steps: int, warmup: int, budget_s: float | None):
    """Time oracle.lowrank_meg_step on the same seeded workload; returns (iters/s, iters timed, seconds)."""
    from oracle import cpu_meg as om
    from oracle import inputs, objectives

    cfg = inputs.CONFIGS[workload]
    obj = objectives.make_objective(cfg)
    x = objectives.initial_iterate(om, cfg, obj)
    t = 0
    for _ in range(warmup):
        x = om.lowrank_meg_step(x, obj.grad_apply(x, t), cfg.eta(t), cfg.eps(t + 1), svd_seed=t,
                                svd_subspace=cfg.subspace).iterate
        t += 1
    done = 0
    t0 = time.perf_counter()
    while done < steps:
        x = om.lowrank_meg_step(x, obj.grad_apply(x, t), cfg.eta(t), cfg.eps(t + 1), svd_seed=t,
                                svd_subspace=cfg.subspace).iterate
        t += 1
        done += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, done, dt


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    w = workload_table()[args.workload]
    warm = max(args.warmup, 3)
    val, done, dt = cpu_reference_run(args.workload, args.steps, warm, budget_s=args.ref_budget)
    sample = (f"{done} consecutive iterations of {args.workload} after {warm} warm-up iterations"
              + ("" if done == args.steps else f" (capped at {args.ref_budget:.0f} s of the requested {args.steps})")
              + ", oracle/cpu_meg.lowrank_meg_step (restatement of meg.py:327-364 + linalg.py:130-241), "
                "factored grad_apply, svd_subspace=64, numpy/OpenBLAS on all host cores")
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": done, "warmup": warm,
        "ms_per_step": 1e3 * dt / done, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": w.dtype, "data": "synthetic (seeded counter-based generator, host-side)", "impl": "reference",
        "config": config_dict(args.workload, 1),
        "parallelism": "host cores (single process, BLAS threads)",
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cpu_cores(), "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device arm


def load_peak():
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        with open(peaks_path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def setup_workload(name: str):
    """Inputs generated in HBM by the seeded device generator; warm start on the device solver."""
    import paper_2012_10469_b200 as pb
    from paper_2012_10469_b200 import inputs

    w = workload_table()[name]
    tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
    if w.kind == "sampled":
        csr = inputs.sampled_instance(w)
        obj = pb.SampledObjective(w.n, *csr)
        x = inputs.initial_iterate(w, tol=tol, csr=csr)
        opb = csr[1].numel() * 12 + (w.n + 1) * 4
    else:
        m = inputs.dense_target(w)
        if w.kind == "stochastic":
            obj = pb.StochasticFrobeniusObjective.from_device(m, w.dtype, batch=w.batch, sigma=w.sigma, seed=w.seed)
        else:
            obj = pb.FrobeniusObjective.from_device(m, w.dtype)
        x = inputs.initial_iterate(w, m, tol=tol)
        opb = operand_bytes(w)
    return w, obj, x, opb


def measure_workload(name: str, W: int, K: int, world: int, dev, peak: float, sampler_gpu=None, clock_ms=50):
    """Device (in-loop events), roofline (pass events) and e2e (host buffers) of one workload."""
    import numpy as np
    import torch

    import paper_2012_10469_b200 as pb
    from paper_2012_10469_b200 import driver, runtime
    import ctypes as C

    w, obj, x, opb = setup_workload(name)
    if w.cert_every:
        W = max(W, w.cert_every)  # the warm-up includes a certificate: the timed ones are warm-started
    solver = runtime.solver_for(w.n)
    lib = solver.lib
    run_kw = dict(eta=w.eta0, eta_decay=w.eta_decay, svd_subspace=w.subspace, block=w.block, timing=False,
                  cert_every=w.cert_every)

    # ---- device: W warm-up + K timed steps in one pipelined native loop
    sampler = ClockSampler(sampler_gpu, clock_ms) if sampler_gpu is not None else None
    if sampler:
        sampler.start()
        time.sleep(0.3)  # let nvidia-smi attach before the timed region
    barrier(world)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"timed_{name}")  # ncu --nvtx-include timed_cfg2/ (launch lists in profiles/)
    rr = driver.run(x, obj, W + K, t0=0, timed_from=W, timed_count=K, **run_kw)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    barrier(world)
    clocks = sampler.stop() if sampler else None
    total_s = rr.timed_ms / 1e3
    value, tmax = aggregate(total_s, K, world, dev)
    passes = rr.passes[W:]
    t = W + K
    x = rr.iterate
    gaps = [] if rr.gap is None else [float(g) for g in rr.gap[W:] if np.isfinite(g)]

    # ---- roofline: every operand pass of a further K-step window bracketed by events
    lib.megb200_profile_enable(solver.handle, 1)
    pm, pc, pbytes = C.c_double(), C.c_int64(), C.c_double()
    lib.megb200_profile_read(solver.handle, C.byref(pm), C.byref(pc), C.byref(pbytes))  # reset
    pr = driver.run(x, obj, K, t0=t, **run_kw)
    lib.megb200_profile_read(solver.handle, C.byref(pm), C.byref(pc), C.byref(pbytes))
    lib.megb200_profile_enable(solver.handle, 0)
    x, t = pr.iterate, t + K
    pass_ms = pm.value / pc.value if pc.value else None
    bytes_per_pass = pbytes.value / pc.value if pc.value else None
    achieved = bytes_per_pass / (pass_ms / 1e3) / 1e9 if pass_ms else None
    ms_per_step = 1e3 * tmax / K
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if achieved else None, "traffic": None,
        "kernel": {"f64": "k_dense_pass_mma (TMA + DMMA/DFMA)", "f32": "k_dense_pass_umma (TMA + tcgen05 split TF32)",
                   "csr": "k_csr_apply_panel (U panels in shared memory, warp per row)"}["csr" if w.kind == "sampled" else w.dtype],
        "bytes_per_pass": bytes_per_pass, "pass_ms": pass_ms, "passes_measured": int(pc.value),
        "share_of_step": (pass_ms * float(np.mean(passes)) / ms_per_step) if pass_ms else None,
    }
    if w.kind != "sampled" and w.dtype == "f64" and pass_ms:
        # the float64 pass against the FP64 tensor-core (DMMA) rate as well: 2 n^2 b flops per pass; 40 TFLOP/s
        # is the nominal B200 figure (DMMA.8x8x4 measured at 16 cycles per SMSP: profiles/r02b_ncu_pass.md)
        fl = 2.0 * w.n * w.n * w.block
        roofline["fp64_tensor"] = {"flops_per_pass": fl, "achieved_tflops": fl / (pass_ms * 1e-3) / 1e12,
                                   "peak_tflops": 40.0, "peak_source": "nominal",
                                   "frac": fl / (pass_ms * 1e-3) / 1e12 / 40.0}

    # ---- e2e through the host-buffer entry point (pinned host V in, V_next out every step)
    Vh = torch.empty((w.n, w.r), dtype=torch.float64).pin_memory()
    Vh.copy_(x.V_device)
    Vn = torch.empty_like(Vh).pin_memory()
    lam, eps, warm, werr = x.lam.copy(), x.eps, x.warm_block, x.warm_orth_err
    stochastic = w.kind == "stochastic"
    stepper = None if stochastic else pb.HostStepper(obj, w.n, w.r, svd_subspace=w.subspace, block=w.block)

    def host_step(Vh, Vn, lam, eps, warm, werr, t):
        if stepper is not None:
            return stepper.step(Vh, lam, eps, w.eta(t), w.eps(t + 1), t, warm=warm, warm_orth_err=werr, out=Vn)
        return pb.lowrank_meg_step_host(Vh, lam, eps, obj, w.eta(t), w.eps(t + 1), svd_seed=t,
                                        svd_subspace=w.subspace, t=t, block=w.block, warm=warm,
                                        warm_orth_err=werr, out=Vn)

    if w.cert_every:
        obj.dual_gap(pb.LowRankIterate(w.n, w.r, Vh.cuda(), lam, eps), block=w.block)  # warm the certificate
    for _ in range(3):
        res = host_step(Vh, Vn, lam, eps, warm, werr, t)
        Vh, Vn = Vn, Vh
        lam, eps, warm, werr = res.lam, res.eps, res.warm_block, res.warm_orth_err
        t += 1
    gap_s = 0.0
    barrier(world)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for i in range(K):
        res = host_step(Vh, Vn, lam, eps, warm, werr, t)
        Vh, Vn = Vn, Vh
        lam, eps, warm, werr = res.lam, res.eps, res.warm_block, res.warm_orth_err
        if w.cert_every and (t + 1) % w.cert_every == 0:
            # the certificate of the config, on the iterate just produced (host V uploaded)
            xg = pb.LowRankIterate(w.n, w.r, Vh.cuda(non_blocking=True), lam, eps)
            obj.dual_gap(xg, block=w.block)
        t += 1
    f1.record()
    torch.cuda.synchronize()
    e2e_s = f0.elapsed_time(f1) / 1e3
    e2e_value, _ = aggregate(e2e_s, K, world, dev)
    h2d = w.n * w.r * 8 + w.r * 8
    d2h = w.n * w.r * 8 + (4 * w.r + 3) * 8 + 8 * 8
    out = {
        "value": value, "ms_per_step": ms_per_step, "steps": K, "warmup": W,
        "passes_per_step": float(np.mean(passes)), "cold_start_passes": int(rr.passes[0]),
        "gpu_launches": int(rr.timed_launches), "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "operand_bytes": int(opb), "clocks": clocks,
    }
    if w.cert_every:
        out["certificates_in_timed_steps"] = len(gaps)
        out["dual_gap_last"] = gaps[-1] if gaps else None
    del obj, x, rr, pr
    return out


def run_device_arm(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(world, "nccl")
    peak, peak_src = load_peak()
    W, K = max(3, args.warmup), args.steps
    head = measure_workload(args.workload, W, K, world, dev, peak, sampler_gpu=local, clock_ms=args.clock_ms)
    head["roofline"]["peak_source"] = peak_src

    extra = {}
    names = [] if args.workloads in ("", "none") else [s for s in args.workloads.split(",") if s != args.workload]
    for name in names:
        torch.cuda.empty_cache()
        kw = min(K, 100)
        r = measure_workload(name, W, kw, world, dev, peak)
        r["config"] = config_dict(name, world)
        r["dtype"] = workload_table()[name].dtype
        extra[name] = r

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, done, dt = cpu_reference_run(args.workload, 10**6, 1, budget_s=args.cpu_budget)
        cpu = {"value": val, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
               "sample": f"{done} consecutive iterations ({dt:.1f} s) of {args.workload} after 1 warm-up iteration, "
                         "oracle/cpu_meg.lowrank_meg_step (restatement of meg.py:327-364 + linalg.py:130-241), "
                         "factored grad_apply, svd_subspace=64, numpy/OpenBLAS on all host cores"}

    if rank == 0:
        w = workload_table()[args.workload]
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": w.dtype, "data": "synthetic (seeded counter-based generator, device-side)", "impl": "b200",
            "config": config_dict(args.workload, world),
            "roofline": head["roofline"],
            "cpu_baseline": cpu,
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
            "passes_per_step": head["passes_per_step"],
            "cold_start_passes": head["cold_start_passes"],
            "timing": "device: W warm-up + K timed steps in ONE call of the pipelined native run loop "
                      "(megb200_meg_run); CUDA events on the solver stream at the start of step W and the end of "
                      "step W+K-1; e2e: per-step host-buffer C-ABI call (megb200_lowrank_meg_step_host via "
                      "pb.HostStepper), V uploaded from pinned host memory, validated, stepped, V_next written back",
            "workloads": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return
    run_device_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
