#!/usr/bin/env python
"""Benchmark: low-rank MEG iterations/sec on B200 (BASELINE.json metric, config 2).

A *step* is one `lowrank_meg_step` (meg.py:327-364) of the config-2 workload
(n = 4096, r = 10, float64, block k = r + 8 = 18, dense 1/2||X - M||_F^2,
eta = 1, eps_t = 0.6/(t+11)^2) continuing one trajectory from the warm start.
Inputs are resident in HBM when the timed region starts.  L2 is not flushed:
the float64 operand (134 MB) is larger than the 126 MB L2 and is streamed with
an evict-first policy, so every step reads it from HBM (checked with ncu,
profiles/r01_l2_check.txt).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs one independent replica per GPU (the path does not shard at this
tier), launched by torch.distributed.run; the time is the max
over ranks.  `--impl reference` times the CPU restatement of the reference
(oracle/, the "port") on the host cores for the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "low-rank MEG iterations/sec at n=4096–32768, r=5–20; achieved HBM GB/s vs peak"
UNIT = "iterations/s"
WORKLOAD_DESC = ("cfg2: deterministic low-rank MEG, dense 1/2||X-M||_F^2, n=4096, r=10, fp64, "
                 "block k=r+8=18, eta=1, eps_t=0.6/(t+11)^2, warm start from the rank-10 projection of M")


def workload_desc(name: str) -> str:
    """The bench line's config.workload for the dense workloads (cfg2 is the headline)."""
    if name == "cfg2":
        return WORKLOAD_DESC
    from paper_2012_10469_b200 import configs

    w = configs.WORKLOADS[name]
    return (f"{name}: deterministic low-rank MEG, dense 1/2||X-M||_F^2, n={w.n}, r={w.r}, {w.dtype}, block k={w.block}, "
            f"eta={w.eta0}, eps_t=0.6/(t+11)^2, warm start from the rank-{w.r} projection of M")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: same as --steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU baseline sampling")
    ap.add_argument("--clock-ms", type=int, default=50, help="nvidia-smi clock sampling interval (ms)")
    ap.add_argument("--prof-stride", type=int, default=16, help="bracket every N-th pass with events (0: off)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (replicas only)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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
    warm = max(args.warmup, 0)
    val, done, dt = cpu_reference_run(args.workload, args.steps, min(warm, 3), budget_s=None)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": done, "warmup": min(warm, 3),
        "ms_per_step": 1e3 * dt / done, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": workload_desc(args.workload), "parallelism": "host cores (single process, BLAS threads)"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
                         "sample": f"{done} consecutive iterations of {args.workload} after {min(warm, 3)} warm-up "
                                   "iterations, oracle/cpu_meg.lowrank_meg_step (restatement of meg.py:327-364 "
                                   "+ linalg.py:130-241), factored grad_apply, svd_subspace=64"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device arm


def run_device_arm(args, world, rank, local):
    import numpy as np
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(world, "nccl")
    import paper_2012_10469_b200 as pb
    from paper_2012_10469_b200 import configs, inputs, runtime

    w = configs.WORKLOADS[args.workload]
    if w.kind != "dense":
        raise SystemExit("bench.py times the dense workloads (cfg1/cfg2/cfg5)")
    m = inputs.dense_target(w)
    obj = pb.FrobeniusObjective.from_device(m, w.dtype)
    tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
    x = inputs.initial_iterate(w, m, tol=tol)
    solver = runtime.solver_for(w.n)
    lib = solver.lib

    def step(xi, t):
        return pb.lowrank_meg_step(xi, obj.grad_operator(xi), w.eta(t), w.eps(t + 1), svd_seed=t,
                                   svd_subspace=w.subspace, block=w.block)

    t = 0
    cold_passes = None
    for _ in range(max(3, args.warmup)):
        res = step(x, t)
        if cold_passes is None:
            cold_passes = res.passes
        x = res.iterate
        t += 1
    # warm the native run loop too (its device slots are allocated on first use; a cudaMalloc
    # inside the timed region made single runs up to 2x slower)
    from paper_2012_10469_b200 import driver

    wr = driver.run(x, obj, max(3, args.warmup), t0=t, svd_subspace=w.subspace, block=w.block, timing=False)
    x, t = wr.iterate, t + max(3, args.warmup)
    torch.cuda.synchronize()

    # ---- device-resident timed region: K steps through the native run loop
    #      (megb200_meg_run), one CUDA-event pair around all K steps.  No L2 flush:
    #      the operand (n^2 * 8 B = 134 MB) exceeds the 126 MB L2 and is streamed
    #      evict-first, so every pass reads it from HBM (profiles/r01_l2_check.txt)
    from paper_2012_10469_b200 import driver
    import ctypes as C

    K = args.steps
    prof_stride = args.prof_stride  # roofline: every 16th pass kernel bracketed by events (small perturbation)
    lib.megb200_profile_enable(solver.handle, prof_stride)
    pm, pc, pb_bytes = C.c_double(), C.c_int64(), C.c_double()
    lib.megb200_profile_read(solver.handle, C.byref(pm), C.byref(pc), C.byref(pb_bytes))  # reset
    sampler = ClockSampler(local, args.clock_ms)
    sampler.start()
    time.sleep(0.3)  # let nvidia-smi attach before the timed region
    barrier(world)
    torch.cuda.synchronize()
    launches0 = solver.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host0 = time.perf_counter()
    torch.cuda.nvtx.range_push("timed")
    e0.record()
    step_timing = os.environ.get("BENCH_STEP_TIMING") == "1"  # diagnostics: per-step events (perturbs)
    rr = driver.run(x, obj, K, t0=t, svd_subspace=w.subspace, block=w.block, timing=step_timing)
    e1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    host_s = time.perf_counter() - host0
    launches = solver.launches - launches0  # our kernels only
    barrier(world)
    clocks = sampler.stop()
    lib.megb200_profile_read(solver.handle, C.byref(pm), C.byref(pc), C.byref(pb_bytes))
    lib.megb200_profile_enable(solver.handle, 0)
    passes = list(rr.passes)
    if step_timing:
        sm = np.asarray(rr.step_ms) * 1e3
        print(f"step us: p10 {np.percentile(sm, 10):.1f} p50 {np.percentile(sm, 50):.1f} p90 {np.percentile(sm, 90):.1f} "
              f"p99 {np.percentile(sm, 99):.1f} max {sm.max():.1f} mean {sm.mean():.1f}", file=sys.stderr)
    total_s = e0.elapsed_time(e1) / 1e3
    value, tmax = aggregate(total_s, K, world, dev)
    x = rr.iterate
    t += K

    # ---- end to end through the public API with host buffers
    K2 = args.e2e_steps or K
    # warm the per-step API path (the run loop's final iterate carries no Ritz block)
    for _ in range(3):
        x = step(x, t).iterate
        t += 1
    torch.cuda.synchronize()
    # the caller's iterate lives in pinned host memory: each step uploads it and reads the next one back
    Vh = torch.empty((w.n, w.r), dtype=torch.float64).pin_memory()
    Vh.copy_(x.V_device)
    Vn = torch.empty_like(Vh).pin_memory()
    lam, eps, warm, werr = x.lam.copy(), x.eps, x.warm_block, x.warm_orth_err
    h2d = w.n * w.r * 8 + w.r * 8
    d2h = w.n * w.r * 8 + (4 * w.r + 3) * 8 + 8 * 8
    # the host-buffer entry point through its session object (structs and result buffers made
    # once; each step is one native call); warmed first (device staging is allocated on first use)
    stepper = pb.HostStepper(obj, w.n, w.r, svd_subspace=w.subspace, block=w.block)
    for _ in range(max(3, args.warmup)):
        res = stepper.step(Vh, lam, eps, w.eta(t), w.eps(t + 1), t, warm=warm, warm_orth_err=werr, out=Vn)
        Vh, Vn = Vn, Vh
        lam, eps, warm, werr = res.lam, res.eps, res.warm_block, res.warm_orth_err
        t += 1
    barrier(world)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for i in range(K2):
        # one reference-facing call with host buffers: upload + validate V, step, read V_next back
        res = stepper.step(Vh, lam, eps, w.eta(t), w.eps(t + 1), t, warm=warm, warm_orth_err=werr, out=Vn)
        Vh, Vn = Vn, Vh
        lam, eps, warm, werr = res.lam, res.eps, res.warm_block, res.warm_orth_err
        t += 1
    f1.record()
    torch.cuda.synchronize()
    e2e_s = f0.elapsed_time(f1) / 1e3
    e2e_value, _ = aggregate(e2e_s, K2, world, dev)

    # ---- roofline of the streamed operator pass (dominant kernel: k_dense_apply_* + k_apply_finish)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    achieved = (pb_bytes.value / pc.value) / (pm.value / pc.value / 1e3) / 1e9 if pc.value else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(args.workload)
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": (achieved / peak) if achieved else None, "traffic": traffic,
        "kernel": ("streamed operator pass k_dense_pass_mma (TMA + DMMA/DFMA)" if w.dtype == "f64" else
                   "streamed operator pass k_dense_pass_umma (TMA + tcgen05 split TF32)") + ", every --prof-stride-th (16th) launch of the timed region "
                  "bracketed by CUDA events on the solver stream (includes its launch latency)",
        "bytes_per_pass": (pb_bytes.value / pc.value) if pc.value else None,
        "pass_ms": (pm.value / pc.value) if pc.value else None, "passes": int(pc.value), "peak_source": peak_src,
        "share_of_step": (pm.value / pc.value * sum(passes) / 1e3) / total_s if total_s and pc.value else None,
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, done, dt = cpu_reference_run(args.workload, 10**6, 1, budget_s=args.cpu_budget)
        cpu = {"value": val, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
               "sample": f"{done} consecutive iterations ({dt:.1f} s) of {args.workload} after 1 warm-up iteration, "
                         "oracle/cpu_meg.lowrank_meg_step (restatement of meg.py:327-364 + linalg.py:130-241), "
                         "factored grad_apply, svd_subspace=64, numpy/OpenBLAS on all host cores"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": max(3, args.warmup),
            "ms_per_step": 1e3 * tmax / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": w.dtype, "data": "synthetic (seeded counter-based generator, device-side)", "impl": "b200",
            "config": {"workload": workload_desc(args.workload), "n": w.n, "r": w.r, "block": w.block,
                       "operand_bytes": w.n * w.n * (8 if w.dtype == "f64" else 4),
                       "l2": f"not flushed: operand {w.n * w.n * (8 if w.dtype == 'f64' else 4) / 1e6:.0f} MB > 126 MB L2, "
                             "streamed evict-first" + ("; ncu --cache-control none shows 135.5 MB DRAM read per pass "
                                                       "in the steady loop" if args.workload == "cfg2" else ""),
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "passes_per_step": float(np.mean(passes)),
            "cold_start_passes": cold_passes,
            "host_ms_per_step": 1e3 * host_s / K,
            "timing": "device: native run loop megb200_meg_run (pipelined), one CUDA-event pair around the K steps "
                      "on the solver stream; e2e: per-step lowrank_meg_step_host (C-ABI megb200_lowrank_meg_step_host): "
                      "V uploaded from pinned host memory, validated, stepped and V_next written back every step "
                      "(pb.HostStepper: one native call per step)",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return
    run_device_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
