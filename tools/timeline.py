"""Device timeline of the steady run loop via torch.profiler (CUPTI): per-kernel
durations and the idle gaps between consecutive kernels (dev tool).

    python tools/timeline.py [cfg2] [--steps 20] [--flush]
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", nargs="?", default="cfg2")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    args = ap.parse_args()
    w = configs.WORKLOADS[args.name]
    m = inputs.dense_target(w)
    obj = pb.FrobeniusObjective.from_device(m, w.dtype)
    tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
    x = inputs.initial_iterate(w, m, tol=tol)
    r0 = driver.run(x, obj, 3, eta=w.eta0, svd_subspace=w.subspace, block=w.block)
    torch.cuda.synchronize()
    flush = (256 << 20) if args.flush else 0
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        rr = driver.run(r0.iterate, obj, args.steps, t0=3, eta=w.eta0, svd_subspace=w.subspace, block=w.block,
                        flush_bytes=flush)
        torch.cuda.synchronize()
    prof.export_chrome_trace(args.out)
    ev = json.load(open(args.out))["traceEvents"]
    k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    k.sort(key=lambda e: e["ts"])
    dur = collections.defaultdict(list)
    gaps = collections.defaultdict(list)
    for a, b in zip(k, k[1:]):
        gaps[(a["name"][:40], b["name"][:40])].append(b["ts"] - (a["ts"] + a["dur"]))
    for e in k:
        dur[e["name"][:60]].append(e["dur"])
    span = (k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]) if k else 0.0
    print(json.dumps({"steps": args.steps, "span_us": span, "us_per_step": span / args.steps,
                      "step_ms_mean": float(rr.step_ms.mean()), "passes": float(rr.passes.mean())}))
    print("kernel durations (us): name, count, mean")
    for nm, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {nm:60s} {len(v):5d} {sum(v) / len(v):9.2f}")
    print("gaps between consecutive device ops (us): prev -> next, count, mean")
    for (a, b), v in sorted(gaps.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {a:40s} -> {b:40s} {len(v):5d} {sum(v) / len(v):8.2f}")


if __name__ == "__main__":
    main()
