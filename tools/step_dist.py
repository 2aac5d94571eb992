"""Distribution of per-step device times of the pipelined run loop (dev tool).

    python tools/step_dist.py [cfg2] [--steps 2000] [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name", nargs="?", default="cfg2")
ap.add_argument("--steps", type=int, default=2000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
w = configs.WORKLOADS[a.name]
m = inputs.dense_target(w)
obj = pb.FrobeniusObjective.from_device(m, w.dtype)
x = inputs.initial_iterate(w, m)
t = 0
r = driver.run(x, obj, 5, t0=t, svd_subspace=w.subspace, block=w.block)
x, t = r.iterate, t + 5
for rep in range(a.reps):
    for timing in (True, False):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = driver.run(x, obj, a.steps, t0=t, svd_subspace=w.subspace, block=w.block, timing=timing)
        e1.record()
        torch.cuda.synchronize()
        x, t = r.iterate, t + a.steps
        tot = e0.elapsed_time(e1) / a.steps * 1e3
        if timing:
            s = np.asarray(r.step_ms) * 1e3
            print(f"rep {rep} timed: mean {tot:.1f} us/step; step us p10 {np.percentile(s, 10):.1f} p50 "
                  f"{np.percentile(s, 50):.1f} p90 {np.percentile(s, 90):.1f} p99 {np.percentile(s, 99):.1f} "
                  f"max {s.max():.1f}; passes {np.mean(r.passes):.2f}", flush=True)
        else:
            print(f"rep {rep} untimed: mean {tot:.1f} us/step -> {1e6 / tot:.0f} it/s", flush=True)
