"""Wall-clock per step of the native run loop with and without per-step CUDA events (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs  # noqa: E402

w = configs.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
m = inputs.dense_target(w)
obj = pb.FrobeniusObjective.from_device(m, w.dtype)
x = inputs.initial_iterate(w, m)
r = driver.run(x, obj, 3, eta=w.eta0, svd_subspace=w.subspace, block=w.block)
x, t = r.iterate, 3
for timing in (True, False, True, False):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = driver.run(x, obj, 500, t0=t, eta=w.eta0, svd_subspace=w.subspace, block=w.block, timing=timing)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 500 * 1e6
    print(f"timing={timing}: wall {wall:.1f} us/step, events {r.step_ms.mean() * 1e3:.1f} us/step, passes {r.passes.mean():.2f}")
    x, t = r.iterate, t + 500
