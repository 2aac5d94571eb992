"""Dual-gap certificate cost, cold vs warm-started from the previous certificate (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs  # noqa: E402

for name in sys.argv[1:] or ("cfg5", "cfg2"):
    w = configs.WORKLOADS[name]
    m = inputs.dense_target(w)
    obj = pb.FrobeniusObjective.from_device(m, w.dtype)
    tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
    x = inputs.initial_iterate(w, m, tol=tol)
    t = 0
    for cert in range(3):
        r = driver.run(x, obj, 10, t0=t, svd_subspace=w.subspace, block=w.block)
        x, t = r.iterate, t + 10
        for warm in ((False, True) if cert else (True,)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gap, lmin = obj.dual_gap(x, tol=tol, block=w.block, warm=warm)
            torch.cuda.synchronize()
            print(f"{name} after {t} steps: warm={warm} gap={gap:.15e} lmin={lmin:.15e} "
                  f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
