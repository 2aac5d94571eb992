"""Phase times of the fused orthonormalisation kernel (k_coop_orth) in cfg4's step loop (dev tool, GPU box:
rebuilds libmegb200.so with -DMEG_PHASE_TIMING in place)."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2012_10469_b200 import build  # noqa: E402

subprocess.run([build.nvcc(), *build.NVCC_FLAGS, "-DMEG_PHASE_TIMING", "-o", build.TARGET, *build.SOURCES], check=True)
import numpy as np  # noqa: E402
import config_profile as cp  # noqa: E402
import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs, runtime  # noqa: E402

w = configs.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
obj, init = cp.objective_for(w)
tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
x = inputs.initial_iterate(w, init, tol=tol)
lib = runtime.solver_for(w.n).lib
lib.megb200_debug_phase_ns.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 64)()
r0 = driver.run(x, obj, 3, eta=w.eta0, eta_decay=w.eta_decay, svd_subspace=w.subspace, block=w.block)
lib.megb200_debug_phase_ns(buf, 64)
v = list(buf)
pm = int(v[49])
print("phases (last orth of the run), us:")
for k in range(51, min(pm, 64)):
    print(f"  slot {k}: {(v[k] - v[k - 1]) / 1e3:8.2f}")
print(f"  total 50 -> {pm}: {(v[min(pm, 63)] - v[50]) / 1e3:8.2f}")
