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

if not os.environ.get("ORTH_PHASE_SKIP_BUILD"):
    subprocess.run([build.nvcc(), *build.NVCC_FLAGS, "-DMEG_PHASE_TIMING", "-o", build.TARGET, *build.SOURCES], check=True)
import numpy as np  # noqa: E402
import config_profile as cp  # noqa: E402
import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs, runtime  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
buf = (C.c_ulonglong * 64)()
if which.startswith("qm"):  # quadratic measurements, e.g. qm100x5 (n = 100, r = 5)
    n, r = (int(v) for v in which[2:].split("x"))
    a, b, y, tau = inputs.quad_meas_instance(n, r, seed=0)
    obj = pb.QuadMeasObjective(a, b, y, tau)
    q, _ = np.linalg.qr(np.random.default_rng(1000).standard_normal((n, r)))
    x = pb.warm_start_wrap(q, np.full(r, 1.0 / r), 0.6 / 121)
    for t in range(4):
        x = pb.lowrank_meg_step(x, obj.grad_operator(x), 1.0 / obj.preset_beta(n, r), 0.6 / (t + 12) ** 2,
                                svd_seed=t).iterate
    lib = runtime.solver_for(n).lib
    lib.megb200_debug_phase_ns.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
else:
    w = configs.WORKLOADS[which]
    obj, init = cp.objective_for(w)
    tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
    import torch
    if isinstance(init, torch.Tensor):
        x = inputs.initial_iterate(w, init, tol=tol)
    else:
        top = pb.lanczos_top_r(init, w.r, tol=tol, seed=w.seed, subspace=64, return_device=True)
        lam = pb.project_simplex(top.eigenvalues, 1.0)
        lam = np.maximum(lam / lam.sum(), 1e-12)
        x = pb.warm_start_wrap(top.eigenvectors, lam / lam.sum(), w.eps(0))
    lib = runtime.solver_for(w.n).lib
    lib.megb200_debug_phase_ns.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    r0 = driver.run(x, obj, 3, eta=w.eta0, eta_decay=w.eta_decay, svd_subspace=w.subspace, block=w.block)
lib.megb200_debug_phase_ns(buf, 64)
v = list(buf)
pm = int(v[49])
print("phases (last orth of the run), us:")
for k in range(51, min(pm, 64)):
    print(f"  slot {k}: {(v[k] - v[k - 1]) / 1e3:8.2f}")
print(f"  total 50 -> {pm}: {(v[min(pm, 63)] - v[50]) / 1e3:8.2f}")
print("last Pythagorean round, CTA 0 thread 0, cycles: G' " + str(v[33] - v[32]) + ", kept-share min " + str(v[34] - v[33]) +
      ", Cholesky + R^-1 " + str(v[35] - v[34]) + ", projection " + str(v[36] - v[35]) + ", (solve follows)")
print("block_cholesky (last call), cycles: load + equilibrate " + str(v[41] - v[40]) + ", factorisation " + str(v[42] - v[41]) +
      ", R^-1 " + str(v[43] - v[42]) + ", outputs " + str(v[44] - v[43]))
print("k_coop_finish (last launch), us: coefficients + L^T U partial " + f"{(v[21] - v[20]) / 1e3:.2f}" + ", reduce E " +
      f"{(v[22] - v[21]) / 1e3:.2f}" + ", W rows " + f"{(v[23] - v[22]) / 1e3:.2f}" + ", H partial " +
      f"{(v[24] - v[23]) / 1e3:.2f}" + ", grid barrier " + f"{(v[25] - v[24]) / 1e3:.2f}" + ", reduce H " +
      f"{(v[26] - v[25]) / 1e3:.2f}")

