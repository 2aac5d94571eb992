"""Phase stamps of the cooperative kernels (finish / orth / Rayleigh-Ritz) in a config's step loop (dev tool).

Needs the library built with -DMEG_PHASE_TIMING (CTA 0 thread 0 stamps %globaltimer at the phase
boundaries; the stamps of the LAST launch of each kernel survive):

    cp tools/scratch/libmegb200_phase.so paper_2012_10469_b200/libmegb200.so   # on the GPU box copy
    python tools/phase_report.py cfg3 cfg4
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import config_profile as cp  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs, runtime  # noqa: E402

GROUPS = {"cholqr": (0, 7), "rr": (10, 16), "finish": (20, 27), "jacobi": (40, 48), "orth": (50, 64)}

for which in sys.argv[1:] or ["cfg4"]:
    w = configs.WORKLOADS[which]
    obj, init = cp.objective_for(w)
    tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
    if isinstance(init, torch.Tensor):
        x = inputs.initial_iterate(w, init, tol=tol)
    else:
        top = pb.lanczos_top_r(init, w.r, tol=tol, seed=w.seed, subspace=64, return_device=True)
        lam = pb.project_simplex(top.eigenvalues, 1.0)
        lam = np.maximum(lam / lam.sum(), 1e-12)
        x = pb.warm_start_wrap(top.eigenvectors, lam / lam.sum(), w.eps(0))
    s = runtime.solver_for(w.n)
    lib = s.lib
    lib.megb200_debug_phase_ns.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    r0 = driver.run(x, obj, 2, eta=w.eta0, eta_decay=w.eta_decay, svd_subspace=w.subspace, block=w.block)
    lib.megb200_trace_enable(s.handle, 1)
    rr = driver.run(r0.iterate, obj, 5, t0=2, eta=w.eta0, eta_decay=w.eta_decay, svd_subspace=w.subspace,
                    block=w.block)
    tb = C.create_string_buffer(4096)
    lib.megb200_trace_report(s.handle, tb, 4096)
    lib.megb200_trace_enable(s.handle, 0)
    buf = (C.c_ulonglong * 64)()
    lib.megb200_debug_phase_ns(buf, 64)
    v = list(buf)
    print(f"== {which}: {np.mean(rr.step_ms):.3f} ms/step, {np.mean(rr.passes):.1f} passes/step")
    print(tb.value.decode())
    for name, (a, b) in GROUPS.items():
        b_eff = b
        if name == "orth":
            b_eff = min(b, int(v[49]) + 1) if 50 < v[49] < 64 else b
        stamps = [(k, v[k]) for k in range(a, b_eff) if v[k] > 0]
        if len(stamps) < 2:
            continue
        stamps.sort(key=lambda kv: kv[0])
        base = stamps[0][1]
        line = " ".join(f"[{k}]{(tv - base) / 1e3:+.1f}" for k, tv in stamps)
        print(f"{name:8s} (us from slot {stamps[0][0]}): {line}")
    del obj, init
    torch.cuda.empty_cache()
