"""Phase times of the fused first-pass kernel (megb200_step.cu) in a config's warm step loop (dev tool).

    MEGB200_FUSED_STAMPS=1 python tools/fused_stamps.py [cfg2] [--steps 60]
"""

import argparse
import ctypes as C
import os
import sys

os.environ.setdefault("MEGB200_FUSED_STAMPS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, inputs, runtime  # noqa: E402

NAMES = {1: "stage U, L rows (CTA 0)", 2: "phase 0 (E)", 3: "phase 1 W rows + H partial (CTA 0)",
         4: "-> last CTA arrives (ticket)", 5: "last: reduce H", 6: "last: Jacobi", 7: "last: epilogue+publish",
         8: "CTA 0: released", 9: "phase 2 rows + partials (CTA 0)", 10: "-> last CTA arrives", 11: "last: reduce",
         12: "last: host pack", 13: "(CTA 0 S, theta loaded after release)", 14: "(CTA 0 Ritz rows + residual rows done)",
         15: "(CTA 0 W rows done, before the H partial)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", nargs="?", default="cfg2")
    ap.add_argument("--steps", type=int, default=60)
    args = ap.parse_args()
    w = configs.WORKLOADS[args.name]
    m = inputs.dense_target(w)
    obj = pb.FrobeniusObjective.from_device(m, w.dtype)
    tol = 1e-10 if w.dtype == "f64" else pb.objectives.F32_TOL_FLOOR
    x = inputs.initial_iterate(w, m, tol=tol)
    lib = runtime.solver_for(w.n).lib
    h = runtime.solver_for(w.n).handle
    lib.megb200_debug_fused_ns.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int32]
    buf = (C.c_ulonglong * 16)()
    acc = np.zeros(16)
    k = 0
    for t in range(args.steps):
        res = pb.lowrank_meg_step(x, obj.grad_operator(x), w.eta(t), w.eps(t + 1), svd_seed=t,
                                  svd_subspace=w.subspace, block=w.block)
        x = res.iterate
        torch.cuda.synchronize()
        lib.megb200_debug_fused_ns(h, buf, 16)
        if t >= 10 and res.passes == 1:
            v = np.array(list(buf), dtype=np.float64)
            acc[1:13] += (v[1:13] - v[0:12]) / 1e3
            acc[13] += (v[13] - v[8]) / 1e3
            acc[14] += (v[14] - v[13]) / 1e3
            acc[15] += (v[15] - v[2]) / 1e3
            k += 1
    print(f"{args.name}: {k} warm steps")
    for i, nm in NAMES.items():
        print(f"  {nm:40s} {acc[i] / max(k, 1):8.2f} us")
    print(f"  {'total (stamp 0 -> 12)':40s} {acc[1:13].sum() / max(k, 1):8.2f} us")


if __name__ == "__main__":
    main()
