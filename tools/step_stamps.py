"""Phase maxima of the fused pass + step tail (k_dense_step_mma) in cfg2's warm per-step loop (dev tool).

    MEGB200_FUSED_STAMPS=1 python tools/step_stamps.py [cfg2] [--steps 60]
"""

import argparse
import ctypes as C
import os
import sys

if "--no-stamps" not in sys.argv:
    os.environ.setdefault("MEGB200_FUSED_STAMPS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, inputs, runtime  # noqa: E402

NAMES = ["main loops done (max over CTAs)", "fix-ups done (max)", "RR CTA starts", "RR solved",
         "phase 2 released (max)", "Ritz rows written (max)", "finish starts", "pack written"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name", nargs="?", default="cfg2")
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--no-stamps", action="store_true", help="plain step loop (for ncu)")
    args = ap.parse_args()
    w = configs.WORKLOADS[args.name]
    m = inputs.dense_target(w)
    obj = pb.FrobeniusObjective.from_device(m, w.dtype)
    x = inputs.initial_iterate(w, m, tol=1e-10)
    s = runtime.solver_for(w.n)
    s.lib.megb200_debug_fused_ns.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int32]
    buf = (C.c_ulonglong * 16)()
    rows = []
    for t in range(args.steps):
        res = pb.lowrank_meg_step(x, obj.grad_operator(x), w.eta(t), w.eps(t + 1), svd_seed=t,
                                  svd_subspace=w.subspace, block=w.block)
        x = res.iterate
        torch.cuda.synchronize()
        s.lib.megb200_debug_fused_ns(s.handle, buf, 16)
        v = np.array(list(buf)[:8], dtype=np.float64)
        if not args.no_stamps and t >= 10 and res.passes == 1 and v.min() > 0:
            rows.append((v - v[0]) / 1e3)
    if args.no_stamps:
        return
    r = np.array(rows)
    print(f"{args.name}: {len(rows)} warm steps, microseconds after the last main loop ended")
    for i, nm in enumerate(NAMES):
        print(f"  {nm:36s} {np.median(r[:, i]):8.2f}  (p90 {np.percentile(r[:, i], 90):.2f})")


if __name__ == "__main__":
    main()
