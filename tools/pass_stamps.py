"""Per-CTA phase timestamps of the float64 DMMA pass (dev tool; needs MEGB200_PASS_STAMPS=1).

    MEGB200_PASS_STAMPS=1 python tools/pass_stamps.py [--n 4096] [--b 18]

Prints, relative to the earliest CTA start: start, dependency wait over, first stage landed, last
stage consumed, end -- min / median / max over the CTAs, for an isolated apply and for the last
pass of a pipelined cfg2-like run.
"""
import argparse
import ctypes as C
import os
import sys

os.environ.setdefault("MEGB200_PASS_STAMPS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, driver, inputs, runtime  # noqa: E402


def report(lib, label, grid=148):
    buf = (C.c_ulonglong * (160 * 8))()
    lib.megb200_debug_pass_ns.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    lib.megb200_debug_pass_ns(buf, 160 * 8)
    a = np.array(buf[:], dtype=np.float64).reshape(160, 8)[:grid, :5]
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    a = (a - t0) / 1e3
    names = ["start", "dep wait over", "first stage landed", "last stage consumed", "end"]
    print(label, f"({len(a)} CTAs)")
    for j, nm in enumerate(names):
        print(f"  {nm:22s} min {a[:, j].min():7.2f}  med {np.median(a[:, j]):7.2f}  max {a[:, j].max():7.2f} us")
    print(f"  stream phase per CTA (first landed -> last consumed): med {np.median(a[:, 3] - a[:, 2]):.2f} us, "
          f"min {np.min(a[:, 3] - a[:, 2]):.2f}, max {np.max(a[:, 3] - a[:, 2]):.2f}")


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--b", type=int, default=18)
a = ap.parse_args()
dev = runtime.device()
m = torch.randn((a.n, a.n), dtype=torch.float64, device=dev)
m = ((m + m.T) * 0.5).contiguous()
op = pb.SymmetricOperator(a.n, dense=m)
u = torch.randn((a.n, a.b), dtype=torch.float64, device=dev)
for _ in range(3):
    op.apply(u)
torch.cuda.synchronize()
lib = op._solver().lib
report(lib, f"isolated apply n={a.n} b={a.b}")
del m, op
w = configs.WORKLOADS["cfg2"]
mt = inputs.dense_target(w)
obj = pb.FrobeniusObjective.from_device(mt, w.dtype)
x = inputs.initial_iterate(w, mt, tol=1e-10)
r = driver.run(x, obj, 60, eta=w.eta0, svd_subspace=w.subspace, block=w.block)
torch.cuda.synchronize()
print("passes of the last steps", r.passes[-5:], "ms/step", float(np.mean(r.step_ms[-20:])))
report(lib, "last pass of a pipelined cfg2 run")
