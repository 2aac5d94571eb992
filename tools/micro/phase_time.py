"""Build a -DMEG_PHASE_TIMING variant of the library and print cooperative-kernel phase times for a config's step loop.

Run on the GPU box only (it rebuilds libmegb200.so in place)."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2012_10469_b200 import build  # noqa: E402

subprocess.run([build.nvcc(), *build.NVCC_FLAGS, "-DMEG_PHASE_TIMING", "-o", build.TARGET, *build.SOURCES], check=True)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, inputs, runtime  # noqa: E402

w = configs.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
m = inputs.dense_target(w)
obj = pb.FrobeniusObjective.from_device(m, w.dtype)
x = inputs.initial_iterate(w, m)
lib = runtime.solver_for(w.n).lib
lib.megb200_debug_phase_ns.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 64)()
names = {1: "chol: gram partial", 2: "chol: sync1", 3: "chol: reduce+sync2", 4: "chol: cholesky(CTA0)",
         5: "chol: sync3", 6: "chol: apply Rinv", 11: "rr: jacobi(CTA0)", 12: "rr: sync1", 13: "rr: ritz+partials",
         14: "rr: sync2", 15: "rr: reduce", 21: "fin: LtU partial+sync", 22: "fin: reduce E+sync",
         23: "fin: rows W", 24: "fin: QtW partial", 25: "fin: sync", 26: "fin: reduce H",
         40: "jac: load H", 41: "jac: norms", 42: "jac: pre 1", 43: "jac: pre 2", 44: "jac: pre 3",
         45: "jac: (pre end)", 46: "jac: sweeps", 47: "jac: sort+store"}
acc = {k: 0.0 for k in names}
K = 0
for t in range(80):
    x = pb.lowrank_meg_step(x, obj.grad_operator(x), 1.0, w.eps(t + 1), svd_seed=t, svd_subspace=w.subspace,
                            block=w.block).iterate
    torch.cuda.synchronize()
    lib.megb200_debug_phase_ns(buf, 64)
    if t >= 20:
        K += 1
        v = list(buf)
        for k in names:
            base = 0 if k < 10 else (10 if k < 20 else (20 if k < 40 else 10))
            prev = k - 1 if k - 1 >= base else base
            acc[k] += (v[k] - v[prev]) / 1e3
for k, nm in names.items():
    print(f"{nm:24s} {acc[k] / K:9.2f} us")
print("(jac rows are cumulative from the rr kernel start; pre rows are 0 when not run)")
