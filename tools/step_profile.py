"""Where does a steady-state MEG step spend its time?  Host phases vs device time (cfg2)."""

import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import configs, inputs, meg, runtime  # noqa: E402

w = configs.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
m = inputs.dense_target(w)
obj = pb.FrobeniusObjective.from_device(m, w.dtype)
x = inputs.initial_iterate(w, m)
for t in range(5):
    x = pb.lowrank_meg_step(x, obj.grad_operator(x), 1.0, w.eps(t + 1), svd_seed=t, svd_subspace=w.subspace,
                            block=w.block).iterate
torch.cuda.synchronize()

# monkeypatch the native call to time it
s = runtime.solver_for(w.n)
lib = s.lib
orig = lib.megb200_lowrank_meg_step
acc = {"native": 0.0}


def timed(*a):
    t0 = time.perf_counter()
    rc = orig(*a)
    acc["native"] += time.perf_counter() - t0
    return rc


class Shim:
    def __getattr__(self, k):
        return timed if k == "megb200_lowrank_meg_step" else getattr(lib, k)


s.lib = Shim()
K = 200
acc["native"] = 0.0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for t in range(5, 5 + K):
    x = pb.lowrank_meg_step(x, obj.grad_operator(x), 1.0, w.eps(t + 1), svd_seed=t, svd_subspace=w.subspace,
                            block=w.block).iterate
e1.record()
torch.cuda.synchronize()
host = (time.perf_counter() - t0) / K
native = acc["native"] / K
lib.megb200_trace_enable(s.handle, 1)
for t in range(5 + K, 5 + 2 * K):
    x = pb.lowrank_meg_step(x, obj.grad_operator(x), 1.0, w.eps(t + 1), svd_seed=t, svd_subspace=w.subspace,
                            block=w.block).iterate
torch.cuda.synchronize()
buf = C.create_string_buffer(4096)
lib.megb200_trace_report(s.handle, buf, 4096)
print(buf.value.decode())
lib.megb200_trace_enable(s.handle, 0)
print(f"per step: host total {host*1e6:.1f} us, inside native call {native*1e6:.1f} us, "
      f"python outside {(host - native)*1e6:.1f} us, device span {e0.elapsed_time(e1)/K*1e3:.1f} us, "
      f"launches/step {s.launches}")

import cProfile
import pstats

pr = cProfile.Profile()
pr.enable()
for t in range(5 + 2 * K, 5 + 3 * K):
    x = pb.lowrank_meg_step(x, obj.grad_operator(x), 1.0, w.eps(t + 1), svd_seed=t, svd_subspace=w.subspace,
                            block=w.block).iterate
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
