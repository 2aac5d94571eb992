"""Matrix-free quadratic-measurement block application (k_qm_fwd + k_qm_bwd): time per application and
achieved GB/s against its algorithmic bytes 4 m n 8 (a and b streamed twice) -- dev tool.

    python tools/qm_apply_bench.py [n r k]...   e.g.  2048x2x10 4096x1x9
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402

for spec in sys.argv[1:] or ["2048x2x10", "4096x1x9"]:
    n, r, k = (int(v) for v in spec.split("x"))
    m = 20 * n * r
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    a /= a.norm(dim=1, keepdim=True)
    b = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    b /= b.norm(dim=1, keepdim=True)
    y = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    obj = pb.QuadMeasObjective(a, b, y, 0.5 * n)
    res = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    u = torch.randn((n, k), dtype=torch.float64, device="cuda", generator=g)
    w = obj.apply_gradient(res, u)
    # spot check against torch (cuBLAS) -- diagnostic only
    want = 0.5 * obj.tau * (a.T @ (res[:, None] * (b @ u)) + b.T @ (res[:, None] * (a @ u)))
    err = float((w - want).norm() / want.norm())
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        obj.apply_gradient(res, u)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    nbytes = 4.0 * m * n * 8
    print(json.dumps({"n": n, "r": r, "k": k, "m": m, "ms_per_apply": ms, "GB/s": nbytes / ms / 1e6,
                      "rel_err_vs_torch": err}), flush=True)
    del a, b, obj, want
    torch.cuda.empty_cache()
