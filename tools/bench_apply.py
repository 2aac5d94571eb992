"""Microbenchmark of the streamed operator pass (K1) alone: GB/s of algorithmic bytes vs HBM peak.

    python tools/bench_apply.py [--reps 20]

Times `SymmetricOperator.apply` on device-resident blocks with CUDA events,
flushing L2 between repetitions, for the config shapes.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2012_10469_b200 as pb  # noqa: E402
from paper_2012_10469_b200 import runtime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--shapes", default="4096:18:f64,4096:32:f64,8192:18:f64,16384:16:f32,32768:32:f32,32768:16:f32")
    args = ap.parse_args()
    peak = 6547.2
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p))["hbm_gbs"]
    dev = runtime.device()
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)
    for spec in args.shapes.split(","):
        n, b, dt = spec.split(":")
        n, b = int(n), int(b)
        tdt = torch.float64 if dt == "f64" else torch.float32
        m = torch.randn((n, n), dtype=tdt, device=dev)
        m = (m + m.T) * 0.5
        op = pb.SymmetricOperator(n, dense=m.contiguous())
        u = torch.randn((n, b), dtype=torch.float64, device=dev)
        w = op.apply(u)
        ref = (m.double() @ u)
        err = float((w - ref).abs().max() / ref.abs().max())
        import ctypes as C

        s = op._solver()
        times = []
        pm, pc, pbytes = C.c_double(), C.c_int64(), C.c_double()
        for _ in range(args.reps):
            flush.zero_()
            s.lib.megb200_profile_enable(s.handle, 1)
            op.apply(u)
            s.lib.megb200_profile_read(s.handle, C.byref(pm), C.byref(pc), C.byref(pbytes))
            s.lib.megb200_profile_enable(s.handle, 0)
            times.append(pm.value)
        times.sort()
        ms = times[len(times) // 2]
        by = n * n * m.element_size() + 2 * n * b * 8
        gbs = by / (ms * 1e-3) / 1e9
        print(json.dumps({"n": n, "b": b, "dtype": dt, "ms_median": ms, "ms_min": times[0], "GBps": gbs,
                          "frac_of_peak": gbs / peak, "rel_err_vs_torch": err}), flush=True)
        del m, op


if __name__ == "__main__":
    main()
