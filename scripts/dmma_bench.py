"""Float64 K x V on the FP64 tensor cores (kv_dmma.cu): correctness against torch float64 and
CUDA-event timing at the BASELINE shapes.  Prints one JSON line per shape.

  python scripts/dmma_bench.py [--reps 5] [--shapes c2m32,c3m64,...]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

SHAPES = {"c2m32": (2, None, 32), "c2m266": (2, None, 266), "c3m64": (3, None, 64), "c3m522": (3, None, 522),
          "c1m16": (1, None, 16), "odd": (2, 4099, 37)}

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--shapes", default="c1m16,odd,c2m32,c2m266,c3m64,c3m522")
ap.add_argument("--peak", type=float, default=36.36)
a = ap.parse_args()
for name in a.shapes.split(","):
    cfg, n, m = SHAPES[name]
    wl = baseline(cfg, n=n)
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp64", path="stored")
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn(m, wl.n, dtype=torch.float64, device="cuda", generator=g)
    st = torch.cuda.ExternalStream(R.sess.handle.stream)
    Y = R.kv_apply(V)
    err = None
    if wl.n <= 16384:
        K = rld.build_covariance(wl.spec, wl.points, dtype="fp64")
        ref = V @ K.T
        err = float((Y - ref).abs().max() / ref.abs().max())
        del K, ref
    for _ in range(2):
        R.kv_apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps):
        R.kv_apply(V)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    tf = 2.0 * wl.n * wl.n * m / (ms * 1e-3) / 1e12
    print(json.dumps({"shape": name, "n": wl.n, "m": m, "ms": ms, "tflops": tf, "frac_fp64_peak": tf / a.peak,
                      "hbm_gbs_K": 8 * wl.n * wl.n / (ms * 1e-3) / 1e9, "max_rel_err_vs_torch": err}), flush=True)
    del R, V, Y
    torch.cuda.empty_cache()
