"""A few stored K.V products on the int8-slice kernel at one BASELINE shape (for ncu): config 3
(n = 65536) or 4, m = s or w, float64 (7 x 7 slices) or float32 (3 x 4)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--dtype", default="fp64")      # fp32: the 3 x 4-slice product (d <= 3 points)
ap.add_argument("--path", default="stored")     # on_the_fly: served from the cached sparse image if it fits
a = ap.parse_args()
wl = baseline(a.config)
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=a.dtype, path=a.path)
V = torch.randn(a.m, wl.n, dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    R.kv_apply(V)
torch.cuda.synchronize()
print("ok")
