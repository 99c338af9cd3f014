"""Run the K x V product at a BASELINE shape a few times (for ncu / timing)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dtype", default="fp32")
a = ap.parse_args()
wl = baseline(a.config)
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=a.dtype, path="stored")
V = torch.randn(a.m, wl.n, dtype=torch.float64, device="cuda")
st = torch.cuda.ExternalStream(R.sess.handle.stream)
for _ in range(2):
    R.kv_apply(V)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(a.reps):
    R.kv_apply(V)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
es = 4 if a.dtype == "fp32" else 8
print(f"config{a.config} n={wl.n} m={a.m}: {ms:.3f} ms/product, {es * wl.n**2 / ms / 1e6:.0f} GB/s (K bytes only)")
