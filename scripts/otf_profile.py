"""Time one on-the-fly K x V product at a BASELINE shape (config 4 / 5) and check
a few rows against float64."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from oracle import rstar_oracle as O  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
wl = baseline(a.config, n=a.n)
m = a.m or wl.config.num_probes
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path="on_the_fly")
g = np.random.default_rng(0)
V = torch.from_numpy(g.standard_normal((m, wl.n))).cuda()
R.kv_apply(V)
st = torch.cuda.ExternalStream(R.sess.handle.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(a.reps):
    Y = R.kv_apply(V)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
n = wl.n
print(f"config{a.config} n={n} m={m} on-the-fly: {ms:.2f} ms/product, {n * n / ms / 1e9:.2f} T entries/s, "
      f"{2 * n * n * m / ms / 1e9:.1f} TFLOP/s useful", flush=True)
Yh = Y.cpu().numpy()
Vh = V.cpu().numpy()
rows = g.choice(n, 8, replace=False)
err = 0.0
for i in rows:
    k = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points,
                           rows=slice(i, i + 1))[0]
    ref = Vh @ k
    err = max(err, float(np.max(np.abs(Yh[:, i] - ref) / (np.abs(Vh) @ np.abs(k)))))
print(f"  max normalized error vs float64 on 8 sampled rows: {err:.2e}")
