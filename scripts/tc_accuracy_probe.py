"""Probe the accuracy of the K x V products (tensor-core vs CUDA-core path) with
positive operands, where |V||K| = V K, so any accumulation bias shows up as a
relative error of the product itself."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from oracle import rstar_oracle as O  # noqa: E402

for n in (2048, 16384, 65536):
    g = np.random.default_rng(1)
    pts = g.uniform(0, 1, (n, 2))
    spec = rld.KernelSpec("matern52", 1.0, 0.3, 1e-2)
    R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path="stored")
    V = np.abs(g.standard_normal((8, n))) + 0.5
    rows = g.choice(n, 64, replace=False)
    Kr = O.covariance_block("matern52", 1.0, 0.3, 1e-2, pts, rows=None) if n <= 16384 else None
    ref = []
    for i in rows:
        k = O.covariance_block("matern52", 1.0, 0.3, 1e-2, pts, rows=slice(i, i + 1))[0]
        k = k.astype(np.float32).astype(np.float64)
        ref.append(V @ k)
    ref = np.array(ref).T
    for mode in ("tc", "simt"):
        if mode == "simt":
            os.environ["RLD_NO_TC"] = "1"
        Y = R.kv_apply(torch.from_numpy(V).cuda()).cpu().numpy()[:, rows]
        os.environ.pop("RLD_NO_TC", None)
        relerr = (Y - ref) / ref
        print(f"n={n} {mode}: mean rel err {relerr.mean():+.3e}  max |rel| {np.abs(relerr).max():.3e}", flush=True)
