"""Repeat fresh-handle estimates and count results that differ from the first (race hunting)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
wl = baseline(cfg)
ref = None
bad = 0
t0 = time.time()
for it in range(iters):
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path=wl.path)
    if it % 2:   # perturb workspace sizes like the test suite does
        R.kv_apply(torch.randn(1 + 37 * it % 300, wl.n, dtype=torch.float64, device="cuda"))
    vals = [R.estimate(wl.config).value for _ in range(2)]
    if ref is None:
        ref = vals[0]
    for v in vals:
        if v != ref:
            bad += 1
            print(f"iter {it}: {v!r} != {ref!r}", flush=True)
    del R
print(f"config {cfg}: {bad} mismatches in {2 * iters} estimates ({time.time() - t0:.1f} s) env={[k for k in os.environ if k.startswith('RLD_')]}")
