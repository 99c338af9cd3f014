"""One device-resident estimate of a BASELINE config (for launch-list profiling)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--dtype", default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
wl = baseline(a.config, n=a.n, dtype=a.dtype)
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=wl.config.dtype, path=wl.path)
for _ in range(a.reps):
    est = R.estimate(wl.config)
torch.cuda.synchronize()
print(f"value {est.value!r} phases {[round(x, 3) for x in est.phase_ms]} launches {est.kernel_launches}")
