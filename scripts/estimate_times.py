"""Wall time (synchronized) of full BASELINE estimates on the on-the-fly path, per K.V kernel
kind (RLD_OTF_KIND), with the phase split the library reports."""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="4,5")
ap.add_argument("--kinds", default="f16,tf32")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
for c in [int(x) for x in a.configs.split(",")]:
    wl = baseline(c)
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=wl.config.dtype, path=wl.path)
    for kind in a.kinds.split(","):
        os.environ["RLD_OTF_KIND"] = kind
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            est = R.estimate(wl.config)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"config{c} n={wl.n} {kind}: {dt:.2f} s/estimate value {est.value!r} "
                  f"phases_ms {[round(x, 1) for x in est.phase_ms]} products {est.kv_products}", flush=True)
