"""Effect of RLD_FP64_SKETCH_DIAGS (slice-pair diagonals of the int8-slice float64 product in the
first q-1 power iterations) on the config-3 / config-1 float64 estimates and their time."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

gl = json.load(open("tests/golden/golden_large.json"))
g1 = {c["name"]: c for c in json.load(open("tests/golden/golden.json"))}
for c, ref in ((3, gl["config3_full"]["value"]), (1, g1["config1_r3"]["value"]), (2, g1["config2_r3"]["value"])):
    wl = baseline(c, dtype="fp64")
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp64", path="stored")
    est = R.estimate(wl.config)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        est = R.estimate(wl.config)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"diags={os.environ.get('RLD_FP64_SKETCH_DIAGS', '8')} config{c}: {dt * 1e3:.1f} ms value {est.value!r} "
          f"rel vs golden {abs(est.value - ref) / abs(ref):.2e} logdetP {est.logdet_P!r} phases "
          f"{[round(x, 1) for x in est.phase_ms]}", flush=True)
    del R
    torch.cuda.empty_cache()
