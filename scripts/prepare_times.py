"""Kernel times of one float64 stored prepare (config 3: points -> int8 slices -> CRT residues),
the work the e2e leg repeats every step."""
import os
import sys
import time
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

wl = baseline(3, dtype="fp64")
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp64", path="stored")
del R
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp64", path="stored")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    prob, keep = R.sess.problem_for(rld.KernelMatrix(wl.spec, wl.points), "fp64", "stored")
    R.sess.handle.check(R.sess.lib.rld_prepare(R.sess.handle.ptr, __import__("ctypes").byref(prob)), "prepare")
    torch.cuda.synchronize()
    print(f"prepare wall: new resident {1e3 * (t1 - t0):.1f} ms, re-prepare same handle {1e3 * (time.perf_counter() - t1):.1f} ms")
    del R
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp64", path="stored")
    torch.cuda.synchronize()
tot = defaultdict(float)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        tot[ev.name] += ev.device_time
for name, us in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
    print(f"{us:10.1f} us  {name[:100]}")
