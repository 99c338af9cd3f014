"""Warm per-kernel device times of one estimate (torch.profiler / CUPTI), grouped by kernel name.

  python scripts/kernel_times.py [--config 2] [--n N] [--reps 3]
"""
import argparse
import os
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--dtype", default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
wl = baseline(a.config, n=a.n, dtype=a.dtype)
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=wl.config.dtype, path=wl.path)
for _ in range(2):
    est = R.estimate(wl.config)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        est = R.estimate(wl.config)
    torch.cuda.synchronize()
tot = defaultdict(float)
cnt = defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        tot[ev.name] += ev.device_time
        cnt[ev.name] += 1
all_us = sum(tot.values()) / a.reps
print(f"phases {[round(x, 3) for x in est.phase_ms]}  kernel-sum/estimate {all_us:.1f} us")
for name, us in sorted(tot.items(), key=lambda kv: -kv[1])[: a.top]:
    print(f"{us / a.reps:9.1f} us {cnt[name] / a.reps:6.1f}x  {name[:110]}")

# device idle gaps of the last estimate: intervals with no kernel / copy running (union over streams)
evs = sorted([(ev.time_range.start, ev.time_range.end, ev.name) for ev in prof.events()
              if ev.device_type == torch.autograd.DeviceType.CUDA], key=lambda x: x[0])
per = len(evs) // a.reps
last = evs[-per:]
gaps, cur_end, prev = [], last[0][1], last[0][2]
for s0, e0, nm in last[1:]:
    if s0 > cur_end:
        gaps.append((s0 - cur_end, prev[:60], nm[:60]))
    if e0 > cur_end:
        cur_end, prev = e0, nm
span = last[-1][1] - last[0][0]
print(f"last estimate: span {span / 1e3:.2f} ms, idle {sum(g[0] for g in gaps) / 1e3:.2f} ms in {len(gaps)} gaps")
for g in sorted(gaps, reverse=True)[:15]:
    print(f"  gap {g[0]:8.1f} us  after {g[1]}  before {g[2]}")
