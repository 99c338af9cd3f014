"""Slice statistics and product times of an on-the-fly float32 problem served from the cached sparse
3-slice image (config 4 by default)."""
import ctypes as C
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = baseline(c)
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path="on_the_fly")
st = (C.c_int64 * 4)()
R.sess.lib.rld_slice_stats(R.sess.handle.ptr, st)
print(f"config{c} n={wl.n}: blocks {st[0]} slices {st[1]} ({st[1] * 4096 / 1e9:.1f} GB, {st[1] / max(st[0], 1):.3f} per block) "
      f"pairs {st[2]} ({st[2] / max(st[0], 1):.3f} per block)", flush=True)
for m in (64, wl.config.precond.rank + 10):
    V = torch.randn(m, wl.n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        R.kv_apply(V)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            R.kv_apply(V)
        torch.cuda.synchronize()
    tot = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            tot[ev.name[:70]] = tot.get(ev.name[:70], 0.0) + ev.device_time / 3e3
    print(f"m={m}: " + "; ".join(f"{k}: {v:.2f} ms" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:5]), flush=True)
