"""Device time of the int8-slice float64 product (ozaki_kv_kernel) at config 3, m = 64 and 522,
from torch.profiler (CUPTI).  RLD_OZ_PROBE=1 / 2 in the environment splits it into its load and
MMA sides (measurement only)."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

wl = baseline(3)
DT = os.environ.get("RLD_PROBE_DTYPE", "fp64")   # fp32: the 3 x 4-slice product of a float32 K
R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=DT, path="stored")
for m in [int(a) for a in sys.argv[1:]] or (64, 522):
    V = torch.randn(m, wl.n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        R.kv_apply(V)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            R.kv_apply(V)
        torch.cuda.synchronize()
    ts = [ev.device_time for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA
          and "ozaki_kv_kernel" in ev.name]
    print(f"{DT} probe={os.environ.get('RLD_OZ_PROBE', '0')} m={m}: ozaki_kv_kernel {sum(ts) / len(ts) / 1e3:.3f} ms "
          f"(n={len(ts)})", flush=True)
