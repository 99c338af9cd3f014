"""INT8-sliced float64 K.V (kv_ozaki.cu, RLD_FP64_PRODUCT=ozaki): accuracy against torch float64
and against the DMMA product, timing at the BASELINE shapes, and an estimate vs the golden value."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

assert os.environ.get("RLD_FP64_PRODUCT", "ozaki") == "ozaki"
shapes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["1:2048:16", "2:4099:37", "2:16384:32", "2:16384:266"]
for sh in shapes:
    cfg, n, m = (int(x) for x in sh.split(":"))
    wl = baseline(cfg, n=n)
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp64", path="stored")
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn(m, wl.n, dtype=torch.float64, device="cuda", generator=g)
    Y = R.kv_apply(V)
    torch.cuda.synchronize()
    rec = {"shape": sh}
    if wl.n <= 16384:
        K = rld.build_covariance(wl.spec, wl.points, dtype="fp64")
        ref = V @ K.T
        scale = V.abs() @ K.abs().T
        rec["max_err_over_abs_scale"] = float(((Y - ref).abs() / scale).max())
        rec["max_rel_err"] = float((Y - ref).abs().max() / ref.abs().max())
        del K, ref, scale
    st = torch.cuda.ExternalStream(R.sess.handle.stream)
    for _ in range(2):
        R.kv_apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        R.kv_apply(V)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    rec.update(ms=ms, equiv_fp64_tflops=2.0 * wl.n * wl.n * m / (ms * 1e-3) / 1e12)
    print(json.dumps(rec), flush=True)
    del R, V, Y
    torch.cuda.empty_cache()
