"""A/B of the on-the-fly float32 K x V kernels: fp16 3-term (kv_otf.cu, default) vs
3xTF32 (kv_tc.cu, RLD_OTF_KIND=tf32).  Accuracy against float64 on small shapes
(all rows) and sampled rows at BASELINE shapes; CUDA-event time per product."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from oracle import rstar_oracle as O  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--small", action="store_true")
ap.add_argument("--configs", default="4,5")
ap.add_argument("--ms", default="")
ap.add_argument("--n5", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--kinds", default="f16,tf32")
a = ap.parse_args()


def product(R, V, kind):
    os.environ["RLD_OTF_KIND"] = kind
    return R.kv_apply(V)


def timed(R, V, kind, reps):
    os.environ["RLD_OTF_KIND"] = kind
    R.kv_apply(V)
    st = torch.cuda.ExternalStream(R.sess.handle.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        Y = R.kv_apply(V)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, Y


if a.small:
    worst = {}
    for fam in ("matern52", "rbf"):
        for d in (1, 2, 3, 4):
            for n, m in ((1000, 1), (1017, 16), (777, 37), (4099, 64), (3001, 130), (2500, 300)):
                g = np.random.default_rng(n + m + d)
                pts = g.uniform(0, 1, (n, d))
                spec = rld.KernelSpec(fam, 1.3, 0.2, 1e-2)
                R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path="on_the_fly")
                V = g.standard_normal((m, n)) * np.exp(g.uniform(-20, 20, (m, 1)))
                Vt = torch.from_numpy(V).cuda()
                K = O.covariance_block(fam, 1.3, 0.2, 1e-2, pts)
                ref = V @ K
                scale = np.abs(V) @ np.abs(K)
                for kind in a.kinds.split(","):
                    Y = product(R, Vt, kind).cpu().numpy()
                    err = float(np.max(np.abs(Y - ref) / scale))
                    worst[kind] = max(worst.get(kind, 0), err)
                    print(f"{fam} d={d} n={n} m={m} {kind}: max normalized err {err:.2e}", flush=True)
    print("worst", worst)

for c in [int(x) for x in a.configs.split(",") if x]:
    wl = baseline(c, n=a.n5 if c == 5 else None)
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path="on_the_fly")
    ms_list = [int(x) for x in a.ms.split(",")] if a.ms else [wl.config.num_probes]
    g = np.random.default_rng(0)
    n = wl.n
    rows = g.choice(n, 6, replace=False)
    kref = [O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points,
                               rows=slice(i, i + 1))[0] for i in rows]
    for m in ms_list:
        V = torch.from_numpy(g.standard_normal((m, n))).cuda()
        Vh = V.cpu().numpy()
        for kind in a.kinds.split(","):
            ms, Y = timed(R, V, kind, a.reps)
            Yh = Y.cpu().numpy()
            err = max(float(np.max(np.abs(Yh[:, i] - Vh @ k) / (np.abs(Vh) @ np.abs(k)))) for i, k in zip(rows, kref))
            print(f"config{c} n={n} m={m} {kind}: {ms:.2f} ms/product, {n * n / ms / 1e9:.3f} T entries/s, "
                  f"{2 * n * n * m / ms / 1e9:.1f} TFLOP/s useful, err {err:.2e}", flush=True)
