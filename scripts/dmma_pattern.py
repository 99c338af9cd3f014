"""Diagnose intermittent DMMA product errors: where are the wrong outputs, and does the error
equal the contribution of a whole 16-column k-step (missing / duplicated / stale stage)?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

wl = baseline(1)
n = wl.n
M = rld.KernelMatrix(wl.spec, wl.points)
R = rld.ResidentMatrix(M, dtype="fp64", path="stored")
K = rld.build_covariance(wl.spec, wl.points, dtype="fp64")
g = torch.Generator(device="cuda").manual_seed(0)
shown = 0
for it in range(200):
    m = (16, 74, 80, 266, 3)[it % 5]
    V = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    Y = R.kv_apply(V)
    ref = V @ K.T
    torch.cuda.synchronize()
    err = (Y - ref).abs()
    bad = err > 1e-12 * ref.abs().max()
    if not bad.any():
        continue
    cs, rs = torch.nonzero(bad, as_tuple=True)
    print(f"it {it} m={m}: {int(bad.sum())} bad of {bad.numel()}; cols(vec) {int(cs.min())}..{int(cs.max())} "
          f"rows {int(rs.min())}..{int(rs.max())} uniq rows%128 {len(set((rs % 128).tolist()))} "
          f"uniq vec {len(set(cs.tolist()))}", flush=True)
    # per-k-step contribution test on the first bad entry
    c, i = int(cs[0]), int(rs[0])
    d = float((Y - ref)[c, i])
    contrib = (K[i] * V[c]).reshape(-1, 16).sum(1)
    best = torch.argmin((contrib - d).abs())
    bestn = torch.argmin((contrib + d).abs())
    print(f"   entry ({c},{i}) diff {d:.3e}; closest +step {int(best)} {float(contrib[best]):.3e}; "
          f"closest -step {int(bestn)} {float(-contrib[bestn]):.3e}", flush=True)
    shown += 1
    if shown >= 6:
        break
print("done")
