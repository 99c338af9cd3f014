"""Debug: per-rank DMMA K.V of virtual shards vs the single-GPU product, sequential and concurrent."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.parallel import VirtualShards, shard_bounds  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

n = 2048
wl = baseline(1, n=n)
M = rld.KernelMatrix(wl.spec, wl.points)
one = rld.ResidentMatrix(M, dtype="fp64", path="stored")
K = rld.build_covariance(wl.spec, wl.points, dtype="fp64")
for m in (8, 16, 74):
    V = torch.randn(m, n, dtype=torch.float64, device="cuda")
    Y = one.kv_apply(V)
    ref = V @ K.T
    print(f"m={m} single vs torch {float((Y - ref).abs().max() / ref.abs().max()):.2e}", flush=True)
    for G in (2, 3):
        with VirtualShards(G) as vs:
            Rs = [rld.ResidentMatrix(M, dtype="fp64", path="stored", session=s) for s in vs.sessions]
            seq = [R.kv_apply(V) for R in Rs]
            conc = vs.run(lambda session: [R for R in Rs if R.sess is session][0].kv_apply(V))
            for r in range(G):
                r0, r1 = shard_bounds(n, G, r)
                a = float((seq[r] - ref[:, r0:r1]).abs().max() / ref.abs().max())
                b = float((conc[r] - ref[:, r0:r1]).abs().max() / ref.abs().max())
                print(f"  G={G} rank {r} rows {r1 - r0}: sequential {a:.2e} concurrent {b:.2e}", flush=True)
            del Rs
