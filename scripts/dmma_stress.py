"""Stress: fp64 stored K.V (DMMA) from several host threads / handles at once, every result
checked against torch float64."""
import os
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200._session import worker_session  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = baseline(1)
M = rld.KernelMatrix(wl.spec, wl.points)
K = rld.build_covariance(wl.spec, wl.points, dtype="fp64")
torch.cuda.synchronize()
bad = []


def body(j):
    with worker_session() as s:
        R = rld.ResidentMatrix(M, dtype="fp64", path="stored", session=s)
        g = torch.Generator(device="cuda").manual_seed(j)
        for it in range(reps):
            m = (16, 74, 80, 266, 3)[(it + j) % 5]
            V = torch.randn(m, wl.n, dtype=torch.float64, device="cuda", generator=g)
            Y = R.kv_apply(V)
            ref = V @ K.T
            torch.cuda.synchronize()
            e = float((Y - ref).abs().max() / ref.abs().max())
            if e > 1e-13:
                bad.append((j, it, m, e))


ths = [threading.Thread(target=body, args=(j,)) for j in range(J)]
[t.start() for t in ths]
[t.join() for t in ths]
print(f"J={J} reps={reps}: {len(bad)} bad products", bad[:10], flush=True)
