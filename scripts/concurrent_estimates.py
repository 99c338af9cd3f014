"""Throughput of J independent estimates running concurrently on one GPU (one handle, stream and
K copy per worker thread; ctypes releases the GIL during each estimate)."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
per = int(sys.argv[2]) if len(sys.argv) > 2 else 10
wl = baseline(cfg)
for J in (1, 2, 3, 4):
    Rs = [rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=wl.config.dtype, path=wl.path)
          for _ in range(J)]
    for R in Rs:
        R.estimate(wl.config)
    torch.cuda.synchronize()
    vals = [[] for _ in range(J)]

    def work(i):
        for _ in range(per):
            vals[i].append(Rs[i].estimate(wl.config).value)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(J)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    same = all(v == vals[0][0] for vs in vals for v in vs)
    print(f"config {cfg}: J={J} concurrent handles: {J * per / dt:.1f} estimates/s (identical results: {same})",
          flush=True)
    del Rs
