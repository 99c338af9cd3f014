"""Debug: is the fp64 stored (DMMA) estimate deterministic when another estimate runs concurrently?"""
import os
import sys
import threading
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200._session import worker_session  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

wl = baseline(1)
cfg = replace(wl.config, algorithm="r1", path="stored")
M = rld.KernelMatrix(wl.spec, wl.points)
one = rld.rstar_logdet(M, cfg).value
for J in (2, 3):
    out = [None] * J

    def body(j):
        with worker_session():
            out[j] = [rld.rstar_logdet(M, cfg).value for _ in range(3)]

    ths = [threading.Thread(target=body, args=(j,)) for j in range(J)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    print(f"J={J}: max rel dev {max(abs(v - one) / abs(one) for vs in out for v in vs):.2e}", flush=True)
