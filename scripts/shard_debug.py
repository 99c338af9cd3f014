"""Debug: row-sharded (virtual shards) estimate vs single GPU at config 1 for several G / paths."""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.parallel import VirtualShards  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
wl = baseline(1, n=n)
for path in ("stored", "on_the_fly"):
    cfg = replace(wl.config, algorithm="r1", path=path)
    M = rld.KernelMatrix(wl.spec, wl.points)
    one = rld.rstar_logdet(M, cfg)
    for G in (2, 3, 4, 5):
        with VirtualShards(G) as vs:
            r = vs.run(lambda: rld.rstar_logdet(M, cfg))[0]
        print(f"{path} n={n} G={G}: value rel {abs(r.value - one.value) / abs(one.value):.2e} "
              f"logdetP rel {abs(r.logdet_P - one.logdet_P) / abs(one.logdet_P):.2e} "
              f"rank_kept {r.rank_kept}/{one.rank_kept} attempts {r.attempts}/{one.attempts} "
              f"qr_fallback {r.qr_fallback}/{one.qr_fallback}", flush=True)
