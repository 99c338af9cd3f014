"""Debug: sharded vs single for the non-rand-svd preconditioners (reorthogonalised Lanczos)."""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.parallel import VirtualShards  # noqa: E402
from paper_2405_03474_b200.precond import PreconditionerConfig  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

wl = baseline(1, n=1500)
for kind in ("partial-cholesky", "diagonal", "rank-one", "rand-svd-scaled", "identity"):
    for path in ("stored", "on_the_fly"):
        cfg = replace(wl.config, precond=PreconditionerConfig(kind, 40, 5), dtype="fp64", path=path)
        M = rld.KernelMatrix(wl.spec, wl.points)
        one = rld.rstar_logdet(M, cfg)
        one2 = rld.rstar_logdet(M, cfg)
        out = []
        for G in (2, 3):
            with VirtualShards(G) as vs:
                r = vs.run(lambda: rld.rstar_logdet(M, cfg))[0]
            out.append(f"G={G} {abs(r.value - one.value) / abs(one.value):.1e}")
        print(f"{kind:18s} {path:10s} repeat {abs(one2.value - one.value) / abs(one.value):.1e} " + " ".join(out),
              flush=True)
