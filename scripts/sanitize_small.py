"""Small estimates that exercise every own kernel family (tcgen05 K.V stored and on the fly, the
DMMA products, cluster Cholesky, eigensolver, RNG) for compute-sanitizer runs."""
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_03474_b200 as rld  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

wl = baseline(1, n=640, rank=32, num_probes=8)
M = rld.KernelMatrix(wl.spec, wl.points)
for dtype, path in (("fp64", "stored"), ("fp32", "stored"), ("fp32", "on_the_fly")):
    e = rld.rstar_logdet(M, replace(wl.config, dtype=dtype, path=path))
    print(dtype, path, e.value, flush=True)
wl = baseline(2, n=1024, rank=96, num_probes=64)   # CTA pairs (NT >= 64) on the tensor-core kernel
e = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(wl.config, dtype="fp32"))
print("pairs", e.value, flush=True)
