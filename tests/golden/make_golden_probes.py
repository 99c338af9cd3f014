"""Golden vectors for normal-orthogonal probes (src/probes.py:15-44)
from the UNMODIFIED reference, run in this container only:
the probe rows themselves for small shapes (including s > n, several blocks) and full
r3 / SLQ estimates that use them.

Usage:  OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_probes.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import ratlogdet  # noqa: E402  (the unmodified reference)
from ratlogdet.linalg import Rng  # noqa: E402
from ratlogdet.probes import make_probes  # noqa: E402

from paper_2405_03474_b200.workloads import baseline  # noqa: E402  (point sets only)


def main():
    out = {"probes": [], "estimates": []}
    for seed, s, n in [(0, 5, 40), (3, 50, 20), (7, 8, 300)]:
        P = make_probes("normal-orthogonal", s, n, Rng(seed).child(2))
        out["probes"].append(dict(seed=seed, s=s, n=n, rows=P.tolist()))
    for idx, n, alg in [(1, 768, "r3"), (1, 768, "slq"), (3, 1024, "r5")]:
        wl = baseline(idx, n=n)
        spec = ratlogdet.KernelSpec(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter)
        M = ratlogdet.build_covariance(spec, wl.points)
        cfg = ratlogdet.EstimatorConfig(alg, 8, 20, "normal-orthogonal", ratlogdet.PreconditionerConfig("rand-svd", 48, 5),
                                        seed=0)
        est = ratlogdet.estimate_logdet(M, cfg)
        out["estimates"].append(dict(name=f"{alg}_normal-orthogonal_{wl.name}_n{n}", config_index=idx, n=n,
                                     algorithm=alg, rank=48, num_probes=8, seed=0, value=est.value,
                                     per_probe=[float(x) for x in est.per_probe_values]))
        print(out["estimates"][-1]["name"], est.value, flush=True)
    (HERE / "golden_probes.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main()
