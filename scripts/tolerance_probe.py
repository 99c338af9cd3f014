"""Measure the parity gaps the tightened tests pin: the reference fixture rows (GPU from points,
GPU from the oracle's dense K, against the reference's stored estimate), the partial-Cholesky
stored-vs-on-the-fly pair (fp64), and the well-posed partial-Cholesky golden cases."""
import json
import os
import sys
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
import paper_2405_03474_b200 as rld  # noqa: E402
from oracle import rstar_oracle as O  # noqa: E402
from paper_2405_03474_b200.linalg import Rng  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

rows = json.load(open(os.path.join(HERE, "tests/golden/fixture_rows.json")))
worst = 0.0
for r in rows:
    pts = Rng(r["seed"]).child(0).normal((r["n"], r["d"]))
    cfg = rld.EstimatorConfig(r["algorithm"], r["s"], r["t"], "rademacher",
                              rld.PreconditionerConfig("rand-svd", r["precond_rank"], r["precond_iters"],
                                                       max(r["jitter"], 1e-12)), r["seed"])
    a = rld.rstar_logdet(rld.KernelMatrix(rld.KernelSpec("rbf", jitter=r["jitter"]), pts), cfg).value
    K = O.covariance_block("rbf", 1.0, 1.0, r["jitter"], pts)
    b = rld.rstar_logdet(K, cfg).value
    ra, rb = abs(a - r["estimate"]) / abs(r["estimate"]), abs(b - r["estimate"]) / abs(r["estimate"])
    worst = max(worst, ra / r["sensitivity"], rb / r["sensitivity"])
    print(f"fixture n={r['n']} {r['algorithm']} sens {r['sensitivity']:.1e}: points {ra:.1e} dense {rb:.1e}")
print(f"fixture worst gap / sensitivity: {worst:.1f}")
wl = baseline(5, n=2048)
cfg = replace(wl.config, dtype="fp64", num_probes=8, precond=rld.PreconditionerConfig("partial-cholesky", 64, 5))
a = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(cfg, path="stored"))
b = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(cfg, path="on_the_fly"))
print(f"pchol stored vs otf: value {abs(a.value - b.value) / abs(a.value):.2e} "
      f"logdetP {abs(a.logdet_P - b.logdet_P) / abs(a.logdet_P):.2e}")
for c in json.load(open(os.path.join(HERE, "tests/golden/golden_precond_wellposed.json"))):
    wl = baseline(c["config_index"], n=c["n"])
    K = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points)
    K = K + np.diag(np.random.default_rng(c["diag_offsets_seed"]).uniform(0.0, c["diag_offsets_max"], c["n"]))
    cf = rld.EstimatorConfig("r3", c["num_probes"], 20, "rademacher",
                             rld.PreconditionerConfig(c["kind"], c["rank"], c["num_iters"], c["scale"]), c["seed"])
    e = rld.rstar_logdet(K, cf)
    print(f"{c['name']}: {abs(e.value - c['value']) / abs(c['value']):.2e} (screen {c['screen']:.1e})")
