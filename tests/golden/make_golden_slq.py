"""Golden vectors for the SLQ estimator, from the
UNMODIFIED reference ``ratlogdet.slq_logdet`` (src/estimators.py:99-122) run in
this container (the reference cannot travel to the GPU box).

Each case records the estimate, the per-probe values, the clamped Ritz-value
count and a perturbation screen: the change of the estimate under a 1e-15
relative symmetric perturbation of K, which bounds the parity tolerance a case
can support (unpreconditioned Lanczos is more sensitive than the r* path).

Usage (this container only):  OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_slq.py
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

from paper_2405_03474_b200.workloads import baseline  # noqa: E402  (point sets only)

CASES = [(1, None), (2, 4096), (3, 4096), (4, 4096), (5, 4096), (2, None)]


def main():
    out = []
    for idx, n in CASES:
        wl = baseline(idx, n=n)
        spec = ratlogdet.KernelSpec(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter)
        M = ratlogdet.build_covariance(spec, wl.points)
        cfg = ratlogdet.EstimatorConfig("slq", wl.config.num_probes, wl.config.lanczos_iters, wl.config.probe_kind,
                                        seed=wl.config.seed)
        est = ratlogdet.slq_logdet(M, cfg)
        g = np.random.default_rng(12345)
        E = g.standard_normal(M.shape)
        E = 0.5 * (E + E.T)
        pert = ratlogdet.slq_logdet(M * (1.0 + 1e-15 * E), cfg).value
        rec = dict(name=f"slq_{wl.name}_n{wl.n}", workload=wl.name, config_index=idx, n=int(wl.n),
                   algorithm="slq", num_probes=cfg.num_probes, lanczos_iters=cfg.lanczos_iters,
                   probe_kind=cfg.probe_kind, seed=cfg.seed, value=est.value, logdet_P=est.logdet_P,
                   trace_term=est.trace_term, per_probe=[float(x) for x in est.per_probe_values],
                   clamped_eigs=int(est.clamped_eigs), screen=abs(pert - est.value) / abs(est.value))
        print(rec["name"], rec["value"], "screen", rec["screen"], flush=True)
        out.append(rec)
    (HERE / "golden_slq.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
