"""Golden values at full BASELINE sizes (configs 3-5), from the matrix-free float64 oracle.

The unmodified reference cannot run there (its dense float64 K would be 34 GB / 550 GB /
8.8 TB), so these values come from the oracle's numpy restatement of the
estimator (``oracle/rstar_oracle.py``: ``src/estimators.py:58-96``, ``src/precond.py:69-115,
168-198, 231-267``, ``src/lanczos.py:34-84``, ``src/linalg.py:125-180``) driving the
matrix-free C++/OpenMP operator (``oracle/mf_kv.cpp``: ``src/kernels.py:40-46, 59-73``).

Before the oracle is trusted at full size it is validated HERE against the unmodified
reference (imported read-only from /root/reference/pkg/src) where the reference still fits in
host RAM: BASELINE config 2 at full n = 16384 (reference values from ``golden.json``) and
config-3 / config-4-style point sets at n = 24576 / 16384 (the reference is run by this
script).  Each validation row records both values and their relative difference.

Every full-size case carries a perturbation screen: the change of the estimate when every
K_ij is multiplied by (1 + 1e-15 h_ij), h symmetric in [-1, 1) -- the floor below which two
correct float64 implementations cannot be told apart.  Configs 4 and 5 screen at reduced n
(stated in the row) because one more full-size run would cost another hour of CPU.

Config 5 runs at n = 2^20 with a reduced preconditioner rank, probe count and iteration
counts (stated in the row): the kernel, the point distribution and n are BASELINE's.

Usage (this container; minutes to hours, run under nice):
  python tests/golden/make_golden_large.py validate|config3|config4|config5|screens
Results merge into tests/golden/golden_large.json.
"""

from __future__ import annotations

import json
import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import mf  # noqa: E402
from oracle import rstar_oracle as O  # noqa: E402
from paper_2405_03474_b200.workloads import baseline  # noqa: E402

OUT = HERE / "golden_large.json"
PERT = 1e-15

# config 5 at n = 2^20: reduced rank / probes / iterations (everything else BASELINE)
C5 = dict(rank=32, num_probes=8, lanczos_iters=10, num_iters=2)


def load():
    return json.loads(OUT.read_text()) if OUT.exists() else {}


def save(key, rec):
    d = load()
    d[key] = rec
    OUT.write_text(json.dumps(d, indent=1))
    print(f"saved {key}", flush=True)


def oracle_run(wl, pert=0.0):
    cfg = wl.config
    X = wl.points
    op = mf.NativePointsOperator(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, X,
                                 pert=pert)
    t0 = time.perf_counter()
    est = O.rstar(op, op.n, int(cfg.algorithm[1]), cfg.num_probes, cfg.lanczos_iters, cfg.probe_kind,
                  cfg.precond.rank, cfg.precond.num_iters, cfg.seed)
    dt = time.perf_counter() - t0
    print(f"  oracle n={op.n} pert={pert}: {est.value!r} ({dt:.0f} s, {op.calls} products)", flush=True)
    return est, dt, op.calls


def case_record(name, wl, est, dt, products, note=""):
    cfg = wl.config
    return dict(
        name=name, workload=wl.name, n=int(wl.n), d=int(wl.points.shape[1]), family=wl.spec.family,
        amplitude=wl.spec.amplitude, length_scale=wl.spec.length_scale, jitter=wl.spec.jitter,
        algorithm=cfg.algorithm, num_probes=cfg.num_probes, lanczos_iters=cfg.lanczos_iters,
        probe_kind=cfg.probe_kind, rank=cfg.precond.rank, num_iters=cfg.precond.num_iters, seed=cfg.seed,
        value=est.value, logdet_P=est.logdet_P, trace_term=est.trace_term,
        per_probe_values=[float(v) for v in est.per_probe_values], attempts=est.attempts,
        oracle_seconds=dt, oracle_products=products, oracle_threads=mf.threads(),
        oracle="rstar_oracle.rstar + mf.NativePointsOperator (float64, matrix-free)", note=note)


def screen_of(wl, value):
    est, dt, _ = oracle_run(wl, pert=PERT)
    return abs(est.value - value) / abs(value), est.value, dt


def validate():
    sys.path.insert(0, "/root/reference/pkg/src")
    import ratlogdet  # the unmodified reference

    rows = []
    gold = {c["name"]: c for c in json.loads((HERE / "golden.json").read_text())}
    # config 2, full n = 16384: the reference's value is in golden.json
    wl = baseline(2, dtype="fp64")
    est, dt, _ = oracle_run(wl)
    ref = gold["config2_r3"]["value"]
    rows.append(dict(case="config2_r3 n=16384", reference=ref, oracle=est.value,
                     rel=abs(est.value - ref) / abs(ref), oracle_seconds=dt))
    print(rows[-1], flush=True)
    for idx, n in ((3, 24576), (4, 16384), (5, 16384)):
        extra = dict(rank=256, num_probes=32) if idx == 5 else {}
        wl = baseline(idx, n=n, dtype="fp64", **extra)
        spec = ratlogdet.KernelSpec(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter)
        t0 = time.perf_counter()
        M = ratlogdet.build_covariance(spec, wl.points)
        r = ratlogdet.rstar_logdet(M, ref_config(wl.config))
        del M
        tr = time.perf_counter() - t0
        est, dt, _ = oracle_run(wl)
        rows.append(dict(case=f"config{idx}-style n={n} {wl.config.algorithm} l={wl.config.precond.rank} "
                              f"s={wl.config.num_probes}",
                         reference=r.value, reference_logdet_P=r.logdet_P, oracle=est.value,
                         oracle_logdet_P=est.logdet_P, rel=abs(est.value - r.value) / abs(r.value),
                         reference_seconds=tr, oracle_seconds=dt))
        print(rows[-1], flush=True)
    save("validation", rows)


def ref_config(cfg):
    import ratlogdet

    return ratlogdet.EstimatorConfig(
        algorithm=cfg.algorithm, num_probes=cfg.num_probes, lanczos_iters=cfg.lanczos_iters,
        probe_kind=cfg.probe_kind,
        precond=ratlogdet.PreconditionerConfig(cfg.precond.kind, cfg.precond.rank, cfg.precond.num_iters,
                                               cfg.precond.scale),
        seed=cfg.seed)


def config5_workload(n=None):
    wl = baseline(5, n=n, dtype="fp64", rank=C5["rank"], num_probes=C5["num_probes"])
    cfg = replace(wl.config, lanczos_iters=C5["lanczos_iters"],
                  precond=replace(wl.config.precond, num_iters=C5["num_iters"]))
    return replace(wl, config=cfg)


def full(idx):
    if idx == 5:
        wl = config5_workload()
        note = (f"n = 2^20 with reduced l = {C5['rank']}, s = {C5['num_probes']}, t = {C5['lanczos_iters']}, "
                f"q = {C5['num_iters']} (BASELINE: l = 2048, s = 128, t = 20, q = 5)")
    else:
        wl = baseline(idx, dtype="fp64")
        note = "full BASELINE configuration"
    est, dt, calls = oracle_run(wl)
    rec = case_record(f"config{idx}_full", wl, est, dt, calls, note)
    if idx == 3:
        sens, pv, sdt = screen_of(wl, est.value)
        rec.update(sensitivity=sens, sensitivity_n=wl.n, perturbed_value=pv)
    save(f"config{idx}_full", rec)


def screens():
    """Perturbation screens of configs 4 and 5 at reduced n (same kernel, points, parameters)."""
    d = {}
    for idx, n in ((4, 32768), (5, 32768)):
        wl = config5_workload(n) if idx == 5 else baseline(idx, n=n, dtype="fp64")
        est, dt, _ = oracle_run(wl)
        sens, pv, _ = screen_of(wl, est.value)
        d[f"config{idx}"] = dict(n=n, value=est.value, perturbed_value=pv, sensitivity=sens)
        print(d, flush=True)
    save("screens_reduced", d)


if __name__ == "__main__":
    sys.path.insert(0, str(HERE.parent))
    what = sys.argv[1]
    mf.build()
    if what == "validate":
        validate()
    elif what.startswith("config"):
        full(int(what[-1]))
    elif what == "screens":
        screens()
    else:
        raise SystemExit(f"unknown mode {what}")
