"""Generate the golden vectors the oracle and the GPU path are pinned against.

Runs the UNMODIFIED reference package ``ratlogdet`` (imported read-only from
/root/reference/pkg/src) in this container -- the reference cannot travel to
the GPU box, so its outputs are committed as small JSON fixtures:

* ``golden.json``      -- full estimator outputs (value, logdet_P, trace_term,
  per-probe values, exact Cholesky where n permits) for BASELINE configs 1-2 at
  full size and configs 3-5 at reduced n, plus the reference's own
  small-problem fixtures; each case carries a perturbation screen (change of
  the estimate under a 1e-15 relative symmetric perturbation of K), which
  bounds the parity tolerance a case can honestly support.
* ``streams.json``     -- RNG stream fragments (Rademacher probes, Gaussian
  sketch rows, raw Philox words) that pin the device generators bit-for-bit.
* ``units.json``       -- small known-answer vectors (Thomas solves, kernel
  values, CGS2, partial fractions).

Usage (this container only):  OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--quick]
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import ratlogdet  # noqa: E402  (the unmodified reference)
from ratlogdet import bench as rbench  # noqa: E402
from ratlogdet import linalg as rlinalg  # noqa: E402
from ratlogdet import rational as rrational  # noqa: E402

from paper_2405_03474_b200.workloads import baseline  # noqa: E402  (point sets only)


def ref_config(cfg):
    """Our EstimatorConfig -> the reference's (same field values)."""
    return ratlogdet.EstimatorConfig(
        algorithm=cfg.algorithm, num_probes=cfg.num_probes, lanczos_iters=cfg.lanczos_iters,
        probe_kind=cfg.probe_kind,
        precond=ratlogdet.PreconditionerConfig(cfg.precond.kind, cfg.precond.rank, cfg.precond.num_iters,
                                               cfg.precond.scale),
        seed=cfg.seed)


def screen(M, rcfg, value, seed=12345):
    """|Delta estimate| / |estimate| under a 1e-15 relative symmetric perturbation of M."""
    g = np.random.default_rng(seed)
    E = g.standard_normal(M.shape)
    E = 0.5 * (E + E.T)
    Mp = M * (1.0 + 1e-15 * E)
    v2 = ratlogdet.rstar_logdet(Mp, rcfg).value
    return abs(v2 - value) / abs(value)


def run_case(name, wl, algorithm, exact=True, do_screen=True):
    from dataclasses import replace

    cfg = replace(wl.config, algorithm=algorithm)
    spec = ratlogdet.KernelSpec(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter)
    t0 = time.perf_counter()
    M = ratlogdet.build_covariance(spec, wl.points)
    rcfg = ref_config(cfg)
    est = ratlogdet.rstar_logdet(M, rcfg)
    rec = dict(
        name=name, workload=wl.name, n=int(wl.n), d=int(wl.points.shape[1]), family=wl.spec.family,
        amplitude=wl.spec.amplitude, length_scale=wl.spec.length_scale, jitter=wl.spec.jitter,
        algorithm=algorithm, num_probes=cfg.num_probes, lanczos_iters=cfg.lanczos_iters,
        probe_kind=cfg.probe_kind, rank=cfg.precond.rank, num_iters=cfg.precond.num_iters, seed=cfg.seed,
        value=est.value, logdet_P=est.logdet_P, trace_term=est.trace_term,
        per_probe_values=[float(v) for v in est.per_probe_values], ref_wall_time=est.wall_time,
    )
    if exact:
        rec["exact"] = rlinalg.cholesky_logdet(M)
    if do_screen:
        rec["sensitivity"] = screen(M, rcfg, est.value)
    print(f"{name}: value={est.value!r} wall={est.wall_time:.2f}s total={time.perf_counter() - t0:.1f}s "
          f"sens={rec.get('sensitivity')}", flush=True)
    return rec


def estimator_cases(quick):
    cases = []
    # BASELINE config 1, full size, all three orders
    for alg in ("r1", "r3", "r5"):
        cases.append(run_case(f"config1_{alg}", baseline(1), alg))
    # BASELINE config 2, full size n = 16384 (fp64 reference; fp32 GPU runs compare to it too)
    if not quick:
        for alg in ("r1", "r3", "r5"):
            cases.append(run_case(f"config2_{alg}", baseline(2), alg, exact=(alg == "r3"), do_screen=(alg == "r3")))
    # reduced-n configs 3-5: same kernels, point distributions and parameters, n small enough for the CPU
    small = 2048 if quick else 4096
    cases.append(run_case(f"config3_n{small}_r3", baseline(3, n=small), "r3"))
    cases.append(run_case(f"config4_n{small}_r5", baseline(4, n=small), "r5"))
    cases.append(run_case(f"config5_n{small}_r3", baseline(5, n=small, rank=256, num_probes=32), "r3"))
    # config 2 at reduced n, every order (cheap parity cases)
    for alg in ("r1", "r3", "r5"):
        cases.append(run_case(f"config2_n2048_{alg}", baseline(2, n=2048), alg))
    return cases


def fixture_rows():
    """The reference's own fixture (pkg/frontend/tests/fixtures/error_vs_n.csv), regenerated by
    running the reference with one BLAS thread and checked against the committed CSV."""
    path = Path("/root/reference/pkg/frontend/tests/fixtures/error_vs_n.csv")
    rows = []
    with open(path) as fh:
        for r in csv.DictReader(fh):
            if r["algorithm"] == "slq":
                continue
            rc = rbench.RunConfig(kernel_family=r["kernel_family"], n=int(r["n"]), d=int(r["d"]),
                                  jitter=float(r["jitter"]), algorithm=r["algorithm"], s=int(r["s"]),
                                  t=int(r["t"]), precond_rank=int(r["precond_rank"]),
                                  precond_iters=int(r["precond_iters"]), seed=int(r["seed"]))
            rec = rbench.run_single(rc)
            M = rbench.build_matrix(rc)
            sens = screen(M, rc.estimator_config(), rec.estimate)
            rows.append(dict(kernel_family=rc.kernel_family, n=rc.n, d=rc.d, jitter=rc.jitter,
                             algorithm=rc.algorithm, s=rc.s, t=rc.t, precond_rank=rc.precond_rank,
                             precond_iters=rc.precond_iters, seed=rc.seed, estimate=rec.estimate, exact=rec.exact,
                             csv_estimate=float(r["estimate"]), csv_exact=float(r["exact"]), sensitivity=sens))
            print(f"fixture n={rc.n} {rc.algorithm} seed={rc.seed}: est={rec.estimate!r} csv={r['estimate']} "
                  f"sens={sens:.1e}", flush=True)
    return rows


def stream_vectors():
    out = {}
    for seed in (0, 1, 4088532484):
        rng = rlinalg.Rng(seed)
        out[f"rademacher_seed{seed}"] = rng.child(2).rademacher((3, 37)).astype(int).tolist()
        out[f"normal_seed{seed}"] = [float(v) for v in rng.child(1).child(0).normal(64)]
        bg = np.random.Philox(np.random.SeedSequence(seed, spawn_key=(2,)))
        out[f"philox_key_seed{seed}_path2"] = [str(int(k)) for k in bg.state["state"]["key"]]
        out[f"philox_raw_seed{seed}_path2"] = [str(int(v)) for v in bg.random_raw(12)]
    return out


def unit_vectors():
    out = {}
    T = rlinalg.TridiagMatrix(np.array([4.0, 5.0, 6.0, 7.0]), np.array([1.0, 0.5, 0.25]))
    b = np.array([1.0, 0.0, 0.0, 0.0])
    out["thomas"] = dict(diag=T.diag.tolist(), off=T.offdiag.tolist(), shift=0.75, rhs=b.tolist(),
                         x=rlinalg.thomas_solve(T, 0.75, b).tolist())
    rng = rlinalg.Rng(5)
    V = rng.normal((4, 9))
    out["cgs2"] = dict(V=V.tolist(), Q=rlinalg.orthonormalize(V).tolist())
    for fam in ("rbf", "matern52"):
        out[f"kernel_r1_{fam}"] = ratlogdet.kernels.kernel_value(ratlogdet.KernelSpec(fam), [0.0], [1.0])
    for order in (1, 3, 5):
        pf = rrational.partial_fraction(order)
        out[f"pf{order}"] = dict(offset=pf.offset, poles=list(pf.poles), residues=list(pf.residues))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", choices=["streams", "units", "cases", "fixtures"], default=None)
    a = ap.parse_args()
    if os.environ.get("OPENBLAS_NUM_THREADS") != "1":
        print("warning: run with OPENBLAS_NUM_THREADS=1 for bit-reproducible fixture rows", file=sys.stderr)
    if a.only in (None, "streams"):
        (HERE / "streams.json").write_text(json.dumps(stream_vectors(), indent=1))
    if a.only in (None, "units"):
        (HERE / "units.json").write_text(json.dumps(unit_vectors(), indent=1))
    if a.only in (None, "fixtures"):
        (HERE / "fixture_rows.json").write_text(json.dumps(fixture_rows(), indent=1))
    if a.only in (None, "cases"):
        (HERE / "golden.json").write_text(json.dumps(estimator_cases(a.quick), indent=1))


if __name__ == "__main__":
    main()
