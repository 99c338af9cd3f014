"""The reference harness's wire format (src/bench.py:47-265) produced by the GPU
build: field names and order, trial seeds, sweep order, %.17g CSV round trip,
failures as records.  Golden values: tests/golden/make_golden_harness.py (run
against the unmodified reference in this container)."""

import math
from dataclasses import asdict

import pytest

from conftest import load_golden, rel
from paper_2405_03474_b200 import harness as H


@pytest.fixture(scope="module")
def golden():
    return load_golden("harness.json")


def test_record_fields_extend_reference(golden):
    assert H.REFERENCE_FIELDS == golden["record_fields"]
    assert H.RECORD_FIELDS[:17] == golden["record_fields"]


def test_trial_seeds_match_reference(golden):
    for sb, vi, tr, seed in golden["trial_seeds"]:
        assert H.trial_seed(sb, vi, tr) == seed


def test_sweep_order_matches_reference(golden):
    spec = H.SweepSpec("n", (200, 400), ("r1", "r3", "slq"), trials=2, seed_base=0)
    got = [asdict(c) for c in H.sweep_configs(spec)]
    want = golden["sweep"]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert {k: g[k] for k in w} == w


def test_sweep_spec_validation():
    with pytest.raises(ValueError):
        H.SweepSpec("bogus", (1,))
    with pytest.raises(ValueError):
        H.SweepSpec("n", ())
    with pytest.raises(ValueError):
        H.SweepSpec("n", (10,), trials=0)
    with pytest.raises(ValueError):
        H.SweepSpec("n", (10,), algorithms=("r2",))


def _records():
    base = dict(kernel_family="rbf", n=400, d=1, jitter=1e-6, algorithm="r3", probe_kind="rademacher", s=35, t=20,
                precond_kind="rand-svd", precond_rank=25, precond_iters=5, seed=4088532484)
    return [H.BenchRecord(**base, estimate=-5366.725170811625, exact=-5366.2, abs_error=0.1 + 0.2,
                          wall_time_ms=1.0 / 3.0, dtype="fp64", path="stored", device_time_ms=2.0 / 7.0,
                          kv_products=26),
            H.BenchRecord(**base, estimate=None, exact=None, abs_error=None, wall_time_ms=None,
                          error="NotPositiveDefinite: x", dtype="fp32")]


def test_csv_round_trip_is_exact(tmp_path):
    recs = _records()
    p = tmp_path / "r.csv"
    H.emit_csv(recs, p)
    header = p.read_text().splitlines()[0].split(",")
    assert header == H.RECORD_FIELDS
    assert H.read_csv(p) == recs


def test_read_reference_csv_columns(tmp_path, golden):
    """A CSV with only the reference's 17 columns reads back with the B200 fields None."""
    import csv

    p = tmp_path / "ref.csv"
    rec = _records()[0]
    d = asdict(rec)
    with open(p, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(golden["record_fields"])
        w.writerow([H._format_cell(k, d[k]) for k in golden["record_fields"]])
    back = H.read_csv(p)[0]
    assert back.estimate == rec.estimate and back.dtype is None and back.kv_products is None


def test_emit_json(tmp_path):
    import json

    p = tmp_path / "r.json"
    H.emit_json(_records(), p)
    assert json.loads(p.read_text())[1]["error"].startswith("NotPositiveDefinite")


@pytest.mark.gpu
def test_run_single_gpu_matches_oracle():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import rstar_oracle as O

    cfg = H.RunConfig("matern52", n=600, d=2, jitter=1e-2, algorithm="r3", s=8, precond_rank=16)
    rec = H.run_single(cfg)
    assert rec.error is None, rec.error
    M = H.build_matrix(cfg)
    K = O.covariance_block("matern52", 1.0, 1.0, 1e-2, M.points)
    ref = O.rstar_dense(K, order=3, s=8, t=20, k=16, q=5, seed=0)
    assert rel(rec.estimate, ref.value) <= 1e-6
    assert rel(rec.exact, O.cholesky_logdet(K)) <= 1e-10
    assert math.isclose(rec.abs_error, abs(rec.estimate - rec.exact))
    assert rec.path == "stored" and rec.kv_products > 0


@pytest.mark.gpu
def test_run_single_failure_becomes_record():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rec = H.run_single(H.RunConfig(n=10, precond_rank=11))   # rank > n -> ValueError (src/precond.py:241-242)
    assert rec.estimate is None and rec.error.startswith("ValueError")


@pytest.mark.gpu
def test_sweep_is_deterministic_and_paired():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec = H.SweepSpec("n", (300, 500), ("r3", "slq"), base=H.RunConfig(jitter=1e-3, s=6), trials=2)
    a, b = H.run_sweep(spec), H.run_sweep(spec)
    assert [r.estimate for r in a] == [r.estimate for r in b]
    # algorithms of one (value, trial) share the seed and the exact log det
    for r1, r2 in zip(a[0::2], a[1::2]):
        assert r1.seed == r2.seed and r1.exact == r2.exact


@pytest.mark.gpu
def test_sweep_jobs_run_concurrently_with_identical_records():
    """jobs > 1: worker threads with their own device handles (the reference's --jobs runs
    processes, src/bench.py:209-215); every record equals the serial one, in the same order."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec = H.SweepSpec("probes", (4, 8, 12), ("r1", "r3"), base=H.RunConfig(n=400, jitter=1e-3), trials=2)
    serial = H.run_sweep(spec)
    par = H.run_sweep(spec, jobs=3)
    key = lambda r: (r.n, r.s, r.seed, r.algorithm, r.estimate, r.exact, r.error)   # noqa: E731
    assert [key(r) for r in par] == [key(r) for r in serial]
    assert all(r.error is None for r in par)
