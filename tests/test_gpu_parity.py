"""GPU parity: the CUDA path (through librld.so's C ABI) against the reference's
golden outputs and the CPU oracle.

Tolerances (north_star): <= 1e-6 relative on log det in fp64 mode, <= 1e-4 in
fp32 mode, given identical probes and sketch rows from the same seed.
"""

from dataclasses import replace

import numpy as np
import pytest

from conftest import rel
from oracle import rstar_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-6, "fp32": 1e-4}


@pytest.fixture(scope="module")
def rld():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03474_b200 as rld

    return rld


def workload(c):
    from paper_2405_03474_b200.workloads import baseline

    return baseline(int(c["workload"][6]), n=c["n"], rank=c["rank"], num_probes=c["num_probes"])


def gpu_estimate(rld, c, dtype, path="stored", source="points"):
    wl = workload(c)
    cfg = replace(wl.config, algorithm=c["algorithm"], dtype=dtype, path=path)
    if source == "points":
        M = rld.KernelMatrix(wl.spec, wl.points)
    elif source == "numpy":
        M = O.covariance_block(c["family"], c["amplitude"], c["length_scale"], c["jitter"], wl.points)
    else:
        M = rld.build_covariance(wl.spec, wl.points, dtype=dtype)
    return rld.rstar_logdet(M, cfg)


# ---------------------------------------------------------------- generators

@pytest.mark.parametrize("shape", [(3, 37), (16, 2048), (5, 100001), (1, 1)])
@pytest.mark.parametrize("seed", [0, 1, 4088532484])
def test_device_rademacher_is_numpy_stream(rld, shape, seed):
    import ctypes as C
    import torch

    from paper_2405_03474_b200._session import session
    from paper_2405_03474_b200.linalg import Rng, philox_key

    s = session()
    out = torch.empty(shape, dtype=torch.float64, device="cuda")
    key = (C.c_uint64 * 2)(*philox_key(seed, (2,)))
    s.handle.check(s.lib.rld_rademacher(s.handle.ptr, C.byref(key), shape[0], shape[1], out.data_ptr()), "rademacher")
    ref = Rng(seed).child(2).rademacher(shape)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("shape", [(1, 1), (3, 37), (266, 16384), (7, 1000003)])
@pytest.mark.parametrize("seed,path", [(0, (1, 0)), (1, (1, 1)), (4088532484, (2,))])
def test_device_normal_is_numpy_stream(rld, shape, seed, path):
    """numpy's Generator.standard_normal (ziggurat over Philox) reproduced on the device."""
    import ctypes as C
    import torch

    from paper_2405_03474_b200._session import session
    from paper_2405_03474_b200.linalg import Rng, philox_key

    s = session()
    out = torch.empty(shape, dtype=torch.float64, device="cuda")
    key = (C.c_uint64 * 2)(*philox_key(seed, path))
    s.handle.check(s.lib.rld_normal(s.handle.ptr, C.byref(key), shape[0], shape[1], out.data_ptr()), "normal")
    got = out.cpu().numpy()
    ref = Rng(seed, path).normal(shape)
    diff = got != ref
    # bit-exact except possibly the last bit of ziggurat-tail draws (|x| > r), where CUDA's
    # log1p may round differently from glibc's
    assert np.all(np.abs(ref[diff]) > 3.6541528853610088)
    np.testing.assert_allclose(got, ref, rtol=4e-16, atol=0)
    assert diff.sum() <= max(2, 1e-4 * ref.size)


@pytest.mark.parametrize("family,ell,d", [("rbf", 1.0, 8), ("matern52", 0.2, 3), ("matern52", 0.05, 2)])
def test_build_covariance_matches_reference_formula(rld, family, ell, d):
    g = np.random.default_rng(3)
    pts = g.uniform(0, 1, (777, d))
    spec = rld.KernelSpec(family, 1.3, ell, 1e-2)
    K = rld.build_covariance(spec, pts, dtype="fp64").cpu().numpy()
    ref = O.covariance_block(family, 1.3, ell, 1e-2, pts)
    np.testing.assert_allclose(K, ref, rtol=1e-11, atol=1e-14)
    assert np.all(np.diag(K) == 1.3 ** 2 + 1e-2)
    # float32 K: float64 r^2, float32 kernel function (MUFU exp): a few float32 ulps
    K32 = rld.build_covariance(spec, pts, dtype="fp32", device="cpu")
    np.testing.assert_allclose(K32, ref, rtol=1e-6, atol=1e-7)
    assert np.all(np.diag(K32) == np.float32(1.3 ** 2 + 1e-2))


@pytest.mark.parametrize("dtype,path", [("fp64", "stored"), ("fp32", "stored"), ("fp64", "on_the_fly"),
                                        ("fp32", "on_the_fly")])
@pytest.mark.parametrize("m", [1, 16, 37])
def test_kv_apply_matches_numpy(rld, dtype, path, m):
    import torch

    g = np.random.default_rng(m)
    n = 1000 + m
    pts = g.uniform(0, 1, (n, 3))
    spec = rld.KernelSpec("matern52", 1.0, 0.2, 1e-2)
    R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype=dtype, path=path)
    V = g.standard_normal((m, n))
    Y = R.kv_apply(torch.from_numpy(V).cuda()).cpu().numpy()
    K = O.covariance_block("matern52", 1.0, 0.2, 1e-2, pts)
    ref = V @ K
    scale = np.abs(V) @ np.abs(K)
    err = np.max(np.abs(Y - ref) / scale)
    assert err <= (1e-13 if dtype == "fp64" else 2e-6), err


@pytest.mark.parametrize("n,m", [(256, 32), (1000, 1), (4099, 64), (16384, 32), (3000, 300), (2048, 400),
                                 (20000, 128), (700, 17), (5000, 266), (1500, 140), (3001, 522)])
def test_tcgen05_product_matches_float64(rld, n, m):
    """fp32 stored K goes through the tcgen05 3xTF32 kernel (stream-K, TMEM A
    operand); check it against float64 numpy and against the CUDA-core path."""
    import os

    import torch

    g = np.random.default_rng(n + m)
    pts = g.standard_normal((n, 4))
    spec = rld.KernelSpec("rbf", 1.0, 1.5, 1e-3)
    R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path="stored")
    V = g.standard_normal((m, n))
    Vt = torch.from_numpy(V).cuda()
    Y = R.kv_apply(Vt).cpu().numpy()
    K = O.covariance_block("rbf", 1.0, 1.5, 1e-3, pts)
    K32 = K.astype(np.float32).astype(np.float64)      # the stored matrix
    scale = np.abs(V) @ np.abs(K)
    err_tc = np.max(np.abs(Y - V @ K32) / scale)
    tol = 2e-6 + 1e-7 * np.sqrt(n)     # fp32 accumulation over n terms
    assert err_tc <= tol, err_tc
    os.environ["RLD_NO_TC"] = "1"
    try:
        Ys = R.kv_apply(Vt).cpu().numpy()
    finally:
        del os.environ["RLD_NO_TC"]
    assert np.max(np.abs(Ys - V @ K32) / scale) <= tol


# ---------------------------------------------------------------- estimator parity

@pytest.mark.parametrize("alg", ["r1", "r3", "r5"])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_config1_parity(rld, golden_cases, alg, dtype):
    c = golden_cases[f"config1_{alg}"]
    est = gpu_estimate(rld, c, dtype)
    assert rel(est.value, c["value"]) <= TOL[dtype]
    assert rel(est.logdet_P, c["logdet_P"]) <= TOL[dtype]
    np.testing.assert_allclose(est.per_probe_values, c["per_probe_values"], rtol=TOL[dtype] * 10,
                               atol=TOL[dtype] * abs(c["value"]) / 10)
    # Cholesky check (north_star): GPU and reference sit at the same distance from the exact value
    assert abs(abs(est.value - c["exact"]) - abs(c["value"] - c["exact"])) <= TOL[dtype] * abs(c["value"])


@pytest.mark.parametrize("source", ["numpy", "torch"])
def test_config1_dense_inputs(rld, golden_cases, source):
    c = golden_cases["config1_r3"]
    est = gpu_estimate(rld, c, "fp64", source=source)
    assert rel(est.value, c["value"]) <= 1e-6


@pytest.mark.parametrize("alg", ["r1", "r3", "r5"])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_config2_full_parity(rld, golden_cases, alg, dtype):
    c = golden_cases[f"config2_{alg}"]
    est = gpu_estimate(rld, c, dtype)
    assert rel(est.value, c["value"]) <= TOL[dtype]
    assert rel(est.logdet_P, c["logdet_P"]) <= TOL[dtype]


@pytest.mark.parametrize("name", ["config3_n4096_r3", "config4_n4096_r5", "config5_n4096_r3",
                                  "config2_n2048_r1", "config2_n2048_r3", "config2_n2048_r5"])
@pytest.mark.parametrize("dtype,path", [("fp64", "stored"), ("fp32", "stored"), ("fp32", "on_the_fly")])
def test_reduced_config_parity(rld, golden_cases, name, dtype, path):
    c = golden_cases[name]
    est = gpu_estimate(rld, c, dtype, path=path)
    assert rel(est.value, c["value"]) <= TOL[dtype]


def test_exact_logdet_matches_cholesky(rld, golden_cases):
    c = golden_cases["config2_r3"]
    wl = workload(c)
    est = rld.exact_logdet(rld.KernelMatrix(wl.spec, wl.points))
    assert rel(est.value, c["exact"]) <= 1e-10


def test_fixture_rows_ill_posed(rld, fixture_rows):
    """The reference's own fixture (RBF d=1, jitter 1e-6, cond ~ 2e8): a 1e-15 relative
    perturbation of K moves these estimates by 1e-5 .. 3e-4 (their `sensitivity`), so two
    correct float64 implementations differ at that level.  Pinned at 25x the row's own
    (single-sample) sensitivity, capped at 1e-3 (SURVEY: these rows pin results to ~1e-3); measured
    gaps 3e-6 .. 4.3e-4 with either float64 product, worst gap / sensitivity 10.4 on the int8
    slices and 6.0 on DMMA (scripts/tolerance_probe.py), both from the points (K built on the
    device from direct differences) and from the oracle's dense K (the reference's r^2 formula)."""
    from paper_2405_03474_b200.linalg import Rng

    for r in fixture_rows:
        pts = Rng(r["seed"]).child(0).normal((r["n"], r["d"]))
        cfg = rld.EstimatorConfig(r["algorithm"], r["s"], r["t"], "rademacher",
                                  rld.PreconditionerConfig("rand-svd", r["precond_rank"], r["precond_iters"],
                                                           max(r["jitter"], 1e-12)), r["seed"])
        tol = max(1e-6, min(1e-3, 25.0 * r["sensitivity"]))
        est = rld.rstar_logdet(rld.KernelMatrix(rld.KernelSpec("rbf", jitter=r["jitter"]), pts), cfg)
        assert rel(est.value, r["estimate"]) <= tol, (r, est.value)
        K = O.covariance_block("rbf", 1.0, 1.0, r["jitter"], pts)
        est = rld.rstar_logdet(K, cfg)
        assert rel(est.value, r["estimate"]) <= tol, (r, est.value)


# ---------------------------------------------------------------- known answers (pkg/tests/test_estimators.py)

def test_identity_matrix_is_exact_zero(rld):
    for alg in ("r1", "r3", "r5"):
        cfg = rld.EstimatorConfig(alg, precond=rld.PreconditionerConfig("identity"), seed=1)
        assert abs(rld.rstar_logdet(np.eye(100), cfg).value) <= 1e-10


@pytest.mark.parametrize("alg", ["r1", "r3", "r5"])
@pytest.mark.parametrize("cval", [0.5, 2.0, 5.0])
def test_scalar_matrix_reduces_to_scalar_rational(rld, alg, cval):
    from paper_2405_03474_b200.rational import eval_partial, partial_fraction

    n = 100
    cfg = rld.EstimatorConfig(alg, precond=rld.PreconditionerConfig("identity"), seed=2)
    est = rld.rstar_logdet(cval * np.eye(n), cfg)
    assert est.value == pytest.approx(n * eval_partial(partial_fraction(int(alg[1])), cval), rel=1e-9)


def test_value_decomposition_and_determinism(rld):
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(1)
    M = rld.KernelMatrix(wl.spec, wl.points)
    a = rld.rstar_logdet(M, wl.config)
    b = rld.rstar_logdet(M, wl.config)
    assert a.value == pytest.approx(a.logdet_P + a.trace_term, rel=1e-12)
    assert a.trace_term == pytest.approx(float(np.mean(a.per_probe_values)), rel=1e-12)
    assert a.value == b.value
    np.testing.assert_array_equal(a.per_probe_values, b.per_probe_values)


def test_diagonal_preconditioner_matches_oracle(rld):
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(1, n=512)
    K = O.covariance_block("matern52", 1.0, 0.2, 1e-2, wl.points)
    cfg = rld.EstimatorConfig("r3", 16, 20, precond=rld.PreconditionerConfig("diagonal"), seed=0)
    est = rld.rstar_logdet(K, cfg)
    # diagonal of a unit-amplitude kernel with jitter is a constant: log det P = n log(1.01)
    assert est.logdet_P == pytest.approx(512 * np.log(1.01), rel=1e-12)


def test_errors_map_to_reference_exceptions(rld):
    with pytest.raises(ValueError):
        rld.rstar_logdet(np.eye(5), rld.EstimatorConfig(precond=rld.PreconditionerConfig(rank=6)))
    with pytest.raises(ValueError):
        rld.rstar_logdet(np.eye(5), rld.EstimatorConfig(precond=rld.PreconditionerConfig(rank=0)))
    with pytest.raises(rld.NotPositiveDefinite):
        rld.exact_logdet(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(ValueError):
        rld.rstar_logdet(np.ones((3, 4)), rld.EstimatorConfig())


def test_injected_probes_and_sketch_equal_reference_streams(rld, golden_cases):
    """Passing the reference's own probe and sketch rows explicitly gives the same
    estimate as letting the device regenerate the streams (Rademacher probes and
    the ziggurat Gaussian sketch)."""
    from paper_2405_03474_b200.linalg import Rng

    c = golden_cases["config1_r3"]
    wl = workload(c)
    M = rld.KernelMatrix(wl.spec, wl.points)
    n, s, w = wl.n, wl.config.num_probes, wl.config.precond.rank + 10
    P = Rng(0).child(2).rademacher((s, n))
    om = [Rng(0).child(1).child(0).normal((w, n))]
    a = rld.rstar_logdet(M, wl.config)
    b = rld.rstar_logdet(M, wl.config, probes=P, omega=om)
    assert rel(a.value, b.value) <= 1e-13


# ---------------------------------------------------------------- full BASELINE sizes: properties

def _large_golden(name):
    from conftest import load_golden

    c = load_golden("golden_large.json").get(name)
    if c is None:
        pytest.skip(f"{name} not in golden_large.json")
    return c


def _large_workload(c):
    from paper_2405_03474_b200.workloads import baseline

    idx = int(c["workload"][-1])
    wl = baseline(idx, n=c["n"], rank=c["rank"], num_probes=c["num_probes"])
    cfg = replace(wl.config, algorithm=c["algorithm"], lanczos_iters=c["lanczos_iters"],
                  precond=replace(wl.config.precond, num_iters=c["num_iters"]))
    return replace(wl, config=cfg)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_config3_full_parity(rld, dtype):
    """BASELINE config 3 at full n = 65536 (stored K: 34 GB fp64 / 17 GB fp32) against the
    matrix-free float64 oracle (tests/golden/golden_large.json, screen 1.7e-15): the
    north_star bar, 1e-6 in fp64 and 1e-4 in fp32."""
    c = _large_golden("config3_full")
    wl = _large_workload(c)
    est = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(wl.config, dtype=dtype, path="stored"))
    assert rel(est.value, c["value"]) <= TOL[dtype], (est.value, c["value"])
    if dtype == "fp64":
        assert rel(est.logdet_P, c["logdet_P"]) <= 1e-9
        np.testing.assert_allclose(est.per_probe_values, c["per_probe_values"], rtol=1e-6,
                                   atol=1e-9 * abs(c["value"]))


def test_config4_full_parity(rld):
    """BASELINE config 4 at full n = 262144 (on the fly, r5, l = 1024, 64 probes) against the
    matrix-free float64 oracle: fp32 bar 1e-4."""
    c = _large_golden("config4_full")
    wl = _large_workload(c)
    est = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(wl.config, dtype="fp32", path="on_the_fly"))
    assert rel(est.value, c["value"]) <= TOL["fp32"], (est.value, c["value"])


def test_config5_full_n_parity(rld):
    """BASELINE config 5's kernel and points at full n = 2^20 (on the fly), reduced rank / probes /
    iterations (the oracle's note), against the matrix-free float64 oracle: fp32 bar 1e-4."""
    c = _large_golden("config5_full")
    wl = _large_workload(c)
    est = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(wl.config, dtype="fp32", path="on_the_fly"))
    assert rel(est.value, c["value"]) <= TOL["fp32"], (est.value, c["value"])


def test_config3_full_size_properties(rld):
    """n = 65536 fp32 stored K (16 GB): no CPU oracle can hold it, so check
    size-independent properties plus row-sampled K.V against float64."""
    import torch

    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(3)
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path="stored")
    a = R.estimate(wl.config)
    b = R.estimate(wl.config)
    assert np.isfinite(a.value) and a.value == b.value
    assert a.value == pytest.approx(a.logdet_P + a.trace_term, rel=1e-12)
    g = np.random.default_rng(0)
    V = g.standard_normal((4, wl.n))
    Y = R.kv_apply(torch.from_numpy(V).cuda()).cpu().numpy()
    rows = g.choice(wl.n, 32, replace=False)
    for i in rows:
        k = O.covariance_block("matern52", 1.0, 0.05, 1e-2, wl.points, rows=slice(i, i + 1))[0]
        ref = V @ k
        assert np.max(np.abs(Y[:, i] - ref) / (np.abs(V) @ np.abs(k))) <= 2e-6


def test_config3_on_the_fly_matches_stored(rld):
    """Full config 3 (n = 65536): the on-the-fly path (K tiles generated from float32 points on
    the tensor-core kernel) against the stored fp32 K -- two independent fp32 routes to the same
    float64 estimate; each is within ~1e-6 of it, so they must agree far inside the 1e-4 budget."""
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(3)
    M = rld.KernelMatrix(wl.spec, wl.points)
    a = rld.estimate_logdet(M, replace(wl.config, path="stored"))
    b = rld.estimate_logdet(M, replace(wl.config, path="on_the_fly"))
    assert rel(a.value, b.value) <= 1e-5, (a.value, b.value, a.logdet_P, b.logdet_P, a.trace_term, b.trace_term,
                                          a.attempts, b.attempts, a.rank_kept, b.rank_kept)
    assert rel(a.logdet_P, b.logdet_P) <= 1e-5


def _otf_rows_check(rld, index, m, nrows, seed):
    import torch

    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(index)
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path="on_the_fly")
    g = np.random.default_rng(seed)
    V = g.standard_normal((m, wl.n))
    Y = R.kv_apply(torch.from_numpy(V).cuda()).cpu().numpy()
    for i in g.choice(wl.n, nrows, replace=False):
        k = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points,
                               rows=slice(i, i + 1))[0]
        assert np.max(np.abs(Y[:, i] - V @ k) / (np.abs(V) @ np.abs(k))) <= 2e-6
    return R, wl


def test_config4_full_size_properties(rld):
    """Full config 4 (n = 262144, on the fly, r5, l = 1024, 64 probes): K cannot be stored,
    so check size-independent properties -- bit-identical repeat, value = log det P + trace
    term -- and row-sampled K.V against float64."""
    R, wl = _otf_rows_check(rld, 4, 3, 16, 1)
    a = R.estimate(wl.config)
    b = R.estimate(wl.config)
    assert np.isfinite(a.value) and a.value == b.value
    assert a.value == pytest.approx(a.logdet_P + a.trace_term, rel=1e-12)
    assert a.kv_products == 26


def test_config5_full_size_products(rld):
    """Full config 5 (n = 2^20, Matern-5/2 on the fly): row-sampled K.V against float64."""
    _otf_rows_check(rld, 5, 2, 12, 2)


# ---------------------------------------------------------------- SLQ

def _slq_cases():
    from conftest import load_golden

    return load_golden("golden_slq.json")


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("case", _slq_cases(), ids=lambda c: c["name"])
def test_slq_matches_reference(rld, case, dtype):
    """slq_logdet (src/estimators.py:99-122) on the device: Lanczos on K with full
    reorthogonalisation, Gauss quadrature of log per probe, against the unmodified
    reference's outputs (tests/golden/make_golden_slq.py)."""
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(case["config_index"], n=case["n"], num_probes=case["num_probes"])
    cfg = replace(wl.config, algorithm="slq", dtype=dtype)
    est = rld.estimate_logdet(rld.KernelMatrix(wl.spec, wl.points), cfg)
    assert est.logdet_P == 0.0 and est.value == est.trace_term
    assert rel(est.value, case["value"]) <= TOL[dtype], (est.value, case["value"])
    if dtype == "fp64":
        np.testing.assert_allclose(est.per_probe_values, case["per_probe"], rtol=1e-6)
        assert est.clamped_eigs == case["clamped_eigs"]


def test_slq_dense_input_deterministic(rld):
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(1, n=1024, num_probes=8)
    K = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points)
    cfg = replace(wl.config, algorithm="slq")
    a = rld.slq_logdet(K, cfg)
    b = rld.slq_logdet(K, cfg)
    assert a.value == b.value
    ref = O.slq_dense(K, s=8, t=20, probe_kind="rademacher", seed=0)
    assert rel(a.value, ref.value) <= 1e-9


def test_slq_on_the_fly_fp32(rld):
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(5, n=4096)
    ref = [c for c in _slq_cases() if c["name"] == "slq_config5_n4096"][0]
    cfg = replace(wl.config, algorithm="slq", dtype="fp32", path="on_the_fly")
    est = rld.estimate_logdet(rld.KernelMatrix(wl.spec, wl.points), cfg)
    assert rel(est.value, ref["value"]) <= TOL["fp32"]


def test_slq_t_equals_n_is_exact(rld):
    """t = n: the Gauss quadrature is exact, so SLQ returns mean |z|^2 e1^T log(K) e1
    -- checked against the oracle at n = 20 (src/lanczos.py full-space reconstruction)."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((20, 20))
    K = A @ A.T + 20 * np.eye(20)
    cfg = rld.EstimatorConfig("slq", 4, 20)
    est = rld.slq_logdet(K, cfg)
    ref = O.slq_dense(K, s=4, t=20, seed=0)
    assert rel(est.value, ref.value) <= 1e-10


# ---------------------------------------------------------------- preconditioner kinds

def _precond_cases():
    from conftest import load_golden

    return load_golden("golden_precond.json")


def load_precond_wellposed():
    from conftest import load_golden

    return load_golden("golden_precond_wellposed.json")


@pytest.mark.parametrize("case", [c for c in _precond_cases() if not c["kind"].startswith("partial-cholesky")],
                         ids=lambda c: c["name"])
def test_precond_kinds_match_reference(rld, case):
    """Seven kinds of src/precond.py:236-267 on the device (dense float64 K, the reference's own
    input) against the unmodified reference at the fp64 bar.  The partial-Cholesky kinds of this
    file start from an n-way pivot tie (the kernel's constant diagonal: screen 4e-3 .. 1e-2) and are
    replaced by the well-posed cases below."""
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(case["config_index"], n=case["n"])
    K = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points)
    cfg = rld.EstimatorConfig("r3", case["num_probes"], 20, "rademacher",
                              rld.PreconditionerConfig(case["kind"], case["rank"], case["num_iters"], case["scale"]),
                              case["seed"], dtype="fp64")
    est = rld.rstar_logdet(K, cfg)
    assert case["screen"] < 1e-12
    assert rel(est.value, case["value"]) <= TOL["fp64"], (est.value, case["value"])
    assert rel(est.logdet_P + 1.0, case["logdet_P"] + 1.0) <= 1e-8


def wellposed_pchol_matrix(case):
    """K + diag(distinct offsets) of tests/golden/make_golden_precond.py wellposed_cases()."""
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(case["config_index"], n=case["n"])
    K = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points)
    off = np.random.default_rng(case["diag_offsets_seed"]).uniform(0.0, case["diag_offsets_max"], case["n"])
    return K + np.diag(off)


@pytest.mark.parametrize("case", load_precond_wellposed(), ids=lambda c: c["name"])
def test_partial_cholesky_wellposed_match_reference(rld, case):
    """Greedy pivoted partial Cholesky (src/precond.py:215-228, 253-259) on K + diag(distinct
    offsets): no pivot ties, screen <= 2e-11.  The "-scaled" kind (base = scale) is pinned at
    1e-12.  The plain kind floors the residual diagonal of its k pivot rows at 1e-12
    (src/precond.py:231-233), so C = A^T diag(base)^-1 A has eigenvalues from ~1 to ~1e12 and the
    1e-14 keep filter and the small eigenvalues of src/precond.py:96-99 are only known to an
    absolute eps * 1e12: any backward-stable eigensolver other than the reference's own LAPACK
    call lands ~1e-5 away (measured 1.6e-5 / 5.8e-6, scripts/tolerance_probe.py), so that kind is
    pinned at 1e-4."""
    K = wellposed_pchol_matrix(case)
    cfg = rld.EstimatorConfig("r3", case["num_probes"], 20, "rademacher",
                              rld.PreconditionerConfig(case["kind"], case["rank"], case["num_iters"], case["scale"]),
                              case["seed"], dtype="fp64")
    est = rld.rstar_logdet(K, cfg)
    tol = 1e-12 if case["kind"].endswith("-scaled") else 1e-4
    assert rel(est.value, case["value"]) <= tol, (est.value, case["value"])


@pytest.mark.parametrize("kind", ["rand-svd-scaled", "trunc-svd", "trunc-svd-scaled", "rank-one", "diagonal"])
def test_precond_kinds_fp32_points(rld, kind):
    """The same kinds from the points with K stored in float32 (tiled) on the device."""
    from paper_2405_03474_b200.workloads import baseline

    case = [c for c in _precond_cases() if c["kind"] == kind and c["config_index"] == 1][0]
    wl = baseline(1, n=case["n"])
    cfg = rld.EstimatorConfig("r3", case["num_probes"], 20, "rademacher",
                              rld.PreconditionerConfig(kind, case["rank"], case["num_iters"], case["scale"]),
                              case["seed"], dtype="fp32", path="stored")
    est = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), cfg)
    assert rel(est.value, case["value"]) <= TOL["fp32"]


@pytest.mark.parametrize("kind", ["trunc-svd", "partial-cholesky"])
@pytest.mark.parametrize("path", ["stored", "on_the_fly"])
def test_perfect_preconditioner_kills_stochastic_part(rld, kind, path):
    """test_estimators.py:45-56: a rank-n preconditioner reproduces K, so the trace term
    vanishes and the estimate is the Cholesky log det."""
    rng = np.random.default_rng(4)
    pts = rng.standard_normal((60, 2))
    spec = rld.KernelSpec("rbf", jitter=1e-3)
    cfg = rld.EstimatorConfig("r3", 35, 20, "rademacher", rld.PreconditionerConfig(kind, 60), 4)
    if kind == "trunc-svd" and path == "on_the_fly":
        path = "stored"
    est = rld.rstar_logdet(rld.KernelMatrix(spec, pts), replace(cfg, path=path))
    K = O.covariance_block("rbf", 1.0, 1.0, 1e-3, pts)
    assert abs(est.trace_term) <= 1e-8 * max(abs(est.logdet_P), 1.0)
    assert rel(est.value, O.cholesky_logdet(K)) <= 1e-8


def test_partial_cholesky_on_the_fly_matches_stored(rld, monkeypatch):
    """The pivoted partial Cholesky reads K columns from the stored K or generates them
    from the points: same pivots, same preconditioner.  With the stored product on the DMMA
    kernel (float64 GEMM) and the on-the-fly one on the DFMA kernel: 1e-9 (measured: identical).
    With the default INT8-slice product the floored base (1e-12 on the 64 pivot rows) amplifies its
    sigma-scaled rounding (~2^-52 n max|K| max|V| per entry) ~1e12-fold through N^-1 K N^-T:
    8.4e-7 (5.6e-8 with the earlier 8 x 7-bit digits: one draw each of the same error level), held
    to the fp64 bar."""
    from paper_2405_03474_b200.workloads import baseline

    monkeypatch.setenv("RLD_FP64_PRODUCT", "dmma")
    wl = baseline(5, n=2048)
    cfg = replace(wl.config, dtype="fp64", num_probes=8,
                  precond=rld.PreconditionerConfig("partial-cholesky", 64, 5))
    a = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(cfg, path="stored"))
    b = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(cfg, path="on_the_fly"))
    assert rel(a.logdet_P, b.logdet_P) <= 1e-9
    assert rel(a.value, b.value) <= 1e-9
    monkeypatch.setenv("RLD_FP64_PRODUCT", "ozaki")
    c = rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), replace(cfg, path="stored"))
    assert rel(c.logdet_P, b.logdet_P) <= 1e-9
    assert rel(c.value, b.value) <= TOL["fp64"]


# ---------------------------------------------------------------- normal-orthogonal probes

def _probe_cases():
    from conftest import load_golden

    return load_golden("golden_probes.json")["estimates"]


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("case", _probe_cases(), ids=lambda c: c["name"])
def test_normal_orthogonal_probes_match_reference(rld, case, dtype):
    """Device Gaussian blocks (stream (seed, (2, i))), device orthonormalisation, chi radii
    continuing the same stream on the host (rld_chi_radii) -- src/probes.py:15-44."""
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(case["config_index"], n=case["n"])
    cfg = rld.EstimatorConfig(case["algorithm"], case["num_probes"], 20, "normal-orthogonal",
                              rld.PreconditionerConfig("rand-svd", case["rank"], 5), case["seed"], dtype=dtype)
    est = rld.estimate_logdet(rld.KernelMatrix(wl.spec, wl.points), cfg)
    assert rel(est.value, case["value"]) <= TOL[dtype], (est.value, case["value"])
    if dtype == "fp64":
        np.testing.assert_allclose(est.per_probe_values, case["per_probe"], rtol=1e-6)


def test_normal_orthogonal_several_blocks(rld):
    """s > n: independent blocks from streams (seed, (2, 0)), (seed, (2, 1)), ... (src/probes.py:38-44)."""
    rng = np.random.default_rng(5)
    pts = rng.uniform(0, 1, (20, 2))
    K = O.covariance_block("matern52", 1.0, 0.3, 1e-2, pts)
    cfg = rld.EstimatorConfig("r3", 50, 20, "normal-orthogonal", rld.PreconditionerConfig("identity"), 3)
    est = rld.rstar_logdet(K, cfg)
    ref = O.rstar_dense(K, order=3, s=50, t=20, probe_kind="normal-orthogonal", k=0, q=5, seed=3, precond="identity")
    assert rel(est.value, ref.value) <= 1e-9


# ---------------------------------------------------------------- dense Cholesky of the preconditioner build

def _dense_cholesky(G):
    import ctypes as C
    import torch

    from paper_2405_03474_b200._session import session

    s = session()
    t = torch.from_numpy(np.ascontiguousarray(G)).cuda()
    info = C.c_int32(-7)
    s.handle.check(s.lib.rld_dense_cholesky(s.handle.ptr, G.shape[0], t.data_ptr(), C.byref(info)), "dense_cholesky")
    return np.tril(t.cpu().numpy()), info.value   # device column-major upper R = tril of the row-major view


@pytest.mark.parametrize("n", [1, 5, 31, 32, 33, 64, 100, 255, 266, 522, 640, 700, 1024, 1034, 2058])
@pytest.mark.parametrize("spectrum", ["wishart", "decaying"])
def test_dense_cholesky_matches_lapack(rld, n, spectrum):
    """One-cluster Cholesky (n <= 640) / its 2 x 2 block recursion on the DMMA kernels (above) vs
    LAPACK: the Gram factor of CholQR and the inner factor of src/precond.py:75-80."""
    g = np.random.default_rng(n)
    if spectrum == "wishart":
        X = g.standard_normal((n + 8, n))
        G = X.T @ X
    else:
        Q, _ = np.linalg.qr(g.standard_normal((n, n)))
        G = (Q * np.logspace(6, -3, n)) @ Q.T
        G = (G + G.T) / 2 + 1e-3 * np.eye(n)
    L, info = _dense_cholesky(G)
    assert info == 0
    Lref = np.linalg.cholesky(G)
    assert np.linalg.norm(L @ L.T - G) <= 1e-14 * np.linalg.norm(G) * max(1, n / 64)
    assert np.linalg.norm(L - Lref) <= 1e-10 * np.linalg.norm(Lref)


@pytest.mark.parametrize("n,bad", [(1, 0), (40, 0), (40, 5), (266, 37), (266, 265), (522, 300), (700, 650),
                                   (700, 100), (1034, 900), (2058, 1500), (2058, 3)])
def test_dense_cholesky_reports_first_bad_pivot(rld, n, bad):
    """info = 1-based index of the first non-positive pivot (LAPACK potrf), which the CholQR weak
    test and the NotPositiveDefinite check read."""
    g = np.random.default_rng(1)
    X = g.standard_normal((n + 8, n))
    G = X.T @ X
    G[bad, bad] = -1.0
    _, info = _dense_cholesky(G)
    assert info == bad + 1


def test_fresh_workspace_poisoned_with_nan_changes_nothing(rld):
    """Every device workspace is written before it is read: with RLD_POISON=1 each new buffer is
    filled with NaN bytes (a fresh process, since the flag is read once) and the estimates of
    configs 1-3 (stored, on the fly, CTA pairs, several preconditioners, normal-orthogonal probes)
    must equal the ones computed here without it."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = r"""
import json, sys
sys.path.insert(0, %r)
import paper_2405_03474_b200 as rld
from paper_2405_03474_b200.workloads import baseline
from dataclasses import replace
out = []
for idx, n, path, kind, probe in [(1, 1024, "stored", "rand-svd", "rademacher"), (2, 4096, "stored", "rand-svd", "rademacher"),
                                  (3, 4096, "on_the_fly", "rand-svd", "gaussian"), (2, 2048, "stored", "partial-cholesky", "normal-orthogonal")]:
    wl = baseline(idx, n=n)
    cfg = replace(wl.config, probe_kind=probe, precond=replace(wl.config.precond, kind=kind), path=path)
    out.append(rld.estimate_logdet(rld.KernelMatrix(wl.spec, wl.points), cfg).value)
print(json.dumps(out))
""" % str(Path(__file__).resolve().parent.parent)
    runs = []
    for poison in ("1", "0"):
        env = dict(os.environ, RLD_POISON=poison)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        runs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert runs[0] == runs[1], runs
    assert all(np.isfinite(v) for v in runs[0])


def _dense_eigh(A):
    import ctypes as C  # noqa: F401
    import torch

    from paper_2405_03474_b200._session import session

    s = session()
    t = torch.from_numpy(np.ascontiguousarray(A)).cuda()   # symmetric: row-major == column-major
    w = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
    s.handle.check(s.lib.rld_dense_eigh(s.handle.ptr, A.shape[0], t.data_ptr(), w.data_ptr()), "dense_eigh")
    return w.cpu().numpy(), t.cpu().numpy().T   # column j of the column-major result <-> w[j]


@pytest.mark.parametrize("n", [2, 3, 10, 64, 74, 256, 266, 288, 300, 512, 522, 544, 560])
@pytest.mark.parametrize("spectrum", ["wishart", "decaying", "degenerate", "rank_deficient", "indefinite",
                                      "clustered", "diagonal"])
def test_dense_eigh_matches_lapack(rld, n, spectrum):
    """The preconditioner's symmetric eigensolver (tri_eig.cu for 3 <= n <= 544, DSYEVD otherwise
    and as the fallback on degenerate unreduced blocks) against LAPACK eigh: eigenvalues,
    reconstruction, orthogonality, and the top-half spectral projector (eigenvectors are defined
    up to sign / rotation inside degenerate eigenspaces)."""
    g = np.random.default_rng(n + len(spectrum))
    Q, _ = np.linalg.qr(g.standard_normal((n, n)))
    if spectrum == "wishart":
        X = g.standard_normal((n + 5, n))
        A = X.T @ X
    elif spectrum == "diagonal":   # already tridiagonal and fully split: one-row blocks
        A = np.diag(g.permutation(np.repeat(np.arange(1.0, 1 + -(-n // 2)), 2)[:n]))
    else:
        if spectrum == "decaying":
            lam = np.logspace(7, -3, n)
        elif spectrum == "degenerate":
            lam = np.repeat([5.0, 2.0, 2.0, 0.5], -(-n // 4))[:n]
        elif spectrum == "indefinite":
            lam = np.linspace(-3.0, 2.0, n) ** 3
        elif spectrum == "clustered":   # pairs 1e-9 apart (relative): close but not degenerate
            base = np.repeat(np.logspace(2, -1, -(-n // 2)), 2)[:n]
            lam = base * (1 + 1e-9 * (np.arange(n) % 2))
        else:
            lam = np.concatenate([np.logspace(3, 0, n - n // 3), np.zeros(n // 3)])
        A = (Q * lam) @ Q.T
        A = (A + A.T) / 2
    w, V = _dense_eigh(A)
    wr, Vr = np.linalg.eigh(A)
    scale = max(1.0, np.max(np.abs(wr)))
    assert np.all(np.diff(w) >= -1e-12 * scale)
    np.testing.assert_allclose(w, wr, rtol=0, atol=1e-11 * scale)
    assert np.linalg.norm(V.T @ V - np.eye(n)) <= 1e-11 * np.sqrt(n)
    assert np.linalg.norm((V * w) @ V.T - A) <= 1e-11 * np.linalg.norm(A)
    h = n // 2
    if wr[h] - wr[h - 1] > 1e-6 * scale:   # a gap: the top-half invariant subspace is well defined
        Pg, Pr = V[:, h:] @ V[:, h:].T, Vr[:, h:] @ Vr[:, h:].T
        assert np.linalg.norm(Pg - Pr) <= 1e-9


def test_tri_eigh_fallback_and_dsyevd_path(rld):
    """tri_eig.cu hands degenerate unreduced blocks to DSYEVD (reported with RLD_TRI_EIG_DEBUG=1)
    and keeps a well-separated spectrum; RLD_TRI_EIG=0 (DSYEVD always) agrees to rounding.  Flags
    are read once per process: subprocesses."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = r"""
import sys
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import numpy as np
from test_gpu_parity import _dense_eigh
out = []
for n, lam in [(266, np.logspace(4, -2, 266)), (64, np.repeat([5.0, 2.0, 2.0, 0.5], 16))]:
    g = np.random.default_rng(n)
    Q, _ = np.linalg.qr(g.standard_normal((n, n)))
    A = (Q * lam) @ Q.T
    A = (A + A.T) / 2
    w, V = _dense_eigh(A)
    out.append(np.linalg.norm((V * w) @ V.T - A) / np.linalg.norm(A))
    out.append(float(w.sum()))
print("res", *out)
""" % (str(Path(__file__).resolve().parent.parent), str(Path(__file__).resolve().parent))
    runs = {}
    for flag in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, RLD_TRI_EIG=flag, RLD_TRI_EIG_DEBUG="1"),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        runs[flag] = (r.stdout, r.stderr)
    fallbacks = [ln for ln in runs["1"][1].splitlines() if "tri_eigh fallback" in ln]
    assert len(fallbacks) == 1 and "k = 64" in fallbacks[0], runs["1"][1][-2000:]
    assert not [ln for ln in runs["0"][1].splitlines() if "tri_eigh fallback" in ln]
    a = [float(x) for x in runs["1"][0].split("res")[1].split()]
    b = [float(x) for x in runs["0"][0].split("res")[1].split()]
    assert a[0] < 1e-13 and b[0] < 1e-13 and a[2] < 1e-13
    np.testing.assert_allclose(a[1], b[1], rtol=1e-12)
    np.testing.assert_allclose(a[3], b[3], rtol=1e-12)


def test_alternative_paths_agree(rld):
    """The alternative one-GPU paths (RLD_CHOLQR_GEMM=0: DTRSM CholQR; RLD_TC_CG2=0: single-CTA
    products; RLD_TRI_EIG=0: cuSOLVER DSYEVD instead of tri_eig.cu) give the default estimate to
    fp32 accuracy (flags are read once: subprocesses)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = r"""
import json, sys
sys.path.insert(0, %r)
import paper_2405_03474_b200 as rld
from paper_2405_03474_b200.workloads import baseline
out = []
for idx, n in [(1, 1024), (2, 4096)]:
    wl = baseline(idx, n=n)
    out.append(rld.estimate_logdet(rld.KernelMatrix(wl.spec, wl.points), wl.config).value)
print(json.dumps(out))
""" % str(Path(__file__).resolve().parent.parent)
    runs = {}
    for name, env in [("default", {}), ("trsm", {"RLD_CHOLQR_GEMM": "0"}),
                      ("single_cta", {"RLD_TC_CG2": "0"}), ("dsyevd", {"RLD_TRI_EIG": "0"})]:
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        runs[name] = json.loads(r.stdout.strip().splitlines()[-1])
    for name, vals in runs.items():
        for v, d, tol in zip(vals, runs["default"], (1e-9, 1e-5)):   # config 1 runs in fp64, config 2 in fp32
            assert rel(v, d) <= tol, (name, v, d)
