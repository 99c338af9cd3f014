"""The on-the-fly float32 product on the kind::f16 tensor cores (csrc/kv_otf.cu): every
instantiated shape (vectors per pass NT = 32 / 64 / 128, point dimension 1-4, both kernel
families) against float64, edge cases of the power-of-two scaling, determinism, and
agreement with the 3xTF32 kernel (RLD_OTF_KIND=tf32) at the estimate level.

Bound: |Y - V K| <= 2e-6 (|V| |K|) entrywise, the float32 budget the 3xTF32 kernel is held
to (head / tail fp16 split: 2^-22 relative per factor, fp32 accumulation with
round-to-nearest group flushes)."""

from dataclasses import replace

import numpy as np
import pytest

from conftest import rel
from oracle import rstar_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rld():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03474_b200 as rld

    return rld


@pytest.fixture(autouse=True)
def _no_slice_cache(monkeypatch):
    """These tests are about the on-the-fly kernel: keep d <= 3 problems from being served from the
    cached sparse int8-slice image (rld_api.cu prepare; tests/test_gpu_streams_dmma.py covers that)."""
    monkeypatch.setenv("RLD_OTF_CACHE", "0")


def _product(rld, spec, pts, V, kind=None, monkeypatch=None):
    import torch

    if kind is not None:
        monkeypatch.setenv("RLD_OTF_KIND", kind)
    R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path="on_the_fly")
    return R.kv_apply(torch.from_numpy(np.ascontiguousarray(V)).cuda()).cpu().numpy()


def _err(spec, pts, V, Y):
    K = O.covariance_block(spec.family, spec.amplitude, spec.length_scale, spec.jitter, pts)
    scale = np.abs(V) @ np.abs(K)
    return float(np.max(np.abs(Y - V @ K) / np.where(scale > 0, scale, 1.0)))


@pytest.mark.parametrize("family", ["matern52", "rbf"])
@pytest.mark.parametrize("d", [1, 2, 3, 4])
@pytest.mark.parametrize("n,m", [(1000, 1), (1017, 16), (777, 37), (4099, 64), (3001, 130), (2500, 300)])
def test_otf16_product_matches_float64(rld, family, d, n, m):
    g = np.random.default_rng(n + m + d)
    pts = g.uniform(0, 1, (n, d))
    spec = rld.KernelSpec(family, 1.3, 0.2, 1e-2)
    # vectors scaled over 2^+-29: the per-vector power-of-two scale must absorb it exactly
    V = g.standard_normal((m, n)) * np.exp(g.uniform(-20, 20, (m, 1)))
    assert _err(spec, pts, V, _product(rld, spec, pts, V)) <= 2e-6


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 129])
def test_otf16_tiny_and_ragged_n(rld, n):
    g = np.random.default_rng(n)
    pts = g.uniform(0, 1, (n, 3))
    spec = rld.KernelSpec("matern52", 1.0, 0.3, 1e-1)
    V = g.standard_normal((5, n))
    assert _err(spec, pts, V, _product(rld, spec, pts, V)) <= 2e-6


def test_otf16_zero_tiny_and_huge_vectors(rld):
    """Zero vectors (scale exponent 0), entries near the float64 subnormal range and near
    1e300, mixed in one block; large amplitude (diagonal far from 1)."""
    g = np.random.default_rng(7)
    n = 3000
    pts = g.uniform(0, 1, (n, 2))
    spec = rld.KernelSpec("rbf", 37.0, 0.1, 5.0)
    V = g.standard_normal((6, n))
    V[0] = 0.0
    V[1] *= 1e-300
    V[2] *= 1e300
    V[3, ::2] = 0.0
    V[4] = 0.0
    V[4, 17] = 1.0        # one-hot: the product returns column 17 of K
    Y = _product(rld, spec, pts, V)
    assert np.all(Y[0] == 0.0)
    K17 = O.covariance_block(spec.family, spec.amplitude, spec.length_scale, spec.jitter, pts, rows=slice(17, 18))[0]
    np.testing.assert_allclose(Y[4], K17, rtol=2e-6, atol=2e-6 * spec.amplitude ** 2)
    for r in (1, 2, 3, 5):
        assert _err(spec, pts, V[r:r + 1], Y[r:r + 1]) <= 2e-6


def test_otf16_deterministic_and_wide(rld):
    """Bit-identical repeats (fixed-order split-k reduction) at a multi-pass width."""
    import torch

    g = np.random.default_rng(11)
    n = 20000
    pts = g.uniform(0, 1, (n, 3))
    spec = rld.KernelSpec("matern52", 1.0, 0.05, 1e-2)
    R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path="on_the_fly")
    V = torch.from_numpy(g.standard_normal((266, n))).cuda()
    a = R.kv_apply(V).cpu().numpy()
    b = R.kv_apply(V).cpu().numpy()
    assert np.array_equal(a, b)
    Vh = V.cpu().numpy()
    for i in g.choice(n, 8, replace=False):
        k = O.covariance_block("matern52", 1.0, 0.05, 1e-2, pts, rows=slice(i, i + 1))[0]
        assert np.max(np.abs(a[:, i] - Vh @ k) / (np.abs(Vh) @ np.abs(k))) <= 2e-6


@pytest.mark.parametrize("index", [4, 5])
def test_otf16_estimate_agrees_with_3xtf32(rld, index, monkeypatch):
    """Reduced BASELINE configs 4 / 5: the fp16 and 3xTF32 on-the-fly kernels are two
    independent float32 routes to the float64 estimate; each is ~1e-6 from it."""
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(index, n=8192, rank=128, num_probes=16)
    cfg = replace(wl.config, dtype="fp32", path="on_the_fly")
    M = rld.KernelMatrix(wl.spec, wl.points)
    monkeypatch.setenv("RLD_OTF_KIND", "f16")
    a = rld.rstar_logdet(M, cfg)
    monkeypatch.setenv("RLD_OTF_KIND", "tf32")
    b = rld.rstar_logdet(M, cfg)
    assert rel(a.value, b.value) <= 1e-5, (a.value, b.value)
    K = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points)
    ref = O.rstar_dense(K, order=int(cfg.algorithm[1]), s=cfg.num_probes, t=cfg.lanczos_iters,
                        probe_kind=cfg.probe_kind, k=cfg.precond.rank, q=cfg.precond.num_iters,
                        seed=cfg.seed)
    assert rel(a.value, ref.value) <= 1e-4, (a.value, ref.value)


@pytest.mark.parametrize("n,m", [(4099, 70), (16384, 266), (19968, 128), (24960, 300), (39936, 522)])
def test_stored_f16_wide_product(rld, n, m):
    """Wide products (m > 64) of a stored fp32 K run on the same fp16 head / tail kernel with the K
    tiles streamed from HBM and per-row power-of-two scales.  The shapes include whole-wave rounds
    plus stream-K tails; (19968, 128) and (39936, 522) hung before the A-ring depth was made a
    multiple of the converter warps (a ring slot shared by two warps).  Sampled rows against the
    float64 product with the stored (float32-rounded) K."""
    import torch

    g = np.random.default_rng(n + m)
    pts = g.standard_normal((n, 4))
    spec = rld.KernelSpec("rbf", 1.0, 1.5, 1e-3)
    R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path="stored")
    V = g.standard_normal((m, n)) * np.exp(g.uniform(-10, 10, (m, 1)))
    Y = R.kv_apply(torch.from_numpy(V).cuda()).cpu().numpy()
    for i in g.choice(n, 12, replace=False):
        k = O.covariance_block("rbf", 1.0, 1.5, 1e-3, pts, rows=slice(i, i + 1))[0].astype(np.float32).astype(np.float64)
        assert np.max(np.abs(Y[:, i] - V @ k) / (np.abs(V) @ np.abs(k))) <= 2e-6


@pytest.mark.parametrize("family,ell", [("matern52", 0.02), ("rbf", 0.03)])
def test_otf16_far_field_skip(rld, monkeypatch, family, ell):
    """On the fly with d <= 3 points at a short length scale: the points go into Morton order and
    (tile, k-step) pairs whose fp16 operands are exactly zero are skipped (no loads, no MMAs), with
    a register flush every k-step.  Against float64 on sampled rows (the 2e-6 bound) and against the
    unsorted product."""
    import torch

    g = np.random.default_rng(17)
    n = 40000
    pts = g.uniform(0, 1, (n, 3))
    spec = rld.KernelSpec(family, 1.0, ell, 1e-1)
    V = g.standard_normal((64, n))
    Vt = torch.from_numpy(V).cuda()
    out = {}
    for sort in ("1", "0"):
        monkeypatch.setenv("RLD_SORT", sort)
        R = rld.ResidentMatrix(rld.KernelMatrix(spec, pts), dtype="fp32", path="on_the_fly")
        out[sort] = R.kv_apply(Vt).cpu().numpy()
    for i in g.choice(n, 10, replace=False):
        k = O.covariance_block(family, 1.0, ell, 1e-1, pts, rows=slice(i, i + 1))[0]
        sc = np.abs(V) @ np.abs(k)
        assert np.max(np.abs(out["1"][:, i] - V @ k) / sc) <= 2e-6
        assert np.max(np.abs(out["1"][:, i] - out["0"][:, i]) / sc) <= 2e-6
