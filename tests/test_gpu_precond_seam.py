"""GPU: the stand-alone preconditioner seam (rld_precond_build /
rld_precond_apply) against the unmodified reference's ``build_preconditioner`` and its
``solve_sqrt`` / ``solve_sqrt_t`` (src/precond.py:102-115, 236-267), golden vectors from
tests/golden/make_golden_preconditioner_apply.py."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import rstar_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rld():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03474_b200 as rld

    return rld


@pytest.mark.parametrize("case", load_golden("golden_preconditioner_apply.json"), ids=lambda c: c["name"])
def test_build_and_apply_match_reference(rld, case):
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(case["config_index"], n=case["n"])
    K = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points)
    cfg = rld.PreconditionerConfig(case["kind"], case["rank"], case["num_iters"], case["scale"])
    P = rld.build_preconditioner(K, cfg, rld.Rng(case["seed"]).child(1))
    assert rel(P.log_det, case["log_det"]) <= 1e-9, (P.log_det, case["log_det"])
    Z = np.random.default_rng(case["z_seed"]).standard_normal((case["n"], 3))
    for name, fn in (("solve_sqrt", P.solve_sqrt), ("solve_sqrt_t", P.solve_sqrt_t)):
        ref = np.array(case[name]).T
        got = fn(Z)
        assert np.max(np.abs(got - ref)) <= 1e-9 * np.max(np.abs(ref)), name
        got1 = fn(Z[:, 0])                       # a single vector, as the reference's op takes it
        assert np.max(np.abs(got1 - ref[:, 0])) <= 1e-9 * np.max(np.abs(ref))
    # P^-1 = N^-T N^-1
    np.testing.assert_allclose(P.solve(Z), P.solve_sqrt_t(P.solve_sqrt(Z)), rtol=0,
                               atol=1e-11 * np.max(np.abs(P.solve(Z))))


def test_precond_build_matches_estimate_logdet(rld):
    """The seam builds the same P as the estimate: log det P equal to the estimate's logdet_P."""
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(1)
    M = rld.KernelMatrix(wl.spec, wl.points)
    est = rld.rstar_logdet(M, wl.config)
    P = rld.build_preconditioner(M, wl.config.precond, rld.Rng(wl.config.seed).child(1))
    assert rel(P.log_det, est.logdet_P) <= 1e-12
    assert P.rank_kept == est.rank_kept
