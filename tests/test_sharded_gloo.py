"""World-size 2 / 3 CPU tests (gloo) of the row-sharded decomposition the
multi-GPU path uses: shard bounds, NCCL-id bootstrap, and a
numpy mirror of rld_api.cu's sharded dataflow (tests/sharded_mirror.py) whose
estimate must equal the single-rank one and the oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import rstar_oracle as O
from paper_2405_03474_b200.parallel import shard_bounds

N, D, K_RANK, Q, S, T, SEED, ORDER = 97, 3, 8, 3, 5, 10, 7, 3


def _problem():
    X = np.random.default_rng(11).uniform(size=(N, D))
    K = O.covariance_block("matern52", 1.0, 0.3, 1e-2, X)
    V = O.probes("rademacher", S, N, SEED)
    w = min(K_RANK + O.OVERSAMPLE, N)
    omega = O.sketch(SEED, 0, w, N)
    return K, V, omega


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_03474_b200.parallel import broadcast_nccl_id
        from sharded_mirror import Comm, sharded_rstar

        nid = broadcast_nccl_id()
        K, V, omega = _problem()
        r0, r1 = shard_bounds(N, world, rank)
        val, ldp, tr, per = sharded_rstar(K, r0, r1, Comm(world, rank), ORDER, V, omega, K_RANK, Q, T)
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.concatenate([[val, ldp, tr], per]))
        with open(os.path.join(outdir, f"id{rank}.bin"), "wb") as f:
            f.write(nid)
    finally:
        dist.destroy_process_group()


def _run(world, tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"r{r}.npy") for r in range(world)]
    ids = [(tmp_path / f"id{r}.bin").read_bytes() for r in range(world)]
    return outs, ids


def test_shard_bounds_cover_rows():
    for n in (1, 7, 97, 16384, 65537):
        for g in (1, 2, 3, 8):
            spans = [shard_bounds(n, g, r) for r in range(g)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            L = -(-n // g)
            assert all(r1 - r0 <= L for r0, r1 in spans)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_mirror_single_rank_matches_oracle():
    from sharded_mirror import Comm, sharded_rstar

    K, V, omega = _problem()
    val, ldp, tr, per = sharded_rstar(K, 0, N, Comm(1, 0), ORDER, V, omega, K_RANK, Q, T)
    ref = O.rstar_dense(K, order=ORDER, s=S, t=T, k=K_RANK, q=Q, seed=SEED, V=V, omega=[omega, omega])
    assert abs(ldp - ref.logdet_P) <= 1e-10 * abs(ref.logdet_P)
    assert abs(val - ref.value) <= 1e-9 * abs(ref.value)
    np.testing.assert_allclose(per, ref.per_probe_values, rtol=1e-8)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gloo_matches_single_rank(world, tmp_path):
    from sharded_mirror import Comm, sharded_rstar

    K, V, omega = _problem()
    one = sharded_rstar(K, 0, N, Comm(1, 0), ORDER, V, omega, K_RANK, Q, T)
    outs, ids = _run(world, tmp_path)
    for o in outs:                       # every rank ends with the same replicated result
        np.testing.assert_array_equal(o, outs[0])
    assert abs(outs[0][0] - one[0]) <= 1e-12 * abs(one[0])
    np.testing.assert_allclose(outs[0][3:], one[3], rtol=1e-10)
    assert len(set(ids)) == 1 and len(ids[0]) == 128   # NCCL unique id reached every rank
