"""The five BASELINE.json configurations as (KernelSpec, points, EstimatorConfig).

Point sets come from one seeded tree that mirrors the reference's ``Rng``
facade (``src/linalg.py:64-91``) and ``bench.build_matrix``
(``src/bench.py:105-109``, points from ``Rng(seed).child(0)``).
§8(d) fixes the recipes; there is no public dataset -- every input is
synthetic and seeded.

``n`` can be overridden to get the same distribution and kernel at a reduced
size (used for CPU-checkable parity cases of configs 3-5).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .estimators import EstimatorConfig
from .kernels import KernelSpec
from .linalg import Rng
from .precond import PreconditionerConfig


@dataclass(frozen=True)
class Workload:
    name: str
    spec: KernelSpec
    points: np.ndarray
    config: EstimatorConfig
    path: str            # "stored" or "on_the_fly"

    @property
    def n(self) -> int:
        return self.points.shape[0]


FULL_N = {1: 2048, 2: 16384, 3: 65536, 4: 262144, 5: 1048576}


def points_for(index: int, n: int | None = None, seed: int = 0) -> np.ndarray:
    """Seeded point set of BASELINE config ``index`` (1-based)."""
    n = FULL_N[index] if n is None else int(n)
    pts_rng = Rng(seed).child(0)
    if index == 1:
        return pts_rng.gen.uniform(0.0, 1.0, (n, 3))
    if index == 2:
        return pts_rng.normal((n, 8))              # sample_index_points(n, 8, ...)
    if index == 3:
        return pts_rng.gen.uniform(0.0, 1.0, (n, 2))
    if index == 4:
        centres = pts_rng.child(0).gen.uniform(0.0, 1.0, (16, 3))
        labels = pts_rng.child(1).gen.integers(0, 16, n)
        return centres[labels] + 0.05 * pts_rng.child(2).normal((n, 3))
    if index == 5:
        return pts_rng.gen.uniform(0.0, 1.0, (n, 3))
    raise ValueError(f"no BASELINE config {index}")


def baseline(index: int, n: int | None = None, seed: int = 0, algorithm: str | None = None,
             dtype: str | None = None, rank: int | None = None, num_probes: int | None = None) -> Workload:
    """BASELINE.json ``configs[index-1]`` (t = 20, q = 5, oversample 10, seed 0)."""
    pts = points_for(index, n, seed)
    if index == 1:
        spec = KernelSpec("matern52", amplitude=1.0, length_scale=0.2, jitter=1e-2)
        cfg = EstimatorConfig("r3", 16, 20, "rademacher", PreconditionerConfig("rand-svd", 64, 5), seed,
                              dtype="fp64")
        path = "stored"
    elif index == 2:
        spec = KernelSpec("rbf", amplitude=1.0, length_scale=1.0, jitter=1e-3)
        cfg = EstimatorConfig("r3", 32, 20, "rademacher", PreconditionerConfig("rand-svd", 256, 5), seed,
                              dtype="fp32")
        path = "stored"
    elif index == 3:
        spec = KernelSpec("matern52", amplitude=1.0, length_scale=0.05, jitter=1e-2)
        cfg = EstimatorConfig("r3", 64, 20, "gaussian", PreconditionerConfig("rand-svd", 512, 5), seed,
                              dtype="fp32")
        path = "stored"
    elif index == 4:
        spec = KernelSpec("rbf", amplitude=1.0, length_scale=0.1, jitter=1e-2)
        cfg = EstimatorConfig("r5", 64, 20, "rademacher", PreconditionerConfig("rand-svd", 1024, 5), seed,
                              dtype="fp32")
        path = "on_the_fly"
    elif index == 5:
        spec = KernelSpec("matern52", amplitude=1.0, length_scale=0.02, jitter=1e-1)
        cfg = EstimatorConfig("r3", 128, 20, "rademacher", PreconditionerConfig("rand-svd", 2048, 5), seed,
                              dtype="fp32")
        path = "on_the_fly"
    else:
        raise ValueError(f"no BASELINE config {index}")
    if algorithm is not None:
        cfg = replace(cfg, algorithm=algorithm)
    if dtype is not None:
        cfg = replace(cfg, dtype=dtype)
    if rank is not None:
        cfg = replace(cfg, precond=replace(cfg.precond, rank=rank))
    if num_probes is not None:
        cfg = replace(cfg, num_probes=num_probes)
    return Workload(f"config{index}", spec, pts, cfg, path)
