"""Preconditioner configuration (``src/precond.py:25-55``).

The device builds all nine kinds of P = diag(base) + A A^T
(``src/precond.py:201-267``): the randomized truncated SVD of the r* hot path
(168-198) and its ``-scaled`` variant, identity, diagonal, the rank-one power
iteration, the pivoted partial Cholesky (``-scaled``), and the dense truncated
eigendecomposition (``-scaled``; one GPU, K materialised in float64), each with
its determinant-lemma log det (69-80) and factored square root (90-115).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["PRECOND_KINDS", "DEVICE_PRECOND_KINDS", "PreconditionerConfig", "OVERSAMPLE", "DIAG_FLOOR"]

PRECOND_KINDS = (
    "identity",
    "diagonal",
    "rank-one",
    "partial-cholesky",
    "partial-cholesky-scaled",
    "trunc-svd",
    "trunc-svd-scaled",
    "rand-svd",
    "rand-svd-scaled",
)
DEVICE_PRECOND_KINDS = {"rand-svd": 0, "identity": 1, "diagonal": 2, "rand-svd-scaled": 3, "partial-cholesky": 4,
                        "partial-cholesky-scaled": 5, "trunc-svd": 6, "trunc-svd-scaled": 7, "rank-one": 8}

OVERSAMPLE = 10          # src/precond.py:165
DIAG_FLOOR = 1e-12       # src/precond.py:37


@dataclass(frozen=True)
class PreconditionerConfig:
    kind: str = "rand-svd"
    rank: int = 25
    num_iters: int = 5
    scale: float = 1e-6

    def __post_init__(self):
        if self.kind not in PRECOND_KINDS:
            raise ValueError(f"unknown preconditioner kind {self.kind!r}")
        if self.rank < 0:
            raise ValueError("rank must be >= 0")
        if self.num_iters < 1:
            raise ValueError("num_iters must be >= 1")
        if self.scale <= 0:
            raise ValueError("scale must be positive")
