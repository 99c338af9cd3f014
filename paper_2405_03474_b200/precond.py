"""Preconditioner configuration (``src/precond.py:25-55``).

The device builds the randomized truncated-SVD preconditioner
P = diag(base) + A A^T (``src/precond.py:168-198, 231-267``) together with its
determinant-lemma log det (69-80) and factored square root (90-115).  The
``identity`` and ``diagonal`` kinds are also built (test doubles for the
reference's own identities); the remaining kinds are out of scope for this
hot path and raise ``NotImplementedError`` when an estimate asks for them.
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
DEVICE_PRECOND_KINDS = {"rand-svd": 0, "identity": 1, "diagonal": 2}

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
