"""Host-side types mirrored from the reference's ``linalg`` module: the error
types the estimator raises, the seeded splittable RNG facade, and the Philox
key derivation the device generators consume.

Reference: ``src/linalg.py:24-33`` (exceptions), ``src/linalg.py:64-91`` (Rng).
"""

from __future__ import annotations

import numpy as np

__all__ = ["NotPositiveDefinite", "SingularShiftedSystem", "RankDeficient", "Rng", "philox_key"]


class NotPositiveDefinite(Exception):
    """Cholesky hit a non-positive pivot (``src/linalg.py:24-25``)."""


class SingularShiftedSystem(Exception):
    """A shifted tridiagonal solve met a pivot below 1e-300 (``src/linalg.py:28-29``)."""


class RankDeficient(Exception):
    """The sketch lost rank in orthonormalisation, after one retry (``src/linalg.py:32-33``)."""


class Rng:
    """Deterministic, splittable stream: Philox keyed by
    ``SeedSequence(seed, spawn_key=path)`` (``src/linalg.py:64-91``)."""

    def __init__(self, seed: int, path: tuple[int, ...] = ()):
        self.seed = int(seed)
        self.path = tuple(int(p) for p in path)
        ss = np.random.SeedSequence(self.seed, spawn_key=self.path)
        self.gen = np.random.Generator(np.random.Philox(ss))

    def child(self, i: int) -> "Rng":
        return Rng(self.seed, self.path + (i,))

    def normal(self, shape) -> np.ndarray:
        return self.gen.standard_normal(shape)

    def rademacher(self, shape) -> np.ndarray:
        return 2.0 * self.gen.integers(0, 2, size=shape).astype(np.float64) - 1.0

    def __repr__(self):
        return f"Rng(seed={self.seed}, path={self.path})"


def philox_key(seed: int, path: tuple[int, ...]) -> tuple[int, int]:
    """The two 64-bit Philox4x64 key words numpy derives for stream
    ``(seed, path)``; the device generators reproduce that stream from them
    (counter starts at 0 and pre-increments, numpy's ``philox_next``)."""
    st = np.random.Philox(np.random.SeedSequence(int(seed), spawn_key=tuple(path))).state["state"]
    key = [int(k) for k in st["key"]]
    ctr = [int(c) for c in st["counter"]]
    if any(ctr):
        raise AssertionError("fresh Philox stream must start at counter 0")
    return key[0], key[1]
