"""Gaussian-process kernels and the device-built covariance matrix.

Mirrors ``src/kernels.py`` (``KernelSpec`` 17-30, ``sample_index_points``
33-37, ``kernel_value`` 49-56, ``build_covariance`` 59-73).  ``build_covariance``
builds K on the GPU (``rld_build_covariance``); ``KernelMatrix`` is the lazy
(spec, points) form the estimator accepts so that K can be streamed from HBM or
generated tile by tile without ever existing on the host.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .linalg import Rng

__all__ = ["KernelSpec", "KernelMatrix", "sample_index_points", "kernel_value", "build_covariance"]

SQRT5 = np.sqrt(5.0)


@dataclass(frozen=True)
class KernelSpec:
    family: str = "rbf"  # "rbf" or "matern52"
    amplitude: float = 1.0
    length_scale: float = 1.0
    jitter: float = 1e-6

    def __post_init__(self):
        if self.family not in ("rbf", "matern52"):
            raise ValueError(f"unknown kernel family {self.family!r}")
        if self.amplitude <= 0 or self.length_scale <= 0:
            raise ValueError("amplitude and length_scale must be positive")
        if self.jitter < 0:
            raise ValueError("jitter must be non-negative")


@dataclass(frozen=True)
class KernelMatrix:
    """K = k(x_i, x_j) + jitter I, given by its points (n x d)."""

    spec: KernelSpec
    points: object  # numpy (host) or torch (cuda) n x d float64 array

    @property
    def n(self) -> int:
        return int(self.points.shape[0])

    @property
    def d(self) -> int:
        return int(self.points.shape[1])


def sample_index_points(n: int, d: int, rng: Rng) -> np.ndarray:
    """n standard-normal index points in d dimensions (src/kernels.py:33-37)."""
    if n < 1 or d < 1:
        raise ValueError("n and d must be >= 1")
    return rng.normal((n, d))


def kernel_value(spec: KernelSpec, x, y) -> float:
    """Covariance between two points, jitter excluded (src/kernels.py:49-56)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    y = np.atleast_1d(np.asarray(y, dtype=np.float64))
    if x.shape != y.shape:
        raise ValueError(f"dimension mismatch: {x.shape} vs {y.shape}")
    r = float(np.linalg.norm(x - y))
    a2 = spec.amplitude ** 2
    if spec.family == "rbf":
        return float(a2 * np.exp(-(r * r) / (2.0 * spec.length_scale ** 2)))
    u = SQRT5 * r / spec.length_scale
    return float(a2 * (1.0 + u + u * u / 3.0) * np.exp(-u))


def build_covariance(spec: KernelSpec, points, dtype: str = "fp64", device: str = "cuda"):
    """Dense K[i, j] = k(x_i, x_j) + jitter [i == j], built on the GPU.

    Returns a torch CUDA tensor (``device="cuda"``) or a numpy array
    (``device="cpu"``; built on the GPU, then copied to the host)."""
    from ._session import session
    from ._native import DEVICE, HOST

    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if pts.ndim != 2:
        raise ValueError("points must be an n x d array")
    sess = session()
    prob, keep = sess.problem_for(KernelMatrix(spec, pts), dtype, "stored")
    n = pts.shape[0]
    if device == "cpu":
        out = np.empty((n, n), dtype=np.float64 if dtype == "fp64" else np.float32)
        sess.handle.check(sess.lib.rld_build_covariance(sess.handle.ptr, C.byref(prob), out.ctypes.data, HOST),
                          "rld_build_covariance")
        return out
    import torch

    out = torch.empty((n, n), dtype=torch.float64 if dtype == "fp64" else torch.float32,
                      device=f"cuda:{sess.handle.device}")
    sess.after_torch()    # the block may still be in use by pending torch kernels
    sess.handle.check(sess.lib.rld_build_covariance(sess.handle.ptr, C.byref(prob), out.data_ptr(), DEVICE),
                      "rld_build_covariance")
    sess.before_torch()   # later torch work on `out` sees the build
    return out
