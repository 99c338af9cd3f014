"""Hutchinson probe rows (``src/probes.py:12-44``).

On the estimator path all three kinds are generated on the GPU from the
reference's numpy streams: Rademacher bit-identical (``rld_rademacher``),
Gaussian through the device ziggurat (``rld_normal``), normal-orthogonal as
device Gaussian blocks orthonormalised on the device, scaled by chi radii that
continue the same stream (``rld_chi_radii``).  ``make_probes`` is the host-side
form used to inject probes explicitly (parity mode).
"""

from __future__ import annotations

import numpy as np

from .linalg import Rng

__all__ = ["PROBE_KINDS", "DEVICE_PROBE_KINDS", "make_probes"]

PROBE_KINDS = ("rademacher", "gaussian", "normal-orthogonal")
DEVICE_PROBE_KINDS = {"rademacher": 0, "gaussian": 1, "normal-orthogonal": 2}


def make_probes(kind: str, s: int, n: int, rng: Rng) -> np.ndarray:
    """s probe rows of length n (mean 0, variance 1 entries)."""
    if kind not in PROBE_KINDS:
        raise ValueError(f"unknown probe kind {kind!r}")
    if s < 1 or n < 1:
        raise ValueError("s and n must be >= 1")
    if kind == "rademacher":
        return rng.rademacher((s, n))
    if kind == "gaussian":
        return rng.normal((s, n))
    raise NotImplementedError("host normal-orthogonal probes: generated on the device by the estimator")
