"""Pure-Python Philox4x64-10 and numpy's consumption rules for it.

TEST INFRASTRUCTURE ONLY (see rstar_oracle.py's header for who may import it).

Restates the counter-based generator numpy's ``Philox`` bit generator uses
(third-party dependency: numpy 2.3.5, ``numpy/random/src/philox/philox.h`` --
Salmon et al., "Parallel random numbers: as easy as 1, 2, 3", SC'11), and the
two consumption rules the reference's streams rely on:

* ``random_raw``: the 256-bit counter is incremented *before* each block of
  four 64-bit words, so word q of a fresh stream is lane q % 4 of
  Philox(counter = q // 4 + 1, key).
* ``integers(0, 2)``: one 32-bit half per draw, low half first, value = bit 31
  (Lemire's bounded method with range 2 never rejects) -- the Rademacher rows
  of ``src/linalg.py:84-85``.

The CUDA generator (``csrc/rld_device.cuh`` philox4x64_10 / philox_word and
``vec_kernels.cu`` rademacher_kernel) implements exactly these formulas; the
CPU tests pin this module against numpy, the GPU tests pin the device against
numpy.
"""

from __future__ import annotations

import numpy as np

M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK = (1 << 64) - 1


def philox4x64_10(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for r in range(10):
        if r:
            k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
        p0, p1 = M0 * c[0], M1 * c[2]
        hi0, lo0 = p0 >> 64, p0 & MASK
        hi1, lo1 = p1 >> 64, p1 & MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


def raw_word(q: int, key) -> int:
    blk = (q >> 2) + 1
    return philox4x64_10([blk & MASK, blk >> 64, 0, 0], key)[q & 3]


def rademacher(key, rows: int, n: int) -> np.ndarray:
    out = np.empty((rows, n))
    for r in range(rows):
        for j in range(n):
            f = r * n + j
            w = raw_word(f >> 1, key)
            u = (w >> 32) if (f & 1) else (w & 0xFFFFFFFF)
            out[r, j] = 1.0 if (u >> 31) else -1.0
    return out
