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

__all__ = ["PRECOND_KINDS", "DEVICE_PRECOND_KINDS", "PreconditionerConfig", "OVERSAMPLE", "DIAG_FLOOR",
           "Preconditioner", "build_preconditioner"]

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


class Preconditioner:
    """A preconditioner built on the GPU and held in its own librld handle: the reference's
    ``Preconditioner`` (``src/precond.py:58-118``) -- ``log_det``, ``solve_sqrt(z)`` = N^-1 z,
    ``solve_sqrt_t(x)`` = N^-T x, and ``solve(u)`` = P^-1 u -- with the factors (U, h, g, sqrt(base))
    resident in HBM.  Vectors are length-n arrays or n x m blocks (numpy or torch CUDA)."""

    def __init__(self, kind, sess, resident_keep, info):
        self.kind = kind
        self.sess = sess
        self._keep = resident_keep
        self.log_det = float(info.log_det)
        self.rank = int(info.rank)
        self.rank_kept = int(info.rank_kept)
        self.attempts = int(info.attempts)
        self.qr_fallback = bool(info.qr_fallback)
        self.n = None

    def _apply(self, op, X):
        import ctypes as C

        import numpy as np
        import torch

        from . import _native as N

        is_torch = isinstance(X, torch.Tensor)
        T = X.detach().to(torch.float64) if is_torch else torch.from_numpy(np.asarray(X, dtype=np.float64))
        vec = T.ndim == 1
        rows = (T[None, :] if vec else T.T).contiguous().to(f"cuda:{self.sess.device}")   # m x n rows
        if rows.shape[1] != self.n:
            raise ValueError(f"expected length {self.n}, got {rows.shape[1]}")
        out = torch.empty_like(rows)
        self.sess.after_torch()
        self.sess.handle.check(self.sess.lib.rld_precond_apply(self.sess.handle.ptr, op, rows.shape[0], rows.data_ptr(),
                                                               out.data_ptr()), "rld_precond_apply")
        res = out[0] if vec else out.T
        if is_torch:
            return res.to(X.device)
        return res.cpu().numpy()

    def solve_sqrt(self, Z):
        """N^-1 Z (src/precond.py:102-108)."""
        from . import _native as N

        return self._apply(N.SOLVE_SQRT, Z)

    def solve_sqrt_t(self, X):
        """N^-T X (src/precond.py:110-115)."""
        from . import _native as N

        return self._apply(N.SOLVE_SQRT_T, X)

    def solve(self, U):
        """P^-1 U = N^-T N^-1 U."""
        from . import _native as N

        return self._apply(N.SOLVE, U)


def build_preconditioner(M, cfg: PreconditionerConfig, rng, dtype: str = "fp64", path: str = "auto") -> Preconditioner:
    """``build_preconditioner(M, cfg, rng)`` of ``src/precond.py:236-267`` on the GPU.

    ``rng`` is the reference's stream facade (``linalg.Rng``): the estimator passes
    ``Rng(seed).child(1)``; the sketch of attempt a is ``rng.child(a)`` (``src/precond.py:183``) and
    the rank-one start vector ``rng`` itself (``src/precond.py:202``), regenerated on the device from
    their Philox keys.  ``M`` is what ``rstar_logdet`` accepts (dense matrix or KernelMatrix)."""
    import ctypes as C

    from . import _native as N
    from ._session import Session
    from .linalg import philox_key

    if cfg.kind not in DEVICE_PRECOND_KINDS:
        raise ValueError(f"unknown preconditioner kind {cfg.kind!r}")
    sess = Session()
    prob, keep = sess.problem_for(M, dtype, path)
    sess.handle.check(sess.lib.rld_prepare(sess.handle.ptr, C.byref(prob)), "rld_prepare")
    n = int(prob.n)
    if cfg.kind not in ("identity", "diagonal", "rank-one") and cfg.rank > n:
        raise ValueError(f"rank {cfg.rank} exceeds dimension {n}")     # src/precond.py:241-242
    c = N.Config()
    c.order, c.num_probes, c.lanczos_iters = 3, 1, 1
    c.precond_kind = DEVICE_PRECOND_KINDS[cfg.kind]
    c.precond_rank, c.precond_iters = cfg.rank, cfg.num_iters
    c.oversample, c.diag_floor, c.keep_rtol, c.orth_rtol = OVERSAMPLE, DIAG_FLOOR, 1e-14, 1e-12
    c.breakdown_rtol = 1e-12
    c.precond_scale = cfg.scale
    for a in range(2):
        o0, o1 = philox_key(rng.seed, rng.path + (a,))
        c.omega_key[2 * a], c.omega_key[2 * a + 1] = o0, o1
    p0, p1 = philox_key(rng.seed, rng.path)
    c.precond_key[0], c.precond_key[1] = p0, p1
    inp = N.Inputs()
    info = N.PrecondInfo()
    sess.handle.check(sess.lib.rld_precond_build(sess.handle.ptr, C.byref(c), C.byref(inp), C.byref(info)),
                      "rld_precond_build")
    P = Preconditioner(cfg.kind, sess, keep, info)
    P.n = n
    return P
