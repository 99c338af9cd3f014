"""The estimator API of the reference (``src/estimators.py``), served by the GPU.

``rstar_logdet(M, cfg)`` / ``estimate_logdet(M, cfg)`` keep the reference's
signature and ``LogDetEstimate`` result (``src/estimators.py:32-55, 77-96,
132-138``).  ``M`` may be what the reference takes -- a dense n x n matrix
(numpy, or a torch CUDA tensor that stays on the device) -- or a
``KernelMatrix(spec, points)`` / ``(spec, points)`` pair, which lets K be built
in HBM or generated tile by tile on the fly (BASELINE configs 4-5 cannot
materialise M anywhere).

Everything below the call runs in ``librld.so`` on the GPU: the rand-SVD
preconditioner, all-probe Lanczos, the multishift solves and the Hutchinson
mean.  There is no CPU fallback: a missing library raises.

Random inputs follow the reference's streams exactly: probes from
``Rng(seed).child(2)`` and the sketch from ``Rng(seed).child(1).child(attempt)``
(``src/estimators.py:61-64``, ``src/precond.py:183``), regenerated on the GPU
from the streams' Philox keys -- Rademacher rows bit-identical to numpy, Gaussian
rows through a device port of numpy's ziggurat.  Explicit ``probes=`` /
``omega=`` rows may still be injected.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .linalg import Rng, philox_key
from .precond import DEVICE_PRECOND_KINDS, OVERSAMPLE, DIAG_FLOOR, PreconditionerConfig
from .probes import DEVICE_PROBE_KINDS, PROBE_KINDS, make_probes

__all__ = ["ALGORITHMS", "EstimatorConfig", "LogDetEstimate", "estimate_logdet", "rstar_logdet", "slq_logdet",
           "exact_logdet", "ResidentMatrix"]

ALGORITHMS = ("r1", "r3", "r5", "slq", "exact")
DTYPES = ("fp64", "fp32")
PATHS = ("auto", "stored", "on_the_fly")


@dataclass(frozen=True)
class EstimatorConfig:
    algorithm: str = "r3"
    num_probes: int = 35
    lanczos_iters: int = 20
    probe_kind: str = "rademacher"
    precond: PreconditionerConfig = field(default_factory=PreconditionerConfig)
    seed: int = 0
    # B200 additions (appended so positional use of the reference fields is unchanged)
    dtype: str = "fp64"       # arithmetic of K and of the K x block products
    path: str = "auto"        # KernelMatrix input: "stored" in HBM, "on_the_fly", or "auto" by capacity

    def __post_init__(self):
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.num_probes < 1 or self.lanczos_iters < 1:
            raise ValueError("num_probes and lanczos_iters must be >= 1")
        if self.dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {DTYPES}, got {self.dtype!r}")
        if self.path not in PATHS:
            raise ValueError(f"path must be one of {PATHS}, got {self.path!r}")


@dataclass
class LogDetEstimate:
    value: float
    logdet_P: float
    trace_term: float
    per_probe_values: np.ndarray
    wall_time: float
    clamped_eigs: int = 0
    # device diagnostics (not in the reference record)
    device_time: float = 0.0
    phase_ms: tuple = ()
    kv_products: int = 0
    kernel_launches: int = 0
    rank_kept: int = 0
    attempts: int = 1
    path: str = "stored"      # where K lived for this estimate: "stored" in HBM or "on_the_fly"
    qr_fallback: bool = False  # the sketch QR fell back from Cholesky-QR to Householder (TSQR when sharded)


def _sketch_width(cfg: EstimatorConfig, n: int) -> int:
    return min(cfg.precond.rank + OVERSAMPLE, n)


def make_config(cfg: EstimatorConfig, n: int) -> N.Config:
    """EstimatorConfig -> rld_config (validation mirrors src/estimators.py:41-45, src/precond.py:241-242).

    ``slq`` runs on K itself (src/estimators.py:106): the preconditioner fields are
    not used, exactly as the reference ignores them."""
    slq = cfg.algorithm == "slq"
    if cfg.algorithm not in ("r1", "r3", "r5", "slq"):
        raise ValueError(f"estimator got algorithm {cfg.algorithm!r}")
    if cfg.probe_kind not in PROBE_KINDS:
        raise ValueError(f"unknown probe kind {cfg.probe_kind!r}")
    if cfg.probe_kind not in DEVICE_PROBE_KINDS:
        raise NotImplementedError(f"probe kind {cfg.probe_kind!r} is outside the r* hot path")
    if not slq and cfg.precond.kind not in ("identity", "diagonal", "rank-one") and cfg.precond.rank > n:
        raise ValueError(f"rank {cfg.precond.rank} exceeds dimension {n}")     # src/precond.py:241-242
    c = N.Config()
    c.estimator = N.ESTIMATOR_SLQ if slq else N.ESTIMATOR_RSTAR
    c.order = 3 if slq else int(cfg.algorithm[1])
    c.num_probes = cfg.num_probes
    c.lanczos_iters = cfg.lanczos_iters
    c.probe_kind = DEVICE_PROBE_KINDS[cfg.probe_kind]
    c.precond_kind = N.PRECOND_IDENTITY if slq else DEVICE_PRECOND_KINDS[cfg.precond.kind]
    c.precond_rank = cfg.precond.rank
    c.precond_iters = cfg.precond.num_iters
    c.oversample = OVERSAMPLE
    c.diag_floor = DIAG_FLOOR
    c.keep_rtol = 1e-14
    c.breakdown_rtol = 1e-12
    c.orth_rtol = 1e-12
    k0, k1 = philox_key(cfg.seed, (2,))
    c.probe_key[0], c.probe_key[1] = k0, k1
    for a in range(2):
        o0, o1 = philox_key(cfg.seed, (1, a))
        c.omega_key[2 * a], c.omega_key[2 * a + 1] = o0, o1
    if cfg.probe_kind == "normal-orthogonal":
        nb = -(-cfg.num_probes // n)
        if nb > N.MAX_PROBE_BLOCKS:
            raise NotImplementedError(f"normal-orthogonal probes need s <= {N.MAX_PROBE_BLOCKS} n")
        for b in range(nb):
            b0, b1 = philox_key(cfg.seed, (2, b))
            c.probe_block_keys[2 * b], c.probe_block_keys[2 * b + 1] = b0, b1
    c.precond_scale = cfg.precond.scale
    p0, p1 = philox_key(cfg.seed, (1,))
    c.precond_key[0], c.precond_key[1] = p0, p1
    return c


class _Inputs:
    """Random rows the caller injects explicitly (kept alive for the duration of a
    call).  By default nothing is injected: the device regenerates the
    reference's streams itself -- Rademacher probes and Gaussian rows (sketch,
    Gaussian probes) bit-identical to numpy's Philox / ziggurat streams."""

    def __init__(self, cfg: EstimatorConfig, n: int, probes=None, omega=None):
        self.keep = []
        self.struct = N.Inputs()
        self.struct.memory = N.HOST
        if probes is not None:
            P = np.ascontiguousarray(np.asarray(probes, dtype=np.float64))
            if P.shape != (cfg.num_probes, n):
                raise ValueError(f"probes must be {cfg.num_probes} x {n}")
            self.keep.append(P)
            self.struct.probes = P.ctypes.data
        if omega is not None and cfg.precond.kind in ("rand-svd", "rand-svd-scaled"):
            w = _sketch_width(cfg, n)
            om = [np.ascontiguousarray(np.asarray(o, dtype=np.float64)) for o in omega]
            for o in om:
                if o.shape != (w, n):
                    raise ValueError(f"sketch rows must be {w} x {n}")
            self.keep.extend(om)
            self.struct.omega0 = om[0].ctypes.data
            if len(om) > 1:
                self.struct.omega1 = om[1].ctypes.data
            self._seed, self._w, self._n = cfg.seed, w, n

    def add_retry_sketch(self):
        o = Rng(self._seed).child(1).child(1).normal((self._w, self._n))
        self.keep.append(o)
        self.struct.omega1 = o.ctypes.data


def _call_with_retry(call, inputs: _Inputs, handle: N.Handle, what: str):
    rc = call()
    handle.check(rc, what)


def _path_of(prob) -> str:
    return "on_the_fly" if (prob.source == N.SOURCE_POINTS and prob.path == N.PATH_ON_THE_FLY) else "stored"


def _result(res: N.Result, per: np.ndarray, start: float, path: str = "stored") -> LogDetEstimate:
    return LogDetEstimate(res.value, res.logdet_P, res.trace_term, per, time.perf_counter() - start,
                          clamped_eigs=int(res.clamped_eigs), device_time=res.wall_time, phase_ms=tuple(res.phase_ms),
                          kv_products=res.kv_products, kernel_launches=res.kernel_launches, rank_kept=res.rank_kept,
                          attempts=res.attempts, path=path, qr_fallback=bool(res.qr_fallback))


def rstar_logdet(M, cfg: EstimatorConfig, probes=None, omega=None) -> LogDetEstimate:
    """Rational-approximation estimate of log det M (algorithms r1/r3/r5) on the GPU."""
    if cfg.algorithm not in ("r1", "r3", "r5"):
        raise ValueError(f"rstar_logdet got algorithm {cfg.algorithm!r}")
    return _run(M, cfg, probes, omega)


def slq_logdet(M, cfg: EstimatorConfig, probes=None) -> LogDetEstimate:
    """Stochastic Lanczos quadrature estimate of log det M (``src/estimators.py:99-122``):
    Lanczos on M itself with full two-pass reorthogonalisation (no preconditioner),
    the same probe stream as the rational estimators, Gauss quadrature of log on
    each probe's tridiagonal (Ritz values <= 0 floored at 1e-300 and counted in
    ``clamped_eigs``).  ``logdet_P`` is 0 and ``value == trace_term``."""
    if cfg.algorithm != "slq":
        raise ValueError(f"slq_logdet got algorithm {cfg.algorithm!r}")
    return _run(M, cfg, probes, None)


def _run(M, cfg: EstimatorConfig, probes, omega) -> LogDetEstimate:
    from ._session import session

    start = time.perf_counter()
    sess = session()
    prob, keep = sess.problem_for(M, cfg.dtype, cfg.path)
    n = int(prob.n)
    c = make_config(cfg, n)
    inputs = _Inputs(cfg, n, probes, omega)
    per = np.empty(cfg.num_probes)
    res = N.Result()
    res.per_probe = per.ctypes.data_as(C.POINTER(C.c_double))
    _call_with_retry(lambda: sess.lib.rld_logdet(sess.handle.ptr, C.byref(prob), C.byref(c),
                                                 C.byref(inputs.struct), C.byref(res)),
                     inputs, sess.handle, "rld_logdet")
    del keep
    return _result(res, per, start, _path_of(prob))


def exact_logdet(M, dtype: str = "fp64") -> LogDetEstimate:
    """Cholesky log det on the GPU (``src/estimators.py:125-129``)."""
    from ._session import session

    start = time.perf_counter()
    sess = session()
    prob, keep = sess.problem_for(M, dtype, "stored")
    sess.handle.check(sess.lib.rld_prepare(sess.handle.ptr, C.byref(prob)), "rld_prepare")
    v = C.c_double()
    sess.handle.check(sess.lib.rld_exact_logdet(sess.handle.ptr, C.byref(v)), "rld_exact_logdet")
    return LogDetEstimate(v.value, v.value, 0.0, np.empty(0), time.perf_counter() - start)


def estimate_logdet(M, cfg: EstimatorConfig) -> LogDetEstimate:
    """Dispatch on cfg.algorithm (``src/estimators.py:132-138``)."""
    if cfg.algorithm in ("r1", "r3", "r5"):
        return rstar_logdet(M, cfg)
    if cfg.algorithm == "slq":
        return slq_logdet(M, cfg)
    return exact_logdet(M)


class ResidentMatrix:
    """K made resident in HBM once (or its points, for the on-the-fly path), so
    that repeated estimates touch no host memory: the device-resident form
    ``bench.py`` times.  Owns its own librld handle."""

    def __init__(self, M, dtype: str = "fp64", path: str = "auto", device: int | None = None,
                 shard: bool | None = None, session=None):
        """``shard`` (default: True under torch.distributed with world size > 1)
        joins the process-wide NCCL session and keeps only this rank's rows of K;
        ``shard=False`` gives an independent single-GPU replica.  ``session`` binds an
        explicit session (a virtual-shard rank of ``parallel.VirtualShards``)."""
        from ._session import Session, dist_world
        from ._session import session as process_session

        rank, world, local = dist_world()
        if shard is None:
            shard = world > 1
        if session is not None:
            self.sess = session
        elif shard and world > 1:
            self.sess = process_session()
        else:
            self.sess = Session(local if device is None else device)
        self.dtype = dtype
        prob, self._keep = self.sess.problem_for(M, dtype, path)
        self.n = int(prob.n)
        self.path = _path_of(prob)
        self.sess.handle.check(self.sess.lib.rld_prepare(self.sess.handle.ptr, C.byref(prob)), "rld_prepare")

    def estimate(self, cfg: EstimatorConfig, probes=None, omega=None, inputs: N.Inputs | None = None) -> LogDetEstimate:
        if cfg.dtype != self.dtype:
            raise ValueError(f"matrix is resident as {self.dtype}, config asks for {cfg.dtype}")
        start = time.perf_counter()
        c = make_config(cfg, self.n)
        per = np.empty(cfg.num_probes)
        res = N.Result()
        res.per_probe = per.ctypes.data_as(C.POINTER(C.c_double))
        if inputs is not None:   # pre-staged (e.g. device-resident) random rows
            self.sess.handle.check(self.sess.lib.rld_logdet_resident(self.sess.handle.ptr, C.byref(c), C.byref(inputs),
                                                                     C.byref(res)), "rld_logdet_resident")
        else:
            inp = _Inputs(cfg, self.n, probes, omega)
            _call_with_retry(lambda: self.sess.lib.rld_logdet_resident(self.sess.handle.ptr, C.byref(c),
                                                                       C.byref(inp.struct), C.byref(res)),
                             inp, self.sess.handle, "rld_logdet_resident")
        return _result(res, per, start, self.path)

    def kv_apply(self, V):
        """Y = V K for device float64 rows V (m x n torch CUDA tensor).  With a
        row-sharded handle (world size > 1) Y holds this rank's columns only,
        m x rows.  Ordered after torch's current stream and before its later work."""
        import torch

        from .parallel import shard_bounds

        V = V.detach().to(torch.float64).contiguous()
        if V.ndim != 2 or V.shape[1] != self.n:
            raise ValueError(f"V must be m x {self.n}")
        r0, r1 = shard_bounds(self.n, self.sess.world_size, self.sess.rank)
        Y = torch.empty((V.shape[0], r1 - r0), dtype=torch.float64, device=V.device)
        cur = torch.cuda.current_stream(V.device)
        ext = self.sess.torch_stream()
        ext.wait_stream(cur)
        self.sess.handle.check(self.sess.lib.rld_kv_apply(self.sess.handle.ptr, V.shape[0], V.data_ptr(),
                                                          Y.data_ptr()), "rld_kv_apply")
        # V and Y belong to torch's current stream; it waits for the product here, so
        # no later reuse of their blocks can overtake it (no record_stream: the handle's
        # stream may be destroyed before the tensors are freed)
        cur.wait_stream(ext)
        return Y

    def exact_logdet(self) -> float:
        v = C.c_double()
        self.sess.handle.check(self.sess.lib.rld_exact_logdet(self.sess.handle.ptr, C.byref(v)), "rld_exact_logdet")
        return v.value
