"""Process-level state: the librld handle this process drives, and the
translation of Python-side inputs (numpy / torch arrays, ``KernelMatrix``) into
the C-ABI structs of ``include/rld.h``.

One process drives one GPU.  Under ``torch.distributed`` with world size > 1
the handle joins an NCCL communicator and owns the row shard
``[rank*ceil(n/G), (rank+1)*ceil(n/G))`` of every n-vector.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _native as N
from .kernels import KernelMatrix, KernelSpec

_DTYPES = {"fp64": N.FP64, "fp32": N.FP32}
_FAMILIES = {"rbf": N.RBF, "matern52": N.MATERN52}


def _torch():
    try:
        import torch

        return torch
    except Exception:  # pragma: no cover - torch is part of the image
        return None


def _is_torch(x) -> bool:
    t = _torch()
    return t is not None and isinstance(x, t.Tensor)


def dist_world():
    """(rank, world_size, local_device) from torch.distributed / env."""
    t = _torch()
    if t is not None and t.distributed.is_available() and t.distributed.is_initialized():
        rank, world = t.distributed.get_rank(), t.distributed.get_world_size()
    else:
        rank, world = 0, 1
    local = int(os.environ.get("LOCAL_RANK", "0")) if world > 1 else 0
    return rank, world, local


def hbm_bytes(device: int) -> int:
    """Total HBM of the device: the 'auto' path choice depends on the problem and the GPU only,
    never on what this process (or another) happens to have allocated, so every trial of a
    sweep takes the same path."""
    t = _torch()
    if t is not None and t.cuda.is_available():
        return int(t.cuda.get_device_properties(device).total_memory)
    return 180 * (1 << 30)


class Session:
    def __init__(self, device: int | None = None, rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None,
                 group: "N.VirtualGroup | None" = None):
        if device is None:
            _, _, device = dist_world()
        self.handle = N.Handle(device, rank, world_size, nccl_id, group)
        self.lib = self.handle.lib
        self.rank, self.world_size, self.device = rank, world_size, device

    # -- stream ordering against torch ---------------------------------------
    def torch_stream(self):
        """The handle's stream as a torch ExternalStream (None without CUDA torch)."""
        t = _torch()
        if t is None or not t.cuda.is_available():
            return None
        if getattr(self, "_ext", None) is None:
            self._ext = t.cuda.ExternalStream(self.handle.stream, device=self.device)
        return self._ext

    def after_torch(self):
        """Order the handle's stream after everything torch has queued on its current stream
        (the handle's stream is non-blocking: without this, a C call could read a torch tensor
        before the kernel producing it ran, or write a block the caching allocator just handed
        out while its previous owner's kernels are still pending)."""
        t = _torch()
        if t is None or not t.cuda.is_available() or not t.cuda.is_initialized():
            return
        self.torch_stream().wait_stream(t.cuda.current_stream(self.device))

    def before_torch(self):
        """Order torch's current stream after the handle's queued work (results it wrote)."""
        t = _torch()
        if t is None or not t.cuda.is_available() or not t.cuda.is_initialized():
            return
        t.cuda.current_stream(self.device).wait_stream(self.torch_stream())

    # -- problem translation -------------------------------------------------
    def resolve_path(self, M, dtype: str, path: str) -> str:
        if not isinstance(M, KernelMatrix):
            return "stored"
        if path in ("stored", "on_the_fly"):
            return path
        if path != "auto":
            raise ValueError(f"unknown path {path!r}")
        n = M.n
        rows = -(-n // self.world_size)
        # fp64 from points: the float64 K (8 bytes per entry) or, by default, its 7 int8 slices; fp32: 4-byte
        # tiles or at most 3 int8 slices
        es = 8 if dtype == "fp64" else 4
        return "stored" if rows * n * es <= 0.5 * hbm_bytes(self.device) else "on_the_fly"

    def problem_for(self, M, dtype: str, path: str = "auto"):
        """(rld_problem, keepalive) for a dense matrix or a KernelMatrix."""
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {sorted(_DTYPES)}, got {dtype!r}")
        if isinstance(M, tuple) and len(M) == 2 and isinstance(M[0], KernelSpec):
            M = KernelMatrix(M[0], M[1])
        p = N.Problem()
        p.dtype = _DTYPES[dtype]
        if isinstance(M, KernelMatrix):
            spec = M.spec
            pts = M.points
            if _is_torch(pts):
                pts = pts.detach().to(dtype=_torch().float64).contiguous()
                mem, ptr = (N.DEVICE, pts.data_ptr()) if pts.is_cuda else (N.HOST, pts.numpy().ctypes.data)
            else:
                pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64))
                mem, ptr = N.HOST, pts.ctypes.data
            if pts.ndim != 2:
                raise ValueError("points must be an n x d array")
            p.source = N.SOURCE_POINTS
            p.path = N.PATH_STORED if self.resolve_path(M, dtype, path) == "stored" else N.PATH_ON_THE_FLY
            p.family = _FAMILIES[spec.family]
            p.n, p.d = int(pts.shape[0]), int(pts.shape[1])
            p.amplitude, p.length_scale, p.jitter = spec.amplitude, spec.length_scale, spec.jitter
            p.data, p.data_memory, p.data_dtype, p.ld = ptr, mem, N.FP64, 0
            self.after_torch()
            return p, pts
        if _is_torch(M):
            T = M.detach()
            if T.ndim != 2 or T.shape[0] != T.shape[1]:
                raise ValueError(f"expected a square matrix, got shape {tuple(T.shape)}")
            torch = _torch()
            if T.dtype not in (torch.float64, torch.float32):
                T = T.to(torch.float64)
            if T.stride(1) != 1:
                T = T.contiguous()
            p.source = N.SOURCE_DENSE
            p.n = int(T.shape[0])
            p.data_dtype = N.FP64 if T.dtype == torch.float64 else N.FP32
            p.ld = int(T.stride(0))
            if T.is_cuda:
                p.data, p.data_memory = T.data_ptr(), N.DEVICE
            else:
                a = T.numpy()
                p.data, p.data_memory = a.ctypes.data, N.HOST
                T = a
            self.after_torch()
            return p, T
        A = np.asarray(M)
        if A.ndim != 2 or A.shape[0] != A.shape[1]:
            raise ValueError(f"expected a square matrix, got shape {A.shape}")
        if A.dtype not in (np.float64, np.float32):
            A = A.astype(np.float64)
        if A.strides[1] != A.itemsize or A.strides[0] % A.itemsize:
            A = np.ascontiguousarray(A)
        p.source = N.SOURCE_DENSE
        p.n = int(A.shape[0])
        p.data_dtype = N.FP64 if A.dtype == np.float64 else N.FP32
        p.ld = A.strides[0] // A.itemsize
        p.data, p.data_memory = A.ctypes.data, N.HOST
        return p, A


_session = None
_session_lock = threading.Lock()
_local = threading.local()


class worker_session:
    """Context manager: this thread's calls use their own handle (own stream, workspace and
    resident problem) instead of the process-wide one, so independent estimates can run
    concurrently from several host threads (``harness.run_sweep(jobs=J)``).  One GPU only.
    ``sess=`` binds an existing session instead (a virtual-shard rank, ``parallel.py``); it is
    then not closed on exit."""

    def __init__(self, device: int | None = None, sess: "Session | None" = None):
        self.device = device
        self.sess = sess
        self.own = sess is None

    def __enter__(self):
        if self.sess is None:
            self.sess = Session(self.device)
        self.prev = getattr(_local, "sess", None)
        _local.sess = self.sess
        return self.sess

    def __exit__(self, *exc):
        _local.sess = self.prev
        if self.own:
            self.sess.handle.close()
        return False


def session() -> Session:
    """The calling thread's worker session if one is active, else the process-wide session
    (created on first use)."""
    mine = getattr(_local, "sess", None)
    if mine is not None:
        return mine
    global _session
    with _session_lock:
        if _session is None:
            rank, world, local = dist_world()
            nccl_id = None
            if world > 1:
                from .parallel import broadcast_nccl_id

                nccl_id = broadcast_nccl_id()
            _session = Session(local, rank, world, nccl_id)
        return _session


def reset_session():
    global _session
    with _session_lock:
        if _session is not None:
            _session.handle.close()
        _session = None
