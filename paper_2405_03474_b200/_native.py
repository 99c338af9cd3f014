"""ctypes binding of ``librld.so`` (the C ABI declared in ``include/rld.h``).

Loading is strict: if the library is missing or does not export the ABI,
``load()`` raises -- there is no CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

# RLD_LIB_PATH: an alternative build of the same library (A/B measurements of kernel variants)
LIB_PATH = Path(os.environ.get("RLD_LIB_PATH") or (Path(__file__).resolve().parent / "librld.so"))

RLD_OK = 0
RLD_ERR_INVALID_ARGUMENT = 1
RLD_ERR_NOT_POSITIVE_DEFINITE = 2
RLD_ERR_SINGULAR_SHIFTED_SYSTEM = 3
RLD_ERR_RANK_DEFICIENT = 4
RLD_ERR_CUDA = 5
RLD_ERR_NCCL = 6
RLD_ERR_OUT_OF_MEMORY = 7
RLD_ERR_NOT_SUPPORTED = 8

FP64, FP32 = 0, 1
RBF, MATERN52 = 0, 1
SOURCE_DENSE, SOURCE_POINTS = 0, 1
PATH_STORED, PATH_ON_THE_FLY = 0, 1
HOST, DEVICE = 0, 1
RADEMACHER, GAUSSIAN, NORMAL_ORTHOGONAL = 0, 1, 2
MAX_PROBE_BLOCKS = 4
PRECOND_RAND_SVD, PRECOND_IDENTITY, PRECOND_DIAGONAL = 0, 1, 2
PRECOND_RAND_SVD_SCALED, PRECOND_PARTIAL_CHOLESKY, PRECOND_PARTIAL_CHOLESKY_SCALED = 3, 4, 5
PRECOND_TRUNC_SVD, PRECOND_TRUNC_SVD_SCALED, PRECOND_RANK_ONE = 6, 7, 8
ESTIMATOR_RSTAR, ESTIMATOR_SLQ = 0, 1
ABI_VERSION = 4
COMM_NCCL, COMM_THREADS = 0, 1

# every symbol include/rld.h declares
EXPORTS = (
    "rld_abi_version", "rld_create", "rld_destroy", "rld_last_error", "rld_logdet", "rld_prepare",
    "rld_logdet_resident", "rld_build_covariance", "rld_kv_apply", "rld_rademacher", "rld_exact_logdet", "rld_dense_cholesky", "rld_dense_eigh",
    "rld_nccl_unique_id", "rld_stream", "rld_normal", "rld_chi_radii", "rld_vgroup_create", "rld_vgroup_destroy",
    "rld_precond_build", "rld_precond_apply", "rld_slice_stats",
)
SOLVE_SQRT, SOLVE_SQRT_T, SOLVE = 0, 1, 2


class PrecondInfo(C.Structure):
    _fields_ = [("log_det", C.c_double), ("rank", C.c_int32), ("rank_kept", C.c_int32), ("attempts", C.c_int32),
                ("qr_fallback", C.c_int32), ("kernel_launches", C.c_int32), ("reserved", C.c_int32)]


class DeviceSet(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32), ("comm_kind", C.c_int32),
                ("nccl_id", C.c_void_p), ("group", C.c_void_p)]


class Problem(C.Structure):
    _fields_ = [("source", C.c_int32), ("path", C.c_int32), ("dtype", C.c_int32), ("family", C.c_int32),
                ("n", C.c_int64), ("d", C.c_int32), ("data_memory", C.c_int32), ("amplitude", C.c_double),
                ("length_scale", C.c_double), ("jitter", C.c_double), ("data", C.c_void_p),
                ("data_dtype", C.c_int32), ("reserved", C.c_int32), ("ld", C.c_int64)]


class Config(C.Structure):
    _fields_ = [("order", C.c_int32), ("num_probes", C.c_int32), ("lanczos_iters", C.c_int32),
                ("probe_kind", C.c_int32), ("precond_kind", C.c_int32), ("precond_rank", C.c_int32),
                ("precond_iters", C.c_int32), ("oversample", C.c_int32), ("diag_floor", C.c_double),
                ("keep_rtol", C.c_double), ("breakdown_rtol", C.c_double), ("orth_rtol", C.c_double),
                ("probe_key", C.c_uint64 * 2), ("omega_key", C.c_uint64 * 4), ("estimator", C.c_int32),
                ("reserved2", C.c_int32), ("precond_scale", C.c_double), ("precond_key", C.c_uint64 * 2),
                ("probe_block_keys", C.c_uint64 * 8)]


class Inputs(C.Structure):
    _fields_ = [("probes", C.c_void_p), ("omega0", C.c_void_p), ("omega1", C.c_void_p), ("memory", C.c_int32),
                ("reserved", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("value", C.c_double), ("logdet_P", C.c_double), ("trace_term", C.c_double),
                ("per_probe", C.POINTER(C.c_double)), ("wall_time", C.c_double), ("attempts", C.c_int32),
                ("rank_kept", C.c_int32), ("kv_products", C.c_int32), ("kernel_launches", C.c_int32),
                ("phase_ms", C.c_double * 8), ("clamped_eigs", C.c_int32), ("qr_fallback", C.c_int32)]


_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    """Load librld.so (raises if it is missing: the product has no CPU path)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2405_03474_b200.build` "
                               "(the estimator has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name in EXPORTS:
            getattr(lib, name)  # AttributeError if the ABI is incomplete
        H = C.c_void_p
        lib.rld_abi_version.restype = C.c_int
        lib.rld_create.argtypes = [C.POINTER(DeviceSet), C.POINTER(H)]
        lib.rld_destroy.argtypes = [H]
        lib.rld_destroy.restype = None
        lib.rld_last_error.argtypes = [H]
        lib.rld_last_error.restype = C.c_char_p
        lib.rld_logdet.argtypes = [H, C.POINTER(Problem), C.POINTER(Config), C.POINTER(Inputs), C.POINTER(Result)]
        lib.rld_prepare.argtypes = [H, C.POINTER(Problem)]
        lib.rld_logdet_resident.argtypes = [H, C.POINTER(Config), C.POINTER(Inputs), C.POINTER(Result)]
        lib.rld_build_covariance.argtypes = [H, C.POINTER(Problem), C.c_void_p, C.c_int32]
        lib.rld_kv_apply.argtypes = [H, C.c_int64, C.c_void_p, C.c_void_p]
        lib.rld_rademacher.argtypes = [H, C.POINTER(C.c_uint64 * 2), C.c_int64, C.c_int64, C.c_void_p]
        lib.rld_normal.argtypes = [H, C.POINTER(C.c_uint64 * 2), C.c_int64, C.c_int64, C.c_void_p]
        lib.rld_exact_logdet.argtypes = [H, C.POINTER(C.c_double)]
        lib.rld_slice_stats.argtypes = [H, C.POINTER(C.c_int64)]
        lib.rld_dense_cholesky.argtypes = [H, C.c_int32, C.c_void_p, C.POINTER(C.c_int32)]
        lib.rld_dense_eigh.argtypes = [H, C.c_int32, C.c_void_p, C.c_void_p]
        lib.rld_chi_radii.argtypes = [C.POINTER(C.c_uint64 * 2), C.c_uint64, C.c_int64, C.c_int64, C.c_void_p]
        lib.rld_nccl_unique_id.argtypes = [C.c_void_p]
        lib.rld_stream.argtypes = [H]
        lib.rld_stream.restype = C.c_void_p
        lib.rld_precond_build.argtypes = [H, C.POINTER(Config), C.POINTER(Inputs), C.POINTER(PrecondInfo)]
        lib.rld_precond_apply.argtypes = [H, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p]
        lib.rld_vgroup_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
        lib.rld_vgroup_destroy.argtypes = [C.c_void_p]
        lib.rld_vgroup_destroy.restype = None
        for name in EXPORTS:
            if name not in ("rld_abi_version", "rld_destroy", "rld_last_error", "rld_stream", "rld_vgroup_destroy"):
                getattr(lib, name).restype = C.c_int
        if lib.rld_abi_version() != ABI_VERSION:
            raise RuntimeError("librld.so ABI version mismatch")
        _lib = lib
        return lib


class Handle:
    """One GPU (one row shard) bound to a librld handle."""

    def __init__(self, device: int = 0, rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None,
                 group: "VirtualGroup | None" = None):
        self.lib = load()
        self._h = C.c_void_p()
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.group = group   # keeps the group alive while this handle uses it
        ds = DeviceSet(device, rank, world_size, COMM_THREADS if group is not None else COMM_NCCL,
                       C.cast(self._id, C.c_void_p) if self._id is not None else None,
                       group.ptr if group is not None else None)
        self.check(self.lib.rld_create(C.byref(ds), C.byref(self._h)), "rld_create")
        self.device, self.rank, self.world_size = device, rank, world_size

    def close(self):
        if self._h:
            self.lib.rld_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ptr(self):
        return self._h

    @property
    def stream(self) -> int:
        """cudaStream_t of the handle (for torch.cuda.ExternalStream)."""
        return int(self.lib.rld_stream(self._h) or 0)

    def last_error(self) -> str:
        msg = self.lib.rld_last_error(self._h) if self._h else b"no handle"
        return msg.decode(errors="replace") if msg else ""

    def check(self, rc: int, what: str):
        if rc == RLD_OK:
            return
        raise_status(rc, f"{what}: {self.last_error() if self._h else ''}")


class VirtualGroup:
    """rld_vgroup: G ranks of one process sharing host-barrier collectives (RLD_COMM_THREADS)."""

    def __init__(self, world_size: int):
        self.lib = load()
        self._g = C.c_void_p()
        rc = self.lib.rld_vgroup_create(int(world_size), C.byref(self._g))
        if rc != RLD_OK:
            raise_status(rc, "rld_vgroup_create")
        self.world_size = int(world_size)

    @property
    def ptr(self):
        return self._g

    def close(self):
        if self._g:
            self.lib.rld_vgroup_destroy(self._g)
            self._g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def raise_status(rc: int, msg: str):
    """Map a status code onto the reference's exception types (src/linalg.py:24-33)."""
    from .linalg import NotPositiveDefinite, RankDeficient, SingularShiftedSystem

    if rc == RLD_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == RLD_ERR_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefinite(msg)
    if rc == RLD_ERR_SINGULAR_SHIFTED_SYSTEM:
        raise SingularShiftedSystem(msg)
    if rc == RLD_ERR_RANK_DEFICIENT:
        raise RankDeficient(msg)
    if rc == RLD_ERR_NOT_SUPPORTED:
        raise NotImplementedError(msg)
    if rc == RLD_ERR_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise RuntimeError(f"rld status {rc}: {msg}")
