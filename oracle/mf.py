"""Matrix-free float64 K @ V for the CPU oracle (ctypes over ``oracle/libmfkv.so``).

TEST INFRASTRUCTURE ONLY -- the checker, never the product (see ``rstar_oracle.py``).
Only ``tests/``, ``__graft_entry__`` and ``bench.py``'s CPU legs use it.

``NativePointsOperator`` is a drop-in for ``rstar_oracle.PointsOperator``: the same
operator ``op(V) = K @ V`` of ``src/estimators.py:72`` / ``src/precond.py:186, 189``, with
K's rows generated from the points by the reference's ``build_covariance`` formula
(``src/kernels.py:40-46, 59-73``) inside OpenMP threads (``mf_kv.cpp``) instead of numpy
row blocks, so full BASELINE sizes (n = 65536 .. 2^20) run in minutes instead of days.
"""

from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "mf_kv.cpp"
LIBS = {"x86-64-v3": HERE / "libmfkv.so", "x86-64-v4": HERE / "libmfkv512.so"}
_FAMILY = {"rbf": 0, "matern52": 1}
_lib = None


def build(force: bool = False) -> Path:
    """g++ -O3 -fopenmp for x86-64-v3 (AVX2, any host here or on the GPU box) and x86-64-v4
    (AVX-512).  No fast-math and no FP contraction: the arithmetic is the one written."""
    for arch, lib_path in LIBS.items():
        if not force and lib_path.exists() and lib_path.stat().st_mtime >= SRC.stat().st_mtime:
            continue
        cmd = ["g++", "-O3", "-std=c++17", f"-march={arch}", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", str(SRC), "-o", str(lib_path), "-lmvec", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    return _pick()


def _pick() -> Path:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        flags = ""
    return LIBS["x86-64-v4"] if " avx512f " in flags and LIBS["x86-64-v4"].exists() else LIBS["x86-64-v3"]


def _blas():
    """(path, dgemm symbol, set-threads symbol) of an OpenBLAS in this environment (scipy's
    32-bit-integer build first: its thread count is separate from numpy's)."""
    import numpy  # noqa: F401

    site = Path(np.__file__).resolve().parent.parent
    for pat, dg, th in ((str(site / "scipy.libs" / "libscipy_openblas-*.so"), "scipy_cblas_dgemm",
                         "scipy_openblas_set_num_threads"),):
        hits = sorted(glob.glob(pat))
        if hits:
            return hits[0], dg, th
    return None, None, None


def lib():
    global _lib
    if _lib is None:
        path = _pick()
        if not path.exists():
            path = build()
        L = C.CDLL(str(path))
        L.mf_init.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p]
        L.mf_init.restype = C.c_int
        L.mf_kv.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_int64, C.c_int,
                            C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int,
                            C.c_int, C.c_double]
        L.mf_kv.restype = C.c_int
        L.mf_kblock.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_int64, C.c_int,
                                C.c_int64, C.c_int64, C.c_void_p]
        L.mf_kblock.restype = C.c_int
        L.mf_threads.restype = C.c_int
        L.mf_simd_width.restype = C.c_int
        path, dg, th = _blas()
        L.blas = bool(path and L.mf_init(path.encode(), dg.encode(), th.encode()))
        _lib = L
    return _lib


class NativePointsOperator:
    """op(V) = K @ V for V of shape (n,) or (n, m), K never materialised."""

    def __init__(self, family, amplitude, ell, jitter, X, rb=64, cb=1024, pert=0.0):
        self.args = (_FAMILY[family], float(amplitude), float(ell), float(jitter))
        self.family = family
        self.X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        self.n, self.d = self.X.shape
        self.rb, self.cb = rb, cb
        self.pert = float(pert)   # perturbation screen: K_ij (1 + pert h(i, j)), h symmetric in [-1, 1)
        self.calls = 0

    def diag(self):
        a = self.args[1]
        d = np.full(self.n, a * a + self.args[3])
        if self.pert:
            i = np.arange(self.n)
            d = d * (1.0 + self.pert * _sym_hash(i, i))
        return d

    def rows_product(self, Vrows, row0=0, rows=None):
        """Y (m x rows) = Vrows (m x n) K[row0:row0+rows, :]^T, vectors as rows."""
        Vrows = np.ascontiguousarray(np.asarray(Vrows, dtype=np.float64))
        m = Vrows.shape[0]
        rows = self.n - row0 if rows is None else rows
        Y = np.empty((m, rows))
        rc = lib().mf_kv(*self.args, self.X.ctypes.data, self.n, self.d, row0, rows, Vrows.ctypes.data, m,
                         Vrows.shape[1], Y.ctypes.data, rows, self.rb, self.cb, self.pert)
        if rc:
            raise ValueError("mf_kv: bad arguments")
        self.calls += 1
        return Y

    def __call__(self, V):
        V = np.asarray(V, dtype=np.float64)
        vec = V.ndim == 1
        if vec:
            V = V[:, None]
        out = self.rows_product(V.T).T            # vectors as rows: (m x n) -> (m x n)
        return out[:, 0] if vec else out

    def block(self, row0, rows):
        """K[row0:row0+rows, :] (tests)."""
        out = np.empty((rows, self.n))
        lib().mf_kblock(*self.args, self.X.ctypes.data, self.n, self.d, row0, rows, out.ctypes.data)
        return out


def _sym_hash(i, j):
    """numpy twin of mf_kv.cpp sym_hash (the diagonal of a perturbed K)."""
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    a, b = np.minimum(i, j), np.maximum(i, j)
    with np.errstate(over="ignore"):
        z = (a << np.uint64(32)) ^ b ^ np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0


def threads() -> int:
    return int(lib().mf_threads())
