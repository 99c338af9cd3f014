"""Build the C-ABI library ``librld.so`` in-tree with nvcc for sm_100a.

Usage: ``python -m paper_2405_03474_b200.build [--force] [-j N]``.

Objects go to ``paper_2405_03474_b200/build/``; the shared library lands next
to this file so it travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "librld.so"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl  # type: ignore

        base = Path(list(nvidia.nccl.__path__)[0])
        inc, lib = base / "include", base / "lib"
        if (inc / "nccl.h").exists() and (lib / "libnccl.so.2").exists():
            return inc, lib
    except Exception:
        pass
    return Path("/usr/include"), Path("/usr/lib/x86_64-linux-gnu")


def _nvcc():
    nvcc = CUDA_HOME / "bin" / "nvcc"
    return str(nvcc) if nvcc.exists() else (shutil.which("nvcc") or "nvcc")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _compile(src: Path, inc_dirs, force: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    deps = [src] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "rld.h"]
    if not force and obj.exists() and all(obj.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return obj
    cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
           "-Xptxas", "-v" if os.environ.get("RLD_PTXAS_VERBOSE") else "-O3",
           *[f"-I{d}" for d in inc_dirs], "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if os.environ.get("RLD_PTXAS_VERBOSE"):
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, jobs: int | None = None) -> Path:
    OBJ.mkdir(exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    inc = [ROOT / "include", CSRC, nccl_inc, CUDA_HOME / "include"]
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, inc, force), srcs))
    if not force and LIB.exists() and all(LIB.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return LIB
    cuda_lib = CUDA_HOME / "lib64"
    cmd = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(LIB),
           f"-L{cuda_lib}", f"-L{nccl_lib}", "-lcublas", "-lcusolver", "-l:libnccl.so.2",
           f"-Xlinker=-rpath,{cuda_lib}", f"-Xlinker=-rpath,{nccl_lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args(argv)
    print(build(force=a.force, jobs=a.j))


if __name__ == "__main__":
    main()
