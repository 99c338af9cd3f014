"""Build an A/B variant of librld.so: recompile one source with extra -D flags and link it
with the in-tree objects into scripts/librld_<name>.so (load it with RLD_LIB_PATH).

Usage: python scripts/build_variant.py <name> <source.cu> [-DFOO=1 ...]"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2405_03474_b200 import build as B  # noqa: E402

name, src, *defs = sys.argv[1:]
B.build()
nccl_inc, nccl_lib = B._nccl_dirs()
inc = [ROOT / "include", B.CSRC, nccl_inc, B.CUDA_HOME / "include"]
srcp = B.CSRC / src
obj = ROOT / "scripts" / f"_{name}_{srcp.stem}.o"
cmd = [B._nvcc(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
       *defs, *[f"-I{d}" for d in inc], "-c", str(srcp), "-o", str(obj)]
subprocess.run(cmd, check=True)
objs = [str(obj) if o.stem == srcp.stem else str(o) for o in sorted(B.OBJ.glob("*.o"))]
out = ROOT / "scripts" / f"librld_{name}.so"
cuda_lib = B.CUDA_HOME / "lib64"
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", str(out), f"-L{cuda_lib}",
                f"-L{nccl_lib}", "-lcublas", "-lcusolver", "-l:libnccl.so.2", f"-Xlinker=-rpath,{cuda_lib}",
                f"-Xlinker=-rpath,{nccl_lib}"], check=True)
obj.unlink()
print(out)
