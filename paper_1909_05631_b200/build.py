"""Build libsdnn.so (CUDA, sm_100a) and libsdnn_gen.so (host generators).

Everything is compiled in-tree with explicit nvcc/gcc command lines so the
shared objects travel with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsdnn.so"
GENLIB = PKG / "libsdnn_gen.so"
ARCH = "-gencode=arch=compute_100a,code=sm_100a"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _run(cmd):
    subprocess.run(cmd, check=True, cwd=str(ROOT))


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(s).stat().st_mtime > t for s in sources)


def build(force: bool = False, verbose: bool = False) -> None:
    gen_src = CSRC / "sdnn_gen.c"
    headers = [ROOT / "include" / "sdnn.h", ROOT / "include" / "sdnn_gen.h"]
    if force or _stale(GENLIB, [gen_src, *headers]):
        _run(["gcc", "-O3", "-std=gnu11", "-fPIC", "-shared", "-Wall", "-o", str(GENLIB),
              str(gen_src), "-lpthread"])
    cu = [CSRC / "sdnn.cu"]
    host_src = CSRC / "sdnn_host.c"
    deps = cu + [CSRC / "sdnn_kernels.cuh", gen_src, host_src, *headers]
    if force or _stale(LIB, deps):
        obj = PKG / "sdnn_gen.o"
        hobj = PKG / "sdnn_host.o"
        _run(["gcc", "-O3", "-std=gnu11", "-fPIC", "-c", "-o", str(obj), str(gen_src)])
        _run(["gcc", "-O3", "-std=gnu11", "-fPIC", "-mavx2", "-fopenmp", "-Wall", "-c", "-o", str(hobj),
              str(host_src)])
        cmd = [NVCC, ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-fopenmp,-mavx2",
               "-cudart", "static", "-o", str(LIB), *map(str, cu), str(obj), str(hobj), "-lpthread", "-lgomp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        _run(cmd)
        obj.unlink(missing_ok=True)
        hobj.unlink(missing_ok=True)


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
