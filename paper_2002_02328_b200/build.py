"""In-tree build of the sm_100a shared library ``_lib/libbd3mg_b200.so``.

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container; the resulting .so travels to the GPU box with the repo snapshot.
Translation units compile in parallel; a unit is rebuilt only when a source
or header is newer than its object.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# BD3MG_BUILD_DIR / BD3MG_DEFS: out-of-tree experiment builds (tuning variants)
LIBDIR = Path(os.environ.get("BD3MG_BUILD_DIR") or PKG / "_lib")
OBJDIR = LIBDIR / "obj"
LIB = LIBDIR / "libbd3mg_b200.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         *os.environ.get("BD3MG_DEFS", "").split()]
UNITS = ["capi.cu", "conv_f64.cu", "conv_f32.cu", "microbench.cu", "io.cu", "separable.cu", "sweep_pk.cu"]


def _deps() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + [INCLUDE / "bd3mg_b200.h"]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [src, *_deps()])


def _compile(unit: str, verbose: bool) -> Path:
    src = CSRC / unit
    obj = OBJDIR / (unit + ".o")
    if not _stale(obj, src):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {unit}:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJDIR.mkdir(parents=True, exist_ok=True)
    if force:
        for o in OBJDIR.glob("*.o"):
            o.unlink()
    with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        objs = list(ex.map(lambda u: _compile(u, verbose), UNITS))
    if LIB.exists() and all(LIB.stat().st_mtime >= o.stat().st_mtime for o in objs):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
