"""In-tree build of libhvb200.so (sm_100a) — used by __graft_entry__.build().

nvcc compiles each .cu under csrc/ for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (so ncu source pages map back), then links one shared
library next to this file. Rebuilds only when a source is newer than the .so.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_obj"
LIB = PKG / "libhvb200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
    # exact IEEE fp64 everywhere (online trainer, discretizer): no FMA contraction
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v" if os.environ.get("HVB200_PTXAS_VERBOSE") else "-O3",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
]


CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-g", f"-I{ROOT / 'include'}", f"-I{CSRC}"]


def sources():
    """CUDA translation units (nvcc) plus host-only .cpp files (host compiler,
    for code that needs intrinsics nvcc's front end does not take)."""
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list((ROOT / "include").glob("*.h")) + [Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def _compile(src: Path) -> Path:
    out = OBJ / (src.stem + ".o")
    if src.suffix == ".cpp":
        cmd = [CXX, *CXX_FLAGS, "-c", str(src), "-o", str(out)]
    else:
        cmd = [NVCC, *ARCH, *NVCC_FLAGS, "-c", str(src), "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed for {src.name}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and os.environ.get("HVB200_PTXAS_VERBOSE"):
        sys.stderr.write(r.stderr)
    return out


def _obj_stale(src: Path) -> bool:
    """An object is rebuilt when it is missing or older than its source, any
    shared header (csrc/*.cuh|*.h, include/*.h) or this build script."""
    out = OBJ / (src.stem + ".o")
    if not out.exists():
        return True
    t = out.stat().st_mtime
    deps = [src, Path(__file__)] + [p for p in CSRC.glob("*") if p.suffix in (".cuh", ".h")]
    deps += list((ROOT / "include").glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    OBJ.mkdir(exist_ok=True)
    todo = [s for s in sources() if force or _obj_stale(s)]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(_compile, todo))
    objs = [OBJ / (s.stem + ".o") for s in sources()]
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-Xlinker", "-soname=libhvb200.so", "-o", str(tmp), *map(str, objs),
           "-lcudart_static", "-lrt", "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
