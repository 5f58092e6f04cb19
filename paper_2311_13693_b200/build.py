"""Build libxtsg.so (CUDA sm_100a + C ABI) in-tree.

Plain nvcc invocations (no torch JIT cache), so the .so lands next to the
sources and travels to the GPU box with the repo snapshot.
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
OBJ = PKG / "_build"
LIB = PKG / "libxtsg.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", str(ROOT / "include"),
    "-Xptxas", "-warn-spills",
]

CU_SOURCES = sorted(CSRC.glob("*.cu"))
CPP_SOURCES = sorted(CSRC.glob("*.cpp"))


def _needs(obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "xtsg.h"]
    jobs = []
    objs = []
    for src in CU_SOURCES + CPP_SOURCES:
        obj = OBJ / (src.stem + ".o")
        objs.append(obj)
        if force or _needs(obj, [src] + headers):
            if src.suffix == ".cu":
                cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
            else:
                cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off",
                       "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
                       "-c", str(src), "-o", str(obj)]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return r

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(run, jobs))
    if jobs or not LIB.exists() or force:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs),
               "-cudart", "static", "-lcuda"]
        run(cmd)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
