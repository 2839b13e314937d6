"""Build the in-tree sm_100a library `paper_2502_04093_b200/libipcomp_b200.so`.

nvcc compiles every csrc/*.cu and csrc/*.cpp for `-gencode arch=compute_100a,code=sm_100a`
with the floating-point flags that keep the kernels bit-exact with the reference's
`-ffp-contract=off` CPU build (CMakeLists.txt:25-27): no FMA contraction, IEEE division
and square root, no flush-to-zero.  Objects are rebuilt only when a source or header is
newer than the object.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libipcomp_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", *ARCH, "-O3", "-lineinfo", "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
           "-ftz=false", "--extended-lambda", "-Xcompiler", "-fPIC,-ffp-contract=off", f"-I{INCLUDE}"]
NVFLAGS += os.environ.get("IPCG_NVCC_EXTRA", "").split()  # dev: variant builds (tools/variants.sh)
PER_FILE: dict = {}  # per-file extra nvcc flags


def _newest_dep() -> float:
    deps = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return max(os.path.getmtime(p) for p in deps)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _newest_dep():
        return obj
    cmd = ["nvcc", *NVFLAGS, *PER_FILE.get(os.path.basename(src), []), "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = ["nvcc", *NVFLAGS, "-x", "cu", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_dep():
        return LIB
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    cmd = ["nvcc", "-shared", *ARCH, "-o", LIB, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
