"""Build libgroot_b200.so in-tree: nvcc for sm_100a only, -lineinfo, no JIT cache.

    python -m paper_2511_18297_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# GROOT_BUILD_TAG=x builds an experiment variant (objects in _build_x/, library
# libgroot_b200_x.so, selected at run time with GROOT_LIB); the product is untagged.
_TAG = os.environ.get("GROOT_BUILD_TAG", "")
OBJ = os.path.join(PKG, "_build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(PKG, "libgroot_b200" + (f"_{_TAG}" if _TAG else "") + ".so")
SOURCES = ["graph_build.cu", "forward.cu", "tile_plan.cu", "plan.cu", "partition_lp.cu", "train.cu", "capi.cpp", "runtime.cpp", "verify.cpp"]
HEADERS = ["common.cuh", "ptx.cuh", "tile_plan.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                  "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"),
                  "-I", CSRC]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _extra() -> list:
    # development knob, e.g. GROOT_NVCC_FLAGS=-DGROOT_TRACE_BUILD (timeline stamps)
    return os.environ.get("GROOT_NVCC_FLAGS", "").split()


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
           [os.path.join(ROOT, "include", "groot.h"), __file__]
    stamp = obj + ".flags"
    flags = " ".join(_extra())
    if not _stale(obj, deps) and os.path.exists(stamp) and open(stamp).read() == flags:
        return obj
    cmd = [nvcc()] + NVFLAGS + _extra() + ["-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(res.stderr)
    with open(stamp, "w") as f:
        f.write(flags)
    if verbose:
        print(f"[build] {src}", file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
