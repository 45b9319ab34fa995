"""Build libhetpipe.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2005_14038_b200.build
"""
from __future__ import annotations

import fcntl
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhetpipe.so")
SOURCES = ["kernels.cu", "engine.cpp", "engine_dist.cpp", "capi.cpp", "comm_nccl.cpp", "pipeline.cpp"]
HEADERS = ["tick_desc.h", "engine.h", "comm.h", os.path.join("..", "..", "include", "hetpipe.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-fmad=false",                 # no FMA contraction anywhere (reading Z10)
    "-Xcompiler", "-fPIC,-O2,-Wall",
    "-Xptxas", "-v",
]


# A/B variants (tuning experiments only): HP_BUILD_DEFINES="-DX=1 ..." and
# HP_BUILD_OUT=<path> build another copy that bench/tests load via HP_LIB.
if os.environ.get("HP_BUILD_OUT"):
    LIB = os.path.abspath(os.environ["HP_BUILD_OUT"])
NVCC_FLAGS += os.environ.get("HP_BUILD_DEFINES", "").split()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    # one builder at a time (parallel test workers share the tree)
    with open(LIB + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        return _build_locked(force, verbose)


def _build_locked(force: bool, verbose: bool) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-shared", "-o", LIB + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libhetpipe.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
