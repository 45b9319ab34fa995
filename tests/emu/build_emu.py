"""Build tests/emu/libhetpipe_emu.so: the REAL engine.cpp + capi.cpp host code
linked against a host emulation of the device kernels (TEST-ONLY; the product
library libhetpipe.so is built by paper_2005_14038_b200/build.py with nvcc)."""
import fcntl
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CSRC = os.path.join(ROOT, "paper_2005_14038_b200", "csrc")
LIB = os.path.join(HERE, "libhetpipe_emu.so")
SRCS = [os.path.join(CSRC, "engine.cpp"), os.path.join(CSRC, "engine_dist.cpp"),
        os.path.join(CSRC, "capi.cpp"),
        os.path.join(HERE, "emu_kernels.cpp"), os.path.join(HERE, "comm_emu.cpp"),
        os.path.join(CSRC, "pipeline.cpp")]
DEPS = SRCS + [os.path.join(CSRC, "engine.h"), os.path.join(CSRC, "tick_desc.h"),
               os.path.join(CSRC, "comm.h"),
               os.path.join(HERE, "cuda_runtime.h"), os.path.join(ROOT, "include", "hetpipe.h")]


ASAN_LIB = os.path.join(HERE, "libhetpipe_emu_asan.so")


def build(asan: bool = False):
    """The emulation library; asan=True: the same sources under AddressSanitizer
    (tests/test_asan_emu.py loads it into a subprocess with libasan preloaded)."""
    lib = ASAN_LIB if asan else LIB
    # one builder at a time (pytest-xdist workers share the tree)
    with open(lib + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        return _build_locked(lib, asan)


def _build_locked(lib, asan):
    if os.path.exists(lib) and all(os.path.getmtime(d) <= os.path.getmtime(lib) for d in DEPS):
        return lib
    flags = (["-O1", "-g", "-fsanitize=address", "-fno-omit-frame-pointer"] if asan else ["-O2"])
    cmd = ["g++", "-std=c++17", *flags, "-fPIC", "-shared", "-ffp-contract=off", "-pthread",
           "-I", HERE, "-o", lib + ".tmp", *SRCS]
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build())
