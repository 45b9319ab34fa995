"""Build tests/emu/libhetpipe_emu.so: the REAL engine.cpp + capi.cpp host code
linked against a host emulation of the device kernels (TEST-ONLY; the product
library libhetpipe.so is built by paper_2005_14038_b200/build.py with nvcc)."""
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


def build():
    if os.path.exists(LIB) and all(os.path.getmtime(d) <= os.path.getmtime(LIB) for d in DEPS):
        return LIB
    cmd = ["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-pthread",
           "-I", HERE, "-o", LIB + ".tmp", *SRCS]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build())
