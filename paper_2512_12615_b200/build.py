"""Builds libgx.so (the C-ABI library: host runtime + verifier + sm_100a kernels) in-tree.

    python -m paper_2512_12615_b200.build      # or __graft_entry__.build()
Compiled with `nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3`, static cudart.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgx.so")
SOURCES = ["gx_exec.cu", "gx_maps.cu", "gx_runtime.cpp", "gx_verifier.cpp"]
HEADERS = ["gx_internal.h", "gx_device.cuh", "gx_verifier.h", os.path.join("..", "..", "include", "gx.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.exists(p) or p == "nvcc"):
            return p
    return "nvcc"


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES + HEADERS)


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    objs = []
    for src in SOURCES:
        obj = os.path.join("/tmp", f"gx_{os.getpid()}_{src}.o")
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c",
               os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        subprocess.check_call(cmd, cwd=CSRC)
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, LIB)
    for o in objs:
        os.unlink(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
