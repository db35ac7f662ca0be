"""Device-side event generation (libgxgen.so) -- INPUT GENERATION ONLY.

generate_device(config, seed, n, i0, n_total) -> torch.uint8 CUDA tensor (n, 32), the same
bytes gxin.gen.generate produces (checked by tests/test_gpu_parity.py::test_device_generator).
"""
from __future__ import annotations

import ctypes as C
import functools
import os
import subprocess

import numpy as np

from . import gen

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libgxgen.so")
SRC = os.path.join(_HERE, "gen_cuda.cu")


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        nvcc = "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc"
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


@functools.lru_cache(maxsize=None)
def _lib():
    L = C.CDLL(build())
    u64, vp = C.c_uint64, C.c_void_p
    L.gxgen_generate.argtypes = [C.c_int, u64, u64, u64, u64, vp, vp, vp, vp, vp, vp, vp]
    L.gxgen_generate.restype = C.c_int
    return L


@functools.lru_cache(maxsize=None)
def _tables(device: int):
    import torch
    dev = torch.device("cuda", device)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(dev)
    return (t(gen.sm_table()), t(gen.zipf_table(gen.NWEIGHT, 0.99)), t(gen.zipf_table(gen.NLISTS, 0.8)),
            t(gen.tenant_table()), t(gen.c4_bounds()))


def generate_device(config: str, seed: int, n: int, i0: int = 0, n_total: int | None = None, device: int = 0,
                    out=None, stream=None):
    import torch
    n_total = n if n_total is None else n_total
    if out is None:
        out = torch.empty((n, 32), dtype=torch.uint8, device=torch.device("cuda", device))
    tabs = _tables(device)
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
    from .configs import GEN_CONFIG
    config = GEN_CONFIG.get(config, config)
    rc = _lib().gxgen_generate(gen.CONFIG_ID[config], seed, i0, n, n_total, *[x.data_ptr() for x in tabs],
                               out.data_ptr(), s)
    if rc:
        raise RuntimeError(f"gxgen_generate failed: cuda error {rc}")
    return out
