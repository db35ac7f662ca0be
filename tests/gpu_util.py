"""Shared helpers for the GPU tests: run a config through the C-ABI library and through the
oracle on the same seeded events, and collect the compared outputs."""
from __future__ import annotations

import numpy as np

from gxin import configs

RINGBUF, PREFETCH_QUEUE = 27, 64


def outputs(engine, setup):
    """Compared outputs: every map's canonical dump; ring buffers as sorted multisets."""
    out = {}
    for (tenant, name), fd in sorted(setup.fds.items()):
        if engine.specs[fd][0] == RINGBUF:
            out[(tenant, name)] = tuple(engine.ringbuf_records(fd))
        elif engine.specs[fd][0] == PREFETCH_QUEUE:   # canonical content: the request set (F-2)
            out[(tenant, name)] = tuple(engine.prefetch_requests(fd))
        else:
            out[(tenant, name)] = engine.dump(fd)
    return out


def oracle_run(config, ev, threshold=None):
    from oracle.oracle import Oracle
    env = Oracle()
    s = configs.setup(env, config, threshold=threshold)
    r0 = env.run(ev, s.prog_arg)
    return env, s, r0


# "jit" lets the runtime pick the event ingest per launch (register loads below 2^22 events, so
# every small parity case); "jit_ring" forces the block-wide TMA ring the large bench batches use.
ENGINES = ("interp", "jit", "jit_ring")


def make_runtime(engine="jit", set_env=True):
    import os
    import paper_2512_12615_b200 as gx
    if set_env and engine == "jit_ring":
        os.environ["GX_JIT_INGEST"] = "ring"
    elif set_env:
        os.environ.pop("GX_JIT_INGEST", None)
    return gx.Runtime(0, engine=gx.GX_ENGINE_INTERP if engine == "interp" else gx.GX_ENGINE_JIT)


def gpu_run(config, ev, threshold=None, want_r0=True, runtime=None, engine="jit"):
    import torch

    rt = runtime or make_runtime(engine)
    s = configs.setup(rt, config, threshold=threshold)
    d_ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda()
    ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda") if want_r0 else None
    rt.run(d_ev, s.prog_arg, ret=ret)
    torch.cuda.synchronize()
    r0 = ret.cpu().numpy().view(np.uint64) if want_r0 else None
    return rt, s, r0


def first_diff(a: bytes, b: bytes):
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return i
    return min(len(a), len(b)) if len(a) != len(b) else -1
