"""Differential fuzz: random verified programs x random event batches, the CUDA path (through the
C ABI) against the oracle, bit-exact (SURVEY.md §4 layer 5, §7 step 6; §8c c.1 / c.3).

gxin/fuzzprog.py draws programs over the whole executed subset -- every ALU/JMP/JMP32 op, MEMSX,
bounded loops, lane-varying branches, every STX ATOMIC op and width on stack / ARRAY / HASH /
per-thread values, XCHG / CMPXCHG on shared maps, map_update_elem ANY / NOEXIST / EXIST / bad flags
on ARRAY and HASH (every error branch), ringbuf output -- and batches whose results are order- and
shard-invariant by construction (checked on the oracle by tests/test_fuzz_oracle.py).  Each case
compares R0 per event, every map's canonical dump, ringbuf multisets and the compared stats.

Sizes: GX_FUZZ_CASES (default 2000 cases on the interpreter, a fifth of that on each JIT ingest);
the JIT cases compile in parallel threads (NVRTC runs without the GIL)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle.oracle import Oracle
import fuzz_util as fu
from gpu_util import make_runtime

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("GX_FUZZ_CASES", "2000"))
SEED0 = int(os.environ.get("GX_FUZZ_SEED0", "0"))    # extended campaigns: a fresh seed range


def _oracle(texts, ev, seed):
    env = Oracle()
    fds, prog = fu.setup(env, texts, seed)
    r0 = env.run(ev, prog)
    return r0, fu.outputs(env, fds)


def _gpu(texts, ev, seed, rt):
    import torch
    fds, prog = fu.setup(rt, texts, seed)
    d_ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda()
    ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda")
    rt.run(d_ev, prog, ret=ret)
    torch.cuda.synchronize()
    r0 = ret.cpu().numpy().view(np.uint64)
    return r0, fu.outputs(rt, fds, keep_stats=True)


def _check(seed, engine):
    texts, ev = fu.case(seed)
    r0o, oo = _oracle(texts, ev, seed)
    rt = make_runtime(engine, set_env=False)
    try:
        r0g, og = _gpu(texts, ev, seed, rt)
        split = og.pop("_stats")["divergent_steps"] if engine == "jit" else og.pop("_stats") and 0
    finally:
        rt.close()
    bad = np.nonzero(r0o != r0g)[0]
    errs = []
    if bad.size:
        errs.append(f"R0 differs at {bad[:6].tolist()}: oracle {[hex(int(x)) for x in r0o[bad[:3]]]} "
                    f"gpu {[hex(int(x)) for x in r0g[bad[:3]]]}")
    for k in oo:
        if oo[k] != og[k]:
            errs.append(f"{k}: {fu.first_diff(oo[k], og[k])}")
    if split:   # GX_JIT_UNIFORM_CHECK=1: a branch the divergence analysis called uniform split
        errs.append(f"{split} warp splits at GXF_UNIFORM branches")
    return seed, len(texts), errs, texts


def _run_cases(engine, seeds, threads):
    fails, n_progs = [], 0
    _check(seeds[0], engine)  # first call in this thread: driver / NVRTC entry points resolved once
    with ThreadPoolExecutor(max_workers=threads) as pool:
        for seed, npg, errs, texts in pool.map(lambda s: _check(s, engine), seeds):
            n_progs += npg
            if errs:
                fails.append((seed, errs, texts))
    assert not fails, (f"{len(fails)} of {len(seeds)} cases differ; first: seed {fails[0][0]}: {fails[0][1]}\n" +
                       "\n----\n".join(fails[0][2]))
    return n_progs


def test_fuzz_interp(gpu):
    os.environ.pop("GX_JIT_INGEST", None)
    n = _run_cases("interp", list(range(SEED0, SEED0 + N_CASES)), threads=8)
    print(f"interp: {N_CASES} cases, {n} programs byte-equal to the oracle")


def test_fuzz_jit(gpu):
    os.environ.pop("GX_JIT_INGEST", None)
    os.environ["GX_JIT_UNIFORM_CHECK"] = "1"   # ballot kept at GXF_UNIFORM branches, splits counted
    ncpu = len(os.sched_getaffinity(0))
    k = max(50, N_CASES // 5)
    try:
        n = _run_cases("jit", list(range(SEED0 + 10000, SEED0 + 10000 + k)), threads=max(4, ncpu))
    finally:
        os.environ.pop("GX_JIT_UNIFORM_CHECK", None)
    print(f"jit (register ingest): {k} cases, {n} programs byte-equal to the oracle, no split at a GXF_UNIFORM branch")


def test_fuzz_jit_ring(gpu):
    os.environ["GX_JIT_INGEST"] = "ring"
    try:
        ncpu = len(os.sched_getaffinity(0))
        k = max(50, N_CASES // 5)
        n = _run_cases("jit", list(range(SEED0 + 20000, SEED0 + 20000 + k)), threads=max(4, ncpu))
    finally:
        os.environ.pop("GX_JIT_INGEST", None)
    print(f"jit (TMA ring ingest): {k} cases, {n} programs byte-equal to the oracle")
