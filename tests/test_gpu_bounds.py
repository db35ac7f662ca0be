"""Bounds checks of our own (SURVEY.md §4 layer 9 / §5; compute-sanitizer is disabled on this GPU
pool): the JIT's GX_JIT_BOUNDS=1 debug mode checks every map access against its map's device
allocation -- loads, stores and atomics through map-value pointers, per-thread physical words,
helper arguments through map-value pointers -- counting (and defusing) any that fall outside.
Every config and a slice of the differential fuzz run in that mode on both JIT ingests: results
still equal the oracle's and no access is out of bounds.  GX_JIT_BOUNDS=2 halves the checked
ranges, and then the checker must fire (its self-test)."""
import numpy as np
import pytest

from gxin import configs
from gpu_util import make_runtime, oracle_run, outputs
import fuzz_util as fu
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu


def _run(config, engine, n):
    import torch
    T = 2 if config == "C3" else None
    ev = configs.events(config, configs.SEEDS[config], n)
    env, so, r0o = oracle_run(config, ev, threshold=T)
    rt = make_runtime(engine)
    s = configs.setup(rt, config, threshold=T)
    ret = torch.zeros(n, dtype=torch.int64, device="cuda")
    rt.run(torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda(), s.prog_arg, ret=ret)
    torch.cuda.synchronize()
    st = rt.stats()
    same = (ret.cpu().numpy().view(np.uint64) == r0o).all() and outputs(rt, s) == outputs(env, so)
    rt.close()
    return same, st


@pytest.mark.parametrize("engine", ["jit", "jit_ring"])
@pytest.mark.parametrize("config", ["C1", "C1d", "C2", "C3", "C4", "C5", "C6"])
def test_configs_in_bounds(gpu, config, engine, monkeypatch):
    monkeypatch.setenv("GX_JIT_BOUNDS", "1")
    same, st = _run(config, engine, (1 << 16) + 37)
    assert same
    assert st["bounds_violations"] == 0


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_in_bounds(gpu, seed, monkeypatch):
    import torch
    monkeypatch.setenv("GX_JIT_BOUNDS", "1")
    texts, ev = fu.case(10_000 + seed)
    env = Oracle()
    fo, po = fu.setup(env, texts, 10_000 + seed)
    r0o = env.run(ev, po)
    rt = make_runtime("jit", set_env=False)
    fg, pg = fu.setup(rt, texts, 10_000 + seed)
    ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda")
    rt.run(torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda(), pg, ret=ret)
    torch.cuda.synchronize()
    og = fu.outputs(rt, fg, keep_stats=True)
    st = og.pop("_stats")
    assert (ret.cpu().numpy().view(np.uint64) == r0o).all()
    assert og == fu.outputs(env, fo)
    assert st["bounds_violations"] == 0
    rt.close()


@pytest.mark.parametrize("config", ["C1", "C2", "C4"])
def test_checker_fires_on_halved_ranges(gpu, config, monkeypatch):
    """Self-test: with every checked range halved, the accesses to the maps' upper halves (C1's keys
    128..255, C2's SMs >= 74, C4's lists >= 2048) are counted."""
    monkeypatch.setenv("GX_JIT_BOUNDS", "2")
    _, st = _run(config, "jit", (1 << 16) + 37)
    assert st["bounds_violations"] > 0
