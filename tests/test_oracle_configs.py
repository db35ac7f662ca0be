"""Pins for the oracle on the config programs.

Closed forms are numpy reductions (closed_forms.py); the paper-printed Fig 2 counts
(tests/golden/fig2_pin.txt); brute-force permutation invariance over all 5040 orders
of 7-event batches; shard (S3) and per-thread-shard (S4) invariance.
"""
import itertools
import os

import numpy as np
import pytest

from gxin import configs, gen, programs
from oracle.oracle import Oracle
import closed_forms as cf

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def oracle_run(config, ev, threshold=None, env=None, **kw):
    env = env or Oracle()
    s = configs.setup(env, config, threshold=threshold)
    r0 = env.run(ev, s.prog_arg, **kw)
    return env, s, r0


def test_p1_four_events_pin():
    """c.8: addr = 0x1000, 0x100000, 0x101008, 0xFFFFF000 -> counts[1]=1... (pages 1, 256, 257, 0xFFFFF)."""
    ev = gen.records(4, addr=np.array([0x1000, 0x100000, 0x101008, 0xFFFFF000], dtype=np.uint64))
    env, s, r0 = oracle_run("C1", ev)
    counts = env.array_u64(s.fds[(0, "counts")])
    # pages 0x1, 0x100, 0x101, 0xFFFFF -> keys 1, 0, 1, 255
    want = np.zeros(256, dtype=np.uint64)
    want[[1, 0, 1, 255]] += np.uint64(1)
    want[1] = 2
    assert (counts == want).all() and int(counts.sum()) == 4 and (r0 == 0).all()
    env2, s2, r02 = oracle_run("C1d", ev)
    assert env2.dump(s2.fds[(0, "counts")]) == counts.tobytes() and (r02 == 1).all()


@pytest.mark.parametrize("n", [1, 31, 33, 1000, 1 << 16])
def test_c1_closed_form(n):
    ev = configs.events("C1", configs.SEEDS["C1"], n)
    env, s, r0 = oracle_run("C1", ev)
    counts = env.array_u64(s.fds[(0, "counts")])
    assert (counts == cf.c1_counts(ev)).all()
    assert int(counts.sum()) == n                      # north star: counter totals = event count
    env2, s2, _ = oracle_run("C1d", ev)
    assert env2.dump(s2.fds[(0, "counts")]) == counts.tobytes()


def test_c2_closed_form():
    ev = configs.events("C2", configs.SEEDS["C2"], 1 << 16)
    env, s, r0 = oracle_run("C2", ev)
    hist, pt = cf.c2_expected(ev)
    assert (env.array_u64(s.fds[(0, "hist")]) == hist).all()
    assert (env.array_u64(s.fds[(0, "lane_pt")]) == pt).all()
    assert int(hist.sum()) == len(ev)


def test_fig2_pin():
    """SM 15 executes 382 threads, SM 6 only 3 (tests/golden/fig2_pin.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLD, "fig2_pin.txt")) if l[0].isdigit()]
    sm = np.concatenate([np.full(int(n), int(s)) for s, n in rows]).astype(np.uint16)
    rng = np.random.default_rng(0)
    ev = gen.records(len(sm), sm_id=sm, warp_id=rng.integers(0, 64, len(sm)).astype(np.uint8), size=4)
    env, s, _ = oracle_run("C2", ev)
    hist = env.array_u64(s.fds[(0, "hist")]).reshape(148, 64).sum(axis=1)
    assert int(hist[15]) == 382 and int(hist[6]) == 3
    assert round(int(hist[15]) / int(hist[6])) == 127


@pytest.mark.parametrize("T,want_rb", [(2, [(5, 2)]), (64, [])])
def test_p3_small_pin(T, want_rb):
    """c.8: pages 5, 5, 7, 5 -> hash {5:3, 7:1}; ringbuf {(5,T)} exactly once iff T <= 3."""
    ev = gen.records(4, addr=np.array([5, 5, 7, 5], dtype=np.uint64) << np.uint64(12))
    for order in itertools.permutations(range(4)):
        env, s, _ = oracle_run("C3", ev, threshold=T, order=np.array(order))
        assert {k: int(v[0]) for k, v in env.hash_items(s.fds[(0, "lfu")]).items()} == {5: 3, 7: 1}
        rb = env.ringbuf_records(s.fds[(0, "rb")])
        assert rb == [p.to_bytes(8, "little") + t.to_bytes(8, "little") for p, t in want_rb]


def test_c3_closed_form():
    ev = configs.events("C3", configs.SEEDS["C3"], 1 << 17)
    env, s, _ = oracle_run("C3", ev)
    table, rb = cf.c3_expected(ev, 64)
    got = {k: int(v[0]) for k, v in env.hash_items(s.fds[(0, "lfu")]).items()}
    assert got == table
    assert env.ringbuf_records(s.fds[(0, "rb")]) == rb
    st = env.stats()
    assert st["hash_full"] == 0 and st["ringbuf_drops"] == 0
    assert len(rb) > 0


def test_c4_closed_form():
    ev = configs.events("C4", configs.SEEDS["C4"], 1 << 16)
    env, s, r0 = oracle_run("C4", ev)
    want = cf.c4_expected(ev, gen.c4_bounds())
    assert (env.array_u64(s.fds[(0, "cstat")]) == want["cstat"]).all()
    got_hits = {k: int(v[0]) for k, v in env.hash_items(s.fds[(0, "list_hits")]).items()}
    assert got_hits == want["hits"]
    assert (env.array_u64(s.fds[(0, "list_bytes")]) == want["list_bytes"]).all()
    assert (env.array_u64(s.fds[(0, "scan_pt")]) == want["scan_pt"]).all()
    assert (r0 == want["r0"]).all()
    assert want["cstat"][0] > 0 and len(want["hits"]) > 10


def test_c5_per_tenant_closed_forms():
    ev = configs.events("C5", configs.SEEDS["C5"], 1 << 16)
    env, s, r0 = oracle_run("C5", ev)
    tenant = (ev["hook"] >> 8) & 0xFF
    st = env.stats()
    assert st["events_run"] == len(ev) and st["events_skipped"] == 0
    e0 = ev[tenant == 0]
    assert (env.array_u64(s.fds[(0, "counts")]) == cf.c1_counts(e0)).all()
    hist, pt = cf.c2_expected(ev[tenant == 1])
    assert (env.array_u64(s.fds[(1, "hist")]) == hist).all()
    assert (env.array_u64(s.fds[(1, "lane_pt")]) == pt).all()
    e2 = ev[tenant == 2]
    table, _ = cf.c3_expected(e2, 1 << 40)
    assert {k: int(v[0]) for k, v in env.hash_items(s.fds[(2, "lfu")]).items()} == table
    fault = e2[(e2["hook"] & 0xFF) == 2]
    want_rb = sorted(int(p >> np.uint64(12)).to_bytes(8, "little") + int(sm).to_bytes(8, "little")
                     for p, sm in zip(fault["addr"], fault["sm_id"]))
    assert env.ringbuf_records(s.fds[(2, "rb")]) == want_rb and len(want_rb) > 0
    w4 = cf.c4_expected(ev[tenant == 3], gen.c4_bounds())
    assert (env.array_u64(s.fds[(3, "list_bytes")]) == w4["list_bytes"]).all()
    assert (r0[tenant == 3] == w4["r0"]).all()


def test_unattached_events_skipped():
    ev = configs.events("C5", configs.SEEDS["C5"], 4096)
    ev["hook"][:100] = (ev["hook"][:100] & 0xFF) | (9 << 8)       # tenant 9: nothing attached
    env, s, _ = oracle_run("C5", ev)
    st = env.stats()
    assert st["events_skipped"] == 100 and st["events_run"] == 4096 - 100


@pytest.mark.parametrize("config,T", [("C1", None), ("C1d", None), ("C2", None), ("C3", 2), ("C4", None), ("C5", None)])
def test_permutation_invariance_bruteforce(config, T):
    """c.5: all 5040 orders of a 7-event batch give identical compared outputs (ORDER_INSENSITIVE)."""
    base = configs.events(config, configs.SEEDS[config], 7 * 32)[::32][:7].copy()
    if config == "C3":
        base["addr"] = (np.array([5, 5, 7, 5, 9, 9, 5], dtype=np.uint64) << np.uint64(12))
    ref_env = Oracle()
    s = configs.setup(ref_env, config, threshold=T)
    ref_r0 = ref_env.run(base, s.prog_arg)
    ref = _outputs(ref_env, s)
    perms = list(itertools.permutations(range(7)))
    if config in ("C3", "C5"):   # 32 MiB ringbuf / 2M-bucket hash per clone: every 10th order
        perms = perms[::10]
    fresh = Oracle()
    s2 = configs.setup(fresh, config, threshold=T)
    for order in perms:
        env = fresh.clone()
        r0 = env.run(base, s2.prog_arg, order=np.array(order))
        assert (r0 == ref_r0).all()
        assert _outputs(env, s2) == ref


def _outputs(env, s):
    out = []
    for (tenant, name), fd in sorted(s.fds.items()):
        if env.specs[fd][0] == 27:
            out.append(tuple(env.ringbuf_records(fd)))
        else:
            out.append(env.dump(fd))
    return out


@pytest.mark.parametrize("config", ["C1", "C2", "C4", "C5"])
def test_shards_equal_unsharded(config):
    """S3: for partition-insensitive programs `--shards G` gives the 1-shard result (c.5 Merge row)."""
    n = 1 << 14
    ev = configs.events(config, configs.SEEDS[config], n)
    ref_env, s, _ = oracle_run(config, ev)
    ref = _outputs(ref_env, s)
    for G in (2, 3, 8):
        init = Oracle()
        si = configs.setup(init, config)
        locals_ = [init.clone() for _ in range(G)]
        cuts = [(g * n // G) & ~31 for g in range(G)] + [n]
        for g, env in enumerate(locals_):
            env.run(ev[cuts[g]:cuts[g + 1]], si.prog_arg, index_base=cuts[g])
        assert init.merge(locals_) == 0
        assert _outputs(init, si) == ref
