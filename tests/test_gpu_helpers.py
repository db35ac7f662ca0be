"""Named GPU tests for the helper and atomic paths the configs never reach, each against the oracle
(SURVEY.md §8c O5/O6, c.3 S1, c.5 'Warp aggregation' row):

* test_warp_aggregation_bruteforce -- every active mask of 8 lanes x every key-collision pattern of
  the active lanes (all set partitions: Bell(9) = 21147 records), plus whole warps whose first 8
  lanes take every partition; every map atomic (ADD/OR/AND/XOR with FETCH and without, XCHG,
  CMPXCHG; W and DW) on ARRAY values.  Keys are record-local, so the oracle's sequential order
  inside a record is the one correct answer: R0 (the fetched values) and the map must match
  bit-exactly -- PAPER.md:286 "preserving eBPF's scalar semantics" under warp aggregation.
* test_update_array_paths -- bpf_map_update_elem on an ARRAY: ANY / EXIST / NOEXIST (-EEXIST),
  key >= max_entries (-E2BIG), flags 3 (-EINVAL), colliding keys in a record.
* test_hash_update_paths -- HASH update ANY / EXIST overwrites of live slots, NOEXIST on present
  keys, EXIST on absent keys (-ENOENT), then a lookup batch reading every value back.
* test_hash_full_exact -- the capacity is exact on the GPU: more distinct inserts than
  max_entries fill the map to exactly max_entries (hash_full = the rest); a full map refuses
  every insert; a hot-key insert storm at the boundary refuses nothing.
* test_ringbuf_overflow_gpu -- -EAGAIN and the drop count when the ring fills.
"""
import numpy as np
import pytest

from gxin import asm, gen
from oracle.oracle import Oracle
from gpu_util import ENGINES, make_runtime

pytestmark = pytest.mark.gpu

ARRAY, HASH, RINGBUF = 2, 1, 27


def set_partitions(n):
    """All set partitions of n elements as restricted growth strings (class id per element)."""
    if n == 0:
        yield ()
        return
    def rec(prefix, mx):
        if len(prefix) == n:
            yield tuple(prefix)
            return
        for c in range(mx + 2):
            yield from rec(prefix + [c], max(mx, c))
    yield from rec([0], 0)


def aggregation_events(seed):
    """Records: (A) for every mask of lanes 0..7 and every partition of its active lanes, lanes in
    the mask run (tenant 0) with keys record*8 + class, the rest are skipped (tenant 1);
    (B) whole warps: lanes 0..7 take every partition of 8, lanes 8..31 a unique key each;
    (C) whole warps on one key.  Returns the events and the number of keys used."""
    recs = []
    for mask in range(256):
        act = [l for l in range(8) if mask >> l & 1]
        for part in set_partitions(len(act)):
            cls = {l: c for l, c in zip(act, part)}
            recs.append(("A", cls))
    for part in set_partitions(8):
        recs.append(("B", dict(enumerate(part))))
    for _ in range(64):
        recs.append(("C", None))
    n = 32 * len(recs)
    key = np.zeros(n, dtype=np.uint64)
    ten = np.ones(n, dtype=np.uint32)
    for r, (kind, cls) in enumerate(recs):
        base = r * 32
        if kind == "A":
            for l, c in cls.items():
                key[base + l] = base + c
                ten[base + l] = 0
        elif kind == "B":
            for l in range(32):
                key[base + l] = base + (cls[l] if l < 8 else l)
            ten[base:base + 32] = 0
        else:
            key[base:base + 32] = base
            ten[base:base + 32] = 0
    rng = np.random.default_rng(seed)
    ev = gen.records(n, addr=key, ts=rng.integers(0, 1 << 64, n, dtype=np.uint64), hook=(ten << 8).astype(np.uint32))
    return ev, n


AGG_OPS = ([f"atomic_fetch_{op}{w}" for op in ("add", "or", "and", "xor") for w in ("64", "32")] +
           [f"atomic_{op}{w}" for op in ("add", "or", "and", "xor") for w in ("64", "32")] +
           ["xchg64", "xchg32", "cmpxchg64", "cmpxchg32"])


def agg_program(op):
    # key = addr (record-local); operand = ts; W ops hit the low or the high half by (ts >> 40) & 1
    w32 = op.endswith("32")
    lines = ["mov64 r6, r1", "ldxdw r2, [r6+0]", "stxw [r10-4], r2", "lddw r1, map:m", "mov64 r2, r10",
             "add64 r2, -4", "call 1", "jeq r0, 0, out", "ldxdw r7, [r6+8]"]
    if w32:
        lines += ["mov64 r3, r7", "rsh64 r3, 40", "and64 r3, 1", "lsh64 r3, 2", "add64 r0, r3"]
    if op.startswith("cmpxchg"):
        # compare value and new value from a 2-bit alphabet so equal compares happen
        lines += ["mov64 r8, r7", "and64 r8, 3", "rsh64 r7, 2", "and64 r7, 3", "mov64 r9, r0", "mov64 r0, r8",
                  f"{op} [r9+0], r7", "exit"]
    else:
        lines += [f"{op} [r0+0], r7", "mov64 r0, r7", "exit"]
    lines += ["out:", "mov64 r0, 0", "exit"]
    return "\n".join(lines)


def _agg_case(engine, op, ev, n_keys, seed):
    import torch
    out = {}
    rng = np.random.default_rng(seed)
    vals = rng.integers(0, 1 << 64, n_keys, dtype=np.uint64)
    if op.startswith("cmpxchg"):
        vals &= np.uint64(0x0000000300000003)
    keys = np.arange(n_keys, dtype=np.uint32)
    for side in ("oracle", "gpu"):
        eng = Oracle() if side == "oracle" else make_runtime(engine)
        fd = eng.create_map(ARRAY, 4, 8, n_keys)
        assert eng.update_many(fd, keys.tobytes(), vals.tobytes(), n_keys) == 0
        p = eng.load_prog(asm.assemble(agg_program(op), {"m": fd}))
        eng.attach(p, 0, 0)
        if side == "oracle":
            r0 = eng.run(ev, -1)
        else:
            d_ev = torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda()
            ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda")
            eng.run(d_ev, -1, ret=ret)
            torch.cuda.synchronize()
            r0 = ret.cpu().numpy().view(np.uint64)
        st = eng.stats()
        out[side] = (r0, eng.dump(fd), st["events_run"], st["events_skipped"])
    return out


@pytest.mark.parametrize("engine", ENGINES)
def test_warp_aggregation_bruteforce(gpu, engine):
    ev, n = aggregation_events(7)
    assert n // 32 == 21147 + 4140 + 64
    for k, op in enumerate(AGG_OPS):
        o = _agg_case(engine, op, ev, n, 100 + k)
        (r0o, mo, ro, so), (r0g, mg, rg, sg) = o["oracle"], o["gpu"]
        bad = np.nonzero(r0o != r0g)[0]
        assert bad.size == 0, (engine, op, "R0 differs at", bad[:6], r0o[bad[:3]], r0g[bad[:3]])
        assert mo == mg, (engine, op, "map differs")
        assert (ro, so) == (rg, sg), (engine, op, (ro, so), (rg, sg))


UPD_ARRAY = """
    mov64 r6, r1
    ldxdw r2, [r6+0]
    stxw [r10-4], r2          ; key (record-local, colliding inside records; >= max_entries for some)
    ldxdw r3, [r6+8]
    stxdw [r10-16], r3        ; value = ts
    lddw r1, map:a
    mov64 r2, r10
    add64 r2, -4
    mov64 r3, r10
    add64 r3, -16
    ldxw r4, [r6+28]          ; flags from ctx.size: 0 ANY, 1 NOEXIST, 2 EXIST, 3 invalid
    call 2
    exit
"""


def _run_both(engine, text, maps, ev, init=None, prog_ret=True, batches=1, texts2=None):
    """Runs `text` over ev on the oracle and the GPU; returns {side: (r0, dumps, stats)}."""
    import torch
    res = {}
    for side in ("oracle", "gpu"):
        eng = Oracle() if side == "oracle" else make_runtime(engine)
        fds = {name: eng.create_map(*spec) for name, spec in maps.items()}
        for name, (keys, vals, ks, vs) in (init or {}).items():
            assert eng.update_many(fds[name], keys, vals, len(keys) // ks) == 0
        r0s = []
        for t in [text] + (texts2 or []):
            p = eng.load_prog(asm.assemble(t, fds))
            if side == "oracle":
                r0s.append(eng.run(ev, p))
            else:
                d_ev = torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda()
                ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda")
                eng.run(d_ev, p, ret=ret)
                torch.cuda.synchronize()
                r0s.append(ret.cpu().numpy().view(np.uint64))
        dumps = {}
        for name, fd in fds.items():
            if maps[name][0] == RINGBUF:
                dumps[name] = tuple(eng.ringbuf_records(fd))
            else:
                dumps[name] = eng.dump(fd)
        st = eng.stats()
        res[side] = (r0s, dumps, {k: st[k] for k in ("events_run", "events_skipped", "ringbuf_drops", "hash_full")})
    return res


def _assert_same(res, what):
    (r0o, do, so), (r0g, dg, sg) = res["oracle"], res["gpu"]
    for k, (a, b) in enumerate(zip(r0o, r0g)):
        bad = np.nonzero(a != b)[0]
        assert bad.size == 0, (what, f"batch {k} R0 differs at", bad[:6], a[bad[:3]], b[bad[:3]])
    for name in do:
        assert do[name] == dg[name], (what, name)
    assert so == sg, (what, so, sg)


@pytest.mark.parametrize("engine", ENGINES)
def test_update_array_paths(gpu, engine):
    n = 32 * 300 + 7
    rng = np.random.default_rng(3)
    rec = np.arange(n) >> 5
    key = (rec * 4 + rng.integers(0, 4, n)).astype(np.uint64)       # 4 keys per record, collisions
    flags = rng.integers(0, 4, n).astype(np.uint32)
    flags[: 32 * 100] = 0                                             # whole records of ANY
    flags[32 * 100: 32 * 150] = 2                                     # and of EXIST
    ev = gen.records(n, addr=key, ts=rng.integers(0, 1 << 64, n, dtype=np.uint64), size=flags)
    maps = {"a": (ARRAY, 4, 8, 1000)}                                 # keys up to 1199: -E2BIG above 999
    res = _run_both(engine, UPD_ARRAY, maps, ev)
    _assert_same(res, "update ARRAY")
    r0 = res["oracle"][0][0].view(np.int64)
    assert {0, -7, -17, -22} <= set(r0.tolist())


UPD_HASH = """
    mov64 r6, r1
    ldxdw r2, [r6+0]
    stxdw [r10-8], r2
    ldxdw r3, [r6+8]
    stxdw [r10-16], r3
    lddw r1, map:h
    mov64 r2, r10
    add64 r2, -8
    mov64 r3, r10
    add64 r3, -16
    mov64 r4, FLAGS
    call 2
    exit
"""
READ_HASH = """
    ldxdw r2, [r1+0]
    stxdw [r10-8], r2
    lddw r1, map:h
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, none
    ldxdw r0, [r0+0]
    exit
none:
    mov64 r0, 0xdead
    exit
"""


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("flags", [0, 1, 2])
def test_hash_update_paths(gpu, engine, flags):
    n = 32 * 256 + 19
    rng = np.random.default_rng(11 + flags)
    rec = np.arange(n) >> 5
    key = (rec * 8 + rng.integers(0, 8, n)).astype(np.uint64)      # record-local keys, collisions
    key[32 * 10: 32 * 20] = (np.arange(32 * 10, 32 * 20) >> 5) * 8  # whole records on one key
    ev = gen.records(n, addr=key, ts=rng.integers(0, 1 << 64, n, dtype=np.uint64))
    present = np.unique(key)[::2].astype(np.uint64)                   # half the keys live before the batch
    init = {"h": (present.tobytes(), rng.integers(0, 1 << 64, len(present), dtype=np.uint64).tobytes(), 8, 8)}
    maps = {"h": (HASH, 8, 8, 4096)}
    res = _run_both(engine, UPD_HASH.replace("FLAGS", str(flags)), maps, ev, init=init, texts2=[READ_HASH])
    _assert_same(res, f"update HASH flags={flags}")


FILL_HASH = UPD_HASH.replace("FLAGS", "0")


@pytest.mark.parametrize("engine", ENGINES)
def test_hash_full_exact(gpu, engine):
    import torch
    # (1) 3000 distinct keys into max_entries = 1000: exactly 1000 live, hash_full = 2000
    n = 3000
    ev = gen.records(n, addr=np.arange(1, n + 1, dtype=np.uint64) * 7919, ts=np.arange(n, dtype=np.uint64))
    rt = make_runtime(engine)
    fd = rt.create_map(HASH, 8, 8, 1000)
    p = rt.load_prog(asm.assemble(FILL_HASH, {"h": fd}))
    ret = torch.zeros(n, dtype=torch.int64, device="cuda")
    rt.run(torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda(), p, ret=ret)
    torch.cuda.synchronize()
    r0 = ret.cpu().numpy()
    items = rt.hash_items(fd)
    assert len(items) == 1000 and int((r0 == 0).sum()) == 1000 and int((r0 == -7).sum()) == 2000
    assert rt.stats()["hash_full"] == 2000
    for k, v in items.items():                       # every live entry is an insert that succeeded
        i = k // 7919 - 1
        assert r0[i] == 0 and int(v[0]) == i
    # (2) the full map refuses every further insert of a new key, overwrites of live keys succeed
    ev2 = gen.records(64, addr=np.arange(5000, 5064, dtype=np.uint64) * 7919 + 1, ts=1)
    ret2 = torch.zeros(64, dtype=torch.int64, device="cuda")
    rt.run(torch.from_numpy(ev2.view(np.uint8).reshape(-1, 32)).cuda(), p, ret=ret2)
    torch.cuda.synchronize()
    assert (ret2.cpu().numpy() == -7).all() and len(rt.hash_items(fd)) == 1000
    rt.close()
    # (3) boundary storm: 1000 keys into max_entries = 1000, each key inserted by ~64 events spread
    # over many warps at once -- no insert may be refused (reservations are exact)
    n = 64000
    rng = np.random.default_rng(5)
    keys = (rng.permutation(n) % 1000 + 1).astype(np.uint64)
    ev3 = gen.records(n, addr=keys, ts=7)
    rt = make_runtime(engine)
    fd = rt.create_map(HASH, 8, 8, 1000)
    p = rt.load_prog(asm.assemble(FILL_HASH, {"h": fd}))
    ret3 = torch.zeros(n, dtype=torch.int64, device="cuda")
    rt.run(torch.from_numpy(ev3.view(np.uint8).reshape(-1, 32)).cuda(), p, ret=ret3)
    torch.cuda.synchronize()
    assert (ret3.cpu().numpy() == 0).all() and rt.stats()["hash_full"] == 0
    assert sorted(rt.hash_items(fd)) == list(range(1, 1001))
    rt.close()


RB_OUT = """
    ldxdw r2, [r1+0]
    stxdw [r10-16], r2
    ldxdw r2, [r1+8]
    stxdw [r10-8], r2
    lddw r1, map:rb
    mov64 r2, r10
    add64 r2, -16
    mov64 r3, 16
    mov64 r4, 0
    call 130
    exit
"""


@pytest.mark.parametrize("engine", ENGINES)
def test_ringbuf_overflow_gpu(gpu, engine):
    """4096-B ring, 24-B records (8-B header + 16-B payload): 170 fit, every other event gets
    -EAGAIN and is counted as a drop (SURVEY.md §8c c.8 'Ringbuf overflow'; which events win is
    order-dependent, so the counts and the payload set are compared)."""
    n = 1000
    ev = gen.records(n, addr=np.arange(n, dtype=np.uint64), ts=np.arange(n, dtype=np.uint64) * 3)
    res = _run_both(engine, RB_OUT, {"rb": (RINGBUF, 0, 0, 4096)}, ev)
    (r0o, do, so), (r0g, dg, sg) = res["oracle"], res["gpu"]
    a, b = r0o[0].view(np.int64), r0g[0].view(np.int64)
    assert int((a == 0).sum()) == int((b == 0).sum()) == 170
    assert int((b == -11).sum()) == 830 and so["ringbuf_drops"] == sg["ringbuf_drops"] == 830
    recs = dg["rb"]
    assert len(recs) == 170
    ok_idx = np.nonzero(b == 0)[0]
    want = sorted(int(i).to_bytes(8, "little") + int(3 * i).to_bytes(8, "little") for i in ok_idx)
    assert list(recs) == want
