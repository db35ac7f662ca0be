"""Oracle pins for the f2 row: the gdev_mem_prefetch helper and the prefetch
queue ("Request prefetch, triggers handler in host driver"; F-1..F-3).
Closed forms (page arithmetic, the stride policy's request set), error cases and capacity."""
import numpy as np
import pytest

from gxin import asm, configs, gen
from oracle.oracle import ARRAY, PREFETCH_QUEUE, Oracle

CALL = """
    ldxdw r2, [r1+0]
    ldxdw r3, [r1+8]
    lddw r1, map:q
    call 1000
    exit
"""


def _one(addr, length, cap=64):
    env = Oracle()
    q = env.create_map(PREFETCH_QUEUE, 0, 0, cap)
    ev = gen.records(1, addr=np.uint64(addr), ts=np.uint64(length))
    r0 = env.run(ev, env.load_prog(asm.assemble(CALL, {"q": q})))
    return int(r0[0]), env.prefetch_requests(q), env


@pytest.mark.parametrize("addr,length,want", [
    (0x1000, 1, (1, 1)),                    # one byte -> its page
    (0x1fff, 2, (1, 2)),                    # straddles a page boundary
    (0x200000, 2 << 20, (512, 512)),        # one aligned 2-MiB chunk
    (0x200001, 2 << 20, (512, 513)),        # unaligned 2 MiB spans 513 pages
    (0, 4096, (0, 1)),
])
def test_prefetch_page_math(addr, length, want):
    r0, req, _ = _one(addr, length)
    assert r0 == 0 and req == [want]


@pytest.mark.parametrize("addr,length", [(0x1000, 0), (0x1000, (2 << 20) + 1), (2**64 - 4096, 8192)])
def test_prefetch_invalid(addr, length):
    r0, req, env = _one(addr, length)
    assert r0 == 2**64 - 22 and req == []          # -EINVAL, nothing queued
    assert env.stats()["helper_errors"] == 1


def test_prefetch_queue_full():
    env = Oracle()
    q = env.create_map(PREFETCH_QUEUE, 0, 0, 64)
    ev = gen.records(65, addr=np.arange(65, dtype=np.uint64) * 4096, ts=np.uint64(1))
    r0 = env.run(ev, env.load_prog(asm.assemble(CALL, {"q": q})))
    assert (r0[:64] == 0).all() and int(r0[64]) == 2**64 - 11   # -EAGAIN for the 65th
    assert env.stats()["ringbuf_drops"] == 1
    assert len(env.prefetch_requests(q)) == 64
    env.prefetch_reset(q)
    assert env.prefetch_requests(q) == []


def test_prefetch_is_a_set():
    """Identical requests collapse (prefetch is idempotent, F-2); the call count is kept."""
    env = Oracle()
    q = env.create_map(PREFETCH_QUEUE, 0, 0, 64)
    ev = gen.records(10, addr=np.uint64(0x5000), ts=np.uint64(100))
    env.run(ev, env.load_prog(asm.assemble(CALL, {"q": q})))
    assert env.prefetch_requests(q) == [(5, 1)] and env.last_pfq_calls == 10


@pytest.mark.parametrize("bad", [(PREFETCH_QUEUE, 0, 0, 32), (PREFETCH_QUEUE, 0, 0, 100), (PREFETCH_QUEUE, 4, 8, 64)])
def test_prefetch_queue_spec(bad):
    with pytest.raises(OSError):
        Oracle().create_map(*bad)


def test_c6_stride_policy_closed_form():
    """P6 over the C3 page trace: requests = {(page(addr) + 1, 16) : addr in a page's last 128 B}."""
    ev = configs.events("C6", configs.SEEDS["C6"], 1 << 16)
    env = Oracle()
    s = configs.setup(env, "C6")
    env.run(ev, s.prog_arg)
    hit = (ev["addr"] & np.uint64(4095)) >= 3968
    want = sorted({(int(a >> np.uint64(12)) + 1, 16) for a in ev["addr"][hit]})
    assert env.prefetch_requests(s.fds[(0, "pfq")]) == want
    assert env.last_pfq_calls == int(hit.sum())
    assert int(env.array_u64(s.fds[(0, "pstat")])[0]) == int(hit.sum())


def test_prefetch_merge_is_union():
    """S3 merge of two shards' queues = the union (each rank's daemon drains its own queue)."""
    ev = configs.events("C6", configs.SEEDS["C6"], 1 << 14)
    env = Oracle()
    s = configs.setup(env, "C6")
    whole = env.clone()
    whole.run(ev, s.prog_arg)
    a, b = env.clone(), env.clone()
    a.run(ev[: len(ev) // 2], s.prog_arg)
    b.run(ev[len(ev) // 2:], s.prog_arg, index_base=len(ev) // 2)
    assert env.merge([a, b]) == 0
    q = s.fds[(0, "pfq")]
    assert env.prefetch_requests(q) == whole.prefetch_requests(q)


# ---- gdev_prefetch_l2 (PAPER.md:342 device-side prefetch.global.L2; F-7): a hint whose
# only observable output is R0 -- the error cases below are read off the helper's definition
L2CALL = """
    ldxdw r2, [r1+0]
    ldxdw r3, [r1+8]
    lddw r1, map:region
    call 1001
    exit
"""
BASE, SPAN = 0x7F00_0000_0000, 1 << 20


@pytest.mark.parametrize("addr,length,want", [
    (BASE, 1, 0),                             # first byte
    (BASE + SPAN - 1, 1, 0),                  # last byte
    (BASE + SPAN - 65536, 65536, 0),          # ends exactly at the region end, maximum length
    (BASE + 100, 65537, -22),                 # longer than 64 KiB
    (BASE + 100, 0, -22),                     # empty
    (BASE - 1, 2, -14),                       # starts one byte before the region
    (BASE + SPAN - 1, 2, -14),                # ends one byte past it
    (BASE + SPAN, 1, -14),                    # just after
    (2**64 - 8, 16, -14),                     # wraps around the address space
    (0, 16, -14),
])
def test_prefetch_l2_cases(addr, length, want):
    from oracle.oracle import Oracle
    env = Oracle()
    reg = env.region_map(BASE, SPAN)
    ev = gen.records(1, addr=np.uint64(addr), ts=np.uint64(length))
    r0 = env.run(ev, env.load_prog(asm.assemble(L2CALL, {"region": reg})))
    assert int(r0[0]) == want % 2**64
    assert env.stats()["helper_errors"] == (1 if want else 0)


def test_prefetch_l2_region_has_no_content():
    """A region is not a keyed map: lookups fault, host writes and dumps are refused."""
    from oracle.oracle import Oracle, OracleFault
    env = Oracle()
    reg = env.region_map(BASE, SPAN)
    assert env.update_map(reg, b"\0" * 4, b"\0" * 8) == -22
    with pytest.raises(OracleFault):
        env.run(gen.records(1), env.load_prog(asm.assemble(
            "stw [r10-4], 0\nlddw r1, map:region\nmov64 r2, r10\nadd64 r2, -4\ncall 1\nmov64 r0, 0\nexit",
            {"region": reg})))
    with pytest.raises(OSError):
        env.region_map(0, 16)


def test_l2_stride_policy_closed_form():
    """P7, the device L2 stride prefetch policy (gxin/instrument.py): for an access at a the hook
    prefetches [a + dist, a + dist + len); R0 is that call's result and outcome[] counts 0 / -EINVAL
    / -EFAULT.  Closed form over a strided access stream crossing the region's end."""
    from gxin import instrument
    from oracle.oracle import ARRAY, Oracle
    env = Oracle()
    n, stride, dist, ln = 5000, 256, 4096, 128
    reg = env.region_map(BASE, n * stride)
    fds = instrument.setup_l2(env, reg, dist, ln)
    addr = BASE + stride * np.arange(n, dtype=np.uint64)
    r0 = env.run(gen.records(n, addr=addr), env.load_prog(asm.assemble(instrument.P7_L2_STRIDE, fds)))
    inside = (addr + np.uint64(dist + ln)) <= np.uint64(BASE + n * stride)
    want = np.where(inside, 0, 2**64 - 14).astype(np.uint64)
    assert (r0 == want).all()
    assert env.array_u64(fds["outcome"]).tolist() == [int(inside.sum()), 0, int((~inside).sum()), 0]


def test_l2_stride_policy_trigger_mask():
    """P7 with a trigger mask: only accesses at a chunk start (addr & mask == 0) prefetch; the others
    return 0 and are counted as not triggered."""
    from gxin import instrument
    from oracle.oracle import Oracle
    env = Oracle()
    n, stride, dist, ln, mask = 4096, 256, 8192, 128, 4095
    reg = env.region_map(BASE, n * stride)
    fds = instrument.setup_l2(env, reg, dist, ln, mask)
    addr = BASE + stride * np.arange(n, dtype=np.uint64)
    r0 = env.run(gen.records(n, addr=addr), env.load_prog(asm.assemble(instrument.P7_L2_STRIDE, fds)))
    trig = (addr & np.uint64(mask)) == 0
    inside = (addr + np.uint64(dist + ln)) <= np.uint64(BASE + n * stride)
    want = np.where(trig & ~inside, 2**64 - 14, 0).astype(np.uint64)
    assert (r0 == want).all()
    assert env.array_u64(fds["outcome"]).tolist() == [int((trig & inside).sum()), 0, int((trig & ~inside).sum()),
                                                      int((~trig).sum())]
    assert int(trig.sum()) == n * stride // (mask + 1)
