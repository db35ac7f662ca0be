"""Pins for the oracle's helpers and maps (SURVEY.md §8c O6, O8, c.8 helper rows; bpf.h contracts)."""
import numpy as np
import pytest

from gxin import asm, gen
from oracle.oracle import ARRAY, HASH, PERTHREAD_ARRAY, RINGBUF, Oracle

E2BIG, EEXIST, EINVAL, ENOENT, EAGAIN = 7, 17, 22, 2, 11


def neg(e):
    return (-e) & ((1 << 64) - 1)


def update_prog(key_size, key, val, flags):
    st = "stdw" if key_size == 8 else "stw"
    return f"""
        {st} [r10-8], {key}
        stdw [r10-16], {val}
        lddw r1, map:m
        mov64 r2, r10
        add64 r2, -8
        mov64 r3, r10
        add64 r3, -16
        mov64 r4, {flags}
        call 2
        exit
    """


def run1(env, text, fds):
    p = env.load_prog(asm.assemble(text, fds))
    return int(env.run(gen.records(1), p)[0])


def test_array_update_errors():
    """bpf.h:1762-1776: NOEXIST on an ARRAY -> -EEXIST; key >= max -> -E2BIG; flags=3 -> -EINVAL."""
    env = Oracle()
    fd = env.create_map(ARRAY, 4, 8, 4)
    assert run1(env, update_prog(4, 1, 9, 0), {"m": fd}) == 0
    assert run1(env, update_prog(4, 1, 9, 1), {"m": fd}) == neg(EEXIST)
    assert run1(env, update_prog(4, 4, 9, 0), {"m": fd}) == neg(E2BIG)
    assert run1(env, update_prog(4, 1, 9, 3), {"m": fd}) == neg(EINVAL)
    assert run1(env, update_prog(4, 2, 5, 2), {"m": fd}) == 0
    assert list(env.array_u64(fd)) == [0, 9, 5, 0]
    assert env.stats()["helper_errors"] == 3


def test_hash_full_and_flags():
    """c.8: max_entries=2, update(ANY) keys 1,2,3 -> 0, 0, -E2BIG; hash_full=1; lookup(3)=NULL."""
    env = Oracle()
    fd = env.create_map(HASH, 8, 8, 2)
    fds = {"m": fd}
    assert [run1(env, update_prog(8, k, 10 * k, 0), fds) for k in (1, 2, 3)] == [0, 0, neg(E2BIG)]
    assert env.stats()["hash_full"] == 1
    look = """
        stdw [r10-8], 3
        lddw r1, map:m
        mov64 r2, r10
        add64 r2, -8
        call 1
        jeq r0, 0, +2
        mov64 r0, 1
        exit
        mov64 r0, 0
        exit
    """
    assert run1(env, look, fds) == 0
    # NOEXIST on present -> -EEXIST, EXIST on absent -> -ENOENT, EXIST on present -> 0
    assert run1(env, update_prog(8, 1, 7, 1), fds) == neg(EEXIST)
    assert run1(env, update_prog(8, 9, 7, 2), fds) == neg(ENOENT)
    assert run1(env, update_prog(8, 1, 7, 2), fds) == 0
    assert env.hash_items(fd) == {1: [7], 2: [20]}


def test_hash_key0_and_allones():
    env = Oracle()
    fd = env.create_map(HASH, 8, 8, 8)
    for k in (0, -1):
        assert run1(env, update_prog(8, k, 5, 0), {"m": fd}) == 0
    items = env.hash_items(fd)
    assert sorted(items) == [0, (1 << 64) - 1]


def test_ringbuf_overflow():
    """c.8: capacity 4096 B, 16-B payload (24-B records): 170 outputs fit (4080 B), the 171st
    returns -EAGAIN; drops = 1 (bpf.h:6064-6066 8-byte header, 8-byte padding)."""
    env = Oracle()
    rb = env.create_map(RINGBUF, 0, 0, 4096)
    text = """
        ldxdw r6, [r1+0]
        stxdw [r10-16], r6
        stdw [r10-8], 7
        lddw r1, map:rb
        mov64 r2, r10
        add64 r2, -16
        mov64 r3, 16
        mov64 r4, 0
        call 130
        exit
    """
    p = env.load_prog(asm.assemble(text, {"rb": rb}))
    r0 = env.run(gen.records(171, addr=np.arange(171, dtype=np.uint64)), p)
    assert (r0[:170] == 0).all() and int(r0[170]) == neg(EAGAIN)
    assert env.stats()["ringbuf_drops"] == 1
    recs = env.ringbuf_records(rb)
    assert len(recs) == 170
    assert sorted(recs) == sorted(i.to_bytes(8, "little") + (7).to_bytes(8, "little") for i in range(170))


def test_ringbuf_bad_flags():
    env = Oracle()
    rb = env.create_map(RINGBUF, 0, 0, 4096)
    text = """
        stdw [r10-8], 1
        lddw r1, map:rb
        mov64 r2, r10
        add64 r2, -8
        mov64 r3, 8
        mov64 r4, 3
        call 130
        exit
    """
    assert run1(env, text, {"rb": rb}) == neg(EINVAL)


def test_perthread_shards_fold():
    """§8c S4: per-thread values fold by SUM over shards; the fold equals the S=1 result."""
    ev = gen.generate("C2", 3, 1 << 12)
    from gxin import programs
    outs = []
    for S in (1, 7, 64):
        env = Oracle()
        env.set_pt_shards(S)
        fds = {n: env.create_map(s.type, s.key_size, s.value_size, s.max_entries)
               for n, s in programs.maps_of("P2").items()}
        p = env.load_prog(programs.build("P2", fds))
        env.run(ev, p)
        outs.append((env.dump(fds["hist"]), env.dump(fds["lane_pt"])))
    assert outs[0] == outs[1] == outs[2]


def test_host_update_perthread_zeroes_other_shards():
    env = Oracle()
    env.set_pt_shards(4)
    fd = env.create_map(PERTHREAD_ARRAY, 4, 8, 2)
    text = """
        stw [r10-4], 1
        lddw r1, map:m
        mov64 r2, r10
        add64 r2, -4
        call 1
        jeq r0, 0, +2
        mov64 r1, 5
        atomic_add64 [r0+0], r1
        mov64 r0, 0
        exit
    """
    p = env.load_prog(asm.assemble(text, {"m": fd}))
    env.run(gen.records(16), p)
    assert list(env.array_u64(fd)) == [0, 80]
    env.update_map(fd, (1).to_bytes(4, "little"), (3).to_bytes(8, "little"))
    assert list(env.array_u64(fd)) == [0, 3]


def test_spec_merge_example():
    """shards {3:+5} and {3:+2} merge to +7 (S3 snapshot-and-merge)."""
    init = Oracle()
    fd = init.create_map(ARRAY, 4, 8, 8)
    init.update_map(fd, (3).to_bytes(4, "little"), (100).to_bytes(8, "little"))
    locals_ = [init.clone(), init.clone()]
    for env, add in zip(locals_, (5, 2)):
        text = f"""
            stw [r10-4], 3
            lddw r1, map:m
            mov64 r2, r10
            add64 r2, -4
            call 1
            jeq r0, 0, +2
            mov64 r1, {add}
            atomic_add64 [r0+0], r1
            mov64 r0, 0
            exit
        """
        run1(env, text, {"m": fd})
    assert init.merge(locals_) == 0
    assert int(init.array_u64(fd)[3]) == 107


def test_merge_conservation_random():
    """canonical = initial + sum of all deltas (10^5 updates, 4 shards, 20 boundaries)."""
    rng = np.random.default_rng(5)
    init = Oracle()
    fd = init.create_map(ARRAY, 4, 8, 64)
    text = """
        ldxdw r2, [r1+0]
        stxw [r10-4], r2
        ldxdw r6, [r1+8]
        lddw r1, map:m
        mov64 r2, r10
        add64 r2, -4
        call 1
        jeq r0, 0, +1
        atomic_add64 [r0+0], r6
        mov64 r0, 0
        exit
    """
    want = np.zeros(64, dtype=np.uint64)
    for boundary in range(20):
        locals_ = [init.clone() for _ in range(4)]
        for env in locals_:
            keys = rng.integers(0, 64, 1250, dtype=np.uint64)
            vals = rng.integers(0, 1 << 62, 1250, dtype=np.uint64)
            p = env.load_prog(asm.assemble(text, {"m": fd}))
            env.run(gen.records(1250, addr=keys, ts=vals), p)
            np.add.at(want, keys.astype(np.int64), vals)
        assert init.merge(locals_) == 0
    assert (init.array_u64(fd) == want).all()
