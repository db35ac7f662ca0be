"""Pins for the oracle's instruction semantics.

ALU/ALU32/JMP/JMP32 are checked against the closed forms in closed_forms.py (integer
arithmetic mod 2^W) over an edge grid of operand pairs, for every op, K and X forms,
both widths; the hand-computed micro-pins of tests/golden/micro_pins.txt; the
hand-encoded P1 slots of tests/golden/p1_encoding.txt.
"""
import itertools
import os

import numpy as np
import pytest

from gxin import asm, gen, programs
from oracle.oracle import Oracle, OracleFault
import closed_forms as cf

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PRE = "ldxdw r0, [r1+0]\nldxdw r2, [r1+8]\n"


def run_prog(text, d, s, maps=None, env=None):
    env = env or Oracle()
    p = env.load_prog(asm.assemble(text, maps or {}))
    ev = gen.records(len(d), addr=np.asarray(d, dtype=np.uint64), ts=np.asarray(s, dtype=np.uint64))
    return env.run(ev, p)


GRID = cf.edge_grid()
PAIRS = list(itertools.product(GRID, GRID))
D = np.array([p[0] for p in PAIRS], dtype=np.uint64)
S = np.array([p[1] for p in PAIRS], dtype=np.uint64)


@pytest.mark.parametrize("W", [64, 32])
@pytest.mark.parametrize("name", [n for n in cf.ALU_NAMES if not (n == "movsx32")] + ["movsx32"])
def test_alu_x_edge_grid(name, W):
    if name == "movsx32" and W == 32:
        pytest.skip("MOVSX32 exists only for ALU64")
    ops = f"{name}{W} r0" if name == "neg" else f"{name}{W} r0, r2"
    r0 = run_prog(PRE + ops + "\nexit", D, S)
    want = np.array([cf.alu(name, W, d, s) for d, s in PAIRS], dtype=np.uint64)
    bad = np.nonzero(r0 != want)[0]
    assert bad.size == 0, [(hex(PAIRS[i][0]), hex(PAIRS[i][1]), hex(int(r0[i])), hex(int(want[i]))) for i in bad[:5]]


K_IMMS = [0, 1, -1, 2, 7, 31, 32, 63, -2, 255, 0x7FFFFFFF, -0x80000000, 0x12345678, -7, 4096]


@pytest.mark.parametrize("W", [64, 32])
@pytest.mark.parametrize("name", ["add", "sub", "mul", "div", "sdiv", "mod", "smod", "or", "and", "xor",
                                  "lsh", "rsh", "arsh", "mov"])
def test_alu_k_edge_grid(name, W):
    d = np.array(GRID, dtype=np.uint64)
    for imm in K_IMMS:
        if name in ("lsh", "rsh", "arsh") and not 0 <= imm < W:
            continue  # immediate shift >= W is rejected by the verifier (I-5)
        r0 = run_prog(PRE + f"{name}{W} r0, {imm}\nexit", d, np.zeros_like(d))
        s = imm & cf.M64 if W == 64 else imm & 0xFFFFFFFF   # K: sign-extend (64) / truncate (32), I-6
        want = np.array([cf.alu(name, W, x, s) for x in GRID], dtype=np.uint64)
        assert (r0 == want).all(), (name, W, imm)


@pytest.mark.parametrize("W", [64, 32])
def test_shift_counts_all(W):
    d = np.array([0x8000000000000001, 0xFFFFFFFFFFFFFFFF, 0x123456789ABCDEF0, 1], dtype=np.uint64)
    for name in ("lsh", "rsh", "arsh"):
        for cnt in range(128):
            r0 = run_prog(PRE + f"{name}{W} r0, r2\nexit", d, np.full(4, cnt, dtype=np.uint64))
            want = [cf.alu(name, W, int(x), cnt) for x in d]
            assert [int(v) for v in r0] == want, (name, W, cnt)


def test_divmod_exhaustive_8bit_patterns():
    """All 2^16 pairs of 8-bit patterns sign-extended to 64 bits, for DIV/MOD/SDIV/SMOD, both widths."""
    v = np.array([cf.signed(x, 8) & cf.M64 for x in range(256)], dtype=np.uint64)
    d, s = np.repeat(v, 256), np.tile(v, 256)
    for W in (64, 32):
        for name in ("div", "mod", "sdiv", "smod"):
            r0 = run_prog(PRE + f"{name}{W} r0, r2\nexit", d, s)
            want = np.array([cf.alu(name, W, int(a), int(b)) for a, b in zip(d, s)], dtype=np.uint64)
            assert (r0 == want).all(), (name, W)


@pytest.mark.parametrize("W", [64, 32])
@pytest.mark.parametrize("name", cf.JMP_NAMES)
def test_jmp_edge_grid(name, W):
    suffix = "32" if W == 32 else ""
    text = PRE + f"mov64 r3, r0\nmov64 r0, 0\n{name}{suffix} r3, r2, +1\nja +1\nmov64 r0, 1\nexit"
    r0 = run_prog(text, D, S)
    want = np.array([cf.jmp(name, W, d, s) for d, s in PAIRS], dtype=np.uint64)
    assert (r0 == want).all()
    d = np.array(GRID, dtype=np.uint64)
    for imm in K_IMMS:
        text = PRE + f"mov64 r3, r0\nmov64 r0, 0\n{name}{suffix} r3, {imm}, +1\nja +1\nmov64 r0, 1\nexit"
        r0 = run_prog(text, d, np.zeros_like(d))
        s = imm & cf.M64 if W == 64 else imm & 0xFFFFFFFF
        want = np.array([cf.jmp(name, W, x, s) for x in GRID], dtype=np.uint64)
        assert (r0 == want).all(), (name, W, imm)


def test_end_bswap_closed_forms():
    d = np.array(GRID, dtype=np.uint64)
    for width in (16, 32, 64):
        M = (1 << width) - 1
        le = run_prog(PRE + f"le{width} r0\nexit", d, d)
        be = run_prog(PRE + f"be{width} r0\nexit", d, d)
        bs = run_prog(PRE + f"bswap{width} r0\nexit", d, d)
        for x, a, b, c in zip(GRID, le, be, bs):
            lo = x & M
            swapped = int.from_bytes(lo.to_bytes(width // 8, "little"), "big")
            assert int(a) == lo and int(b) == swapped and int(c) == swapped


def _golden_cases():
    out = []
    with open(os.path.join(GOLD, "micro_pins.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, ops, d, s, want = [x.strip() for x in line.split("|")]
            out.append((name, ops.replace(" / ", "\n"), int(d, 0), int(s, 0), int(want, 0)))
    return out


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c[0])
def test_micro_pins(case):
    name, ops, d, s, want = case
    r0 = run_prog(PRE + ops + "\nexit", [d], [s])
    assert int(r0[0]) == want, (name, hex(int(r0[0])), hex(want))


def test_p1_encoding_golden():
    slots = []
    with open(os.path.join(GOLD, "p1_encoding.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            slots.append(bytes(int(x, 16) for x in line.split(";")[0].split()))
    assert programs.build("P1", {"counts": 3}) == b"".join(slots)


def test_ldimm64_encoding():
    b = asm.assemble("lddw r0, 0x0123456789ABCDEF\nexit")
    assert b[:8] == bytes([0x18, 0, 0, 0]) + (0x89ABCDEF).to_bytes(4, "little")
    assert b[8:16] == bytes(4) + (0x01234567).to_bytes(4, "little")


def test_spec_interpret_examples():
    """a constant-0 program returns 0; a bounded loop of 3 increments 0 -> 3."""
    assert int(run_prog("mov64 r0, 0\nexit", [0], [0])[0]) == 0
    env = Oracle()
    fd = env.create_map(2, 4, 8, 1)
    text = """
        mov64 r6, 3
    loop:
        stw [r10-4], 0
        lddw r1, map:faults
        mov64 r2, r10
        add64 r2, -4
        call 1
        jeq r0, 0, out
        mov64 r1, 1
        atomic_add64 [r0+0], r1
        sub64 r6, 1
        jne r6, 0, loop
    out:
        mov64 r0, 0
        exit
    """
    run_prog(text, [0], [0], {"faults": fd}, env)
    assert int(env.array_u64(fd)[0]) == 3


def test_determinism():
    """identical (program, ctx, maps) give identical results."""
    ev = gen.generate("C1", 1, 4096)
    outs = []
    for _ in range(2):
        env = Oracle()
        fd = env.create_map(2, 4, 8, 256)
        p = env.load_prog(programs.build("P1", {"counts": fd}))
        outs.append((env.run(ev, p).tobytes(), env.dump(fd)))
    assert outs[0] == outs[1]


@pytest.mark.parametrize("text,why", [
    ("ldxdw r0, [r10-8]\nexit", "uninitialised stack"),
    ("ldxdw r0, [r1+32]\nexit", "out-of-bounds"),
    ("ldxdw r0, [r1+4]\nexit", "misaligned"),
    ("stdw [r1+0], 1\nmov64 r0, 0\nexit", "write to ctx"),
    ("exit", "r0 at exit"),
    ("mov64 r0, r10\nexit", "r0 at exit"),
    ("mov64 r0, r2\nexit", "uninitialised register"),
    ("call 93\nmov64 r0, 0\nexit", "forbidden helper"),
    ("loop: ja loop", "step limit"),
])
def test_oracle_faults_on_unsafe_programs(text, why):
    """O7: an unsafe program is an oracle fault (the dynamic half of 'verifier rejects OOB')."""
    env = Oracle()
    p = env.load_prog(asm.assemble(text))
    with pytest.raises(OracleFault, match=why):
        env.run(gen.records(1), p)


def test_atomic_and_memsx_mnemonic_encodings():
    """The assembler's atomic / MEMSX mnemonics emit the bpf.h encodings the hand-encoded pins use
    (bpf.h:23 BPF_ATOMIC 0xc0, :49-51 BPF_FETCH 0x01 / BPF_XCHG 0xe1 / BPF_CMPXCHG 0xf1,
    bpf_common.h:31-48 BPF_ADD 0x00 / BPF_OR 0x40 / BPF_AND 0x50 / BPF_XOR 0xa0; MEMSX 0x80)."""
    cases = {
        "atomic_add64 [r10-8], r4": "db 4a f8 ff 00 00 00 00",
        "atomic_fetch_or64 [r10-8], r4": "db 4a f8 ff 41 00 00 00",
        "atomic_and32 [r10-8], r4": "c3 4a f8 ff 50 00 00 00",
        "atomic_fetch_xor32 [r10-8], r4": "c3 4a f8 ff a1 00 00 00",
        "xchg32 [r10-8], r4": "c3 4a f8 ff e1 00 00 00",
        "cmpxchg64 [r10-8], r4": "db 4a f8 ff f1 00 00 00",
        "ldxsh r0, [r10-2]": "89 a0 fe ff 00 00 00 00",
        "ldxsw r0, [r10-4]": "81 a0 fc ff 00 00 00 00",
    }
    for text, hexs in cases.items():
        assert asm.assemble(text) == bytes.fromhex(hexs.replace(" ", "")), text
