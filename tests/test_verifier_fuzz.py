"""Verifier soundness fuzz (SURVEY.md §8c c.5 'Verifier' row, c.7): random programs from a grammar
that mixes safe and unsafe instructions; every program the verifier ACCEPTS must run on random
events in the oracle without an oracle fault (O7 pointer/bounds/alignment/initialisation checks).
The oracle is the dynamic check; the verifier is the code under test."""
import numpy as np
import pytest

import paper_2512_12615_b200 as gx
from gxin import asm, gen
from oracle.oracle import Oracle, OracleFault

HASH, ARRAY, PT, RINGBUF = 1, 2, 6, 27
SPECS = {"arr": (ARRAY, 4, 16, 8), "h": (HASH, 8, 8, 64), "pt": (PT, 4, 16, 4), "rb": (RINGBUF, 0, 0, 1 << 16)}


def rand_program(rng) -> str:
    lines = [] if rng.random() < 0.1 else [f"mov64 {r}, {int(rng.integers(0, 64))}" for r in ("r0", "r2", "r3", "r4", "r6", "r7", "r8")]
    n = int(rng.integers(2, 12))
    regs = ["r0", "r2", "r3", "r4", "r6", "r7"]
    for i in range(n):
        k = int(rng.integers(0, 15))
        r = regs[int(rng.integers(0, len(regs)))]
        s = regs[int(rng.integers(0, len(regs)))]
        off = int(rng.choice([-16, -12, -8, -4, -3, 0, 4, 8, 12, 16, 24, 28, 32]))
        imm = int(rng.choice([0, 1, 3, 7, 8, 15, 16, 255, -1, 1 << 20]))
        if k == 0:
            lines.append(f"mov64 {r}, {imm}")
        elif k == 1:
            op = rng.choice(["add", "sub", "and", "or", "xor", "lsh", "rsh", "mul", "mod", "div"])
            w = rng.choice(["64", "32"])
            lines.append(f"{op}{w} {r}, {s}" if rng.random() < 0.5 else f"{op}{w} {r}, {imm & 31 if op in ('lsh', 'rsh') else (imm or 1)}")
        elif k == 2:
            sz = rng.choice(["b", "h", "w", "dw"])
            lines.append(f"ldx{sz} {r}, [r1+{abs(off) % 40}]")
        elif k == 3:
            sz = rng.choice(["w", "dw"])
            lines.append(f"st{sz} [r10{off - 8:+d}], {imm}")
        elif k == 4:
            sz = rng.choice(["w", "dw"])
            lines.append(f"stx{sz} [r10{off - 8:+d}], {r}")
        elif k == 5:
            sz = rng.choice(["w", "dw", "b"])
            lines.append(f"ldx{sz} {r}, [r10{off - 8:+d}]")
        elif k in (6, 7):
            m = rng.choice(["arr", "pt", "h"])
            koff = -8 if m == "h" else -4
            st = "stdw" if m == "h" else "stw"
            lines += [f"{st} [r10{koff:+d}], {abs(imm) % 10}", f"lddw r1, map:{m}", "mov64 r2, r10",
                      f"add64 r2, {koff}", "call 1"]
            if rng.random() < 0.85:
                lines.append("jeq r0, 0, out")
            sz = rng.choice(["w", "dw"])
            lines.append(f"ldx{sz} r6, [r0{rng.choice([0, 4, 8, 16]):+d}]" if rng.random() < 0.5
                         else f"atomic_add{'64' if sz == 'dw' else '32'} [r0+{rng.choice([0, 8, 12])}], r6")
            lines.append("mov64 r1, r6")
        elif k == 8:
            cond = rng.choice(["jeq", "jne", "jgt", "jsgt", "jset"])
            lines.append(f"{cond} {r}, {imm}, out")
        elif k == 9:
            lines += [f"stdw [r10-16], {imm}", f"stdw [r10-8], {imm}", "lddw r1, map:rb", "mov64 r2, r10",
                      f"add64 r2, {int(rng.choice([-16, -12, -8]))}", f"mov64 r3, {int(rng.choice([8, 16, 24]))}",
                      "mov64 r4, 0", "call 130"]
        elif k == 10:
            lines.append(f"mov64 {r}, r10")
            lines.append(f"add64 {r}, {off - 8}")
        elif k == 11:
            lines.append(f"stxdw [{r}+0], {s}")
        elif k == 12:
            lines += ["mov64 r8, 3", "loop%d: add64 r7, 1" % i, "sub64 r8, 1", "jne r8, 0, loop%d" % i]
        elif k == 13:
            lines += [f"stdw [r10-8], {abs(imm) % 10}", f"stdw [r10-16], {imm}", "lddw r1, map:h", "mov64 r2, r10",
                      "add64 r2, -8", "mov64 r3, r10", "add64 r3, -16", "mov64 r4, 0", "call 2"]
        else:
            lines.append(f"mov64 {r}, {s}")
    lines += ["out:", "mov64 r0, 0" if rng.random() < 0.8 else "mov64 r0, r0", "exit"]
    return "\n".join(l for l in lines if l)


def test_accepted_programs_never_fault():
    rng = np.random.default_rng(1234)
    ev = gen.records(96, addr=rng.integers(0, 1 << 63, 96, dtype=np.uint64),
                     ts=rng.integers(0, 1 << 63, 96, dtype=np.uint64), hook=0, size=8)
    n_acc = 0
    for it in range(3000):
        text = rand_program(rng)
        env = Oracle()
        fds = {name: env.create_map(*spec) for name, spec in SPECS.items()}
        try:
            slots = asm.assemble(text, fds)
        except Exception:
            continue
        maps = {fd: SPECS[name] for name, fd in fds.items()}
        v, rep, log = gx.gx_verify_offline(slots, maps)
        if v != 0:
            continue
        n_acc += 1
        p = env.load_prog(slots)
        try:
            env.run(ev, p)
        except OracleFault as e:
            pytest.fail(f"verifier accepted an unsafe program ({e}):\n{text}")
    assert n_acc > 100, n_acc
