"""Text assembler / disassembler for standard Linux eBPF instruction slots.

INPUT-GENERATION module (see gxin/__init__.py): it turns policy text into the
8-byte `struct bpf_insn` slots that BOTH the CUDA path (through gx_load_prog)
and the CPU oracle (through its own decoder) consume.  It holds no execution
semantics -- only the encoding.

Encoding (bpf.h:72-77 `struct bpf_insn`):
    byte 0      code   = op | source | class   (bpf_common.h:6-51, bpf.h:17-51)
    byte 1      dst_reg (low nibble) | src_reg (high nibble)
    bytes 2-3   off    (s16, little endian)
    bytes 4-7   imm    (s32, little endian)
`lddw` (code 0x18) takes two slots; the second slot is all zero except imm,
which carries the upper 32 bits (bpf.h:1244-1266).  src_reg of the first slot
selects the pseudo source: 0 plain constant, 1 BPF_PSEUDO_MAP_FD, 2
BPF_PSEUDO_MAP_VALUE.

The text syntax follows SPEC.md:55-63's idea of a mnemonic assembler, with the
mnemonics of the listing in SURVEY.md §8d (P1):

    label:                         ; comments with ';' or '#'
    mov64 r2, r10 / mov32 r2, 7    ; ALU: add sub mul div sdiv mod smod or and
    lsh64 r2, 12                   ;      xor lsh rsh arsh mov movsx8/16/32, {64,32}
    neg64 r2                       ; NEG
    be16 r2 / le32 r2 / bswap64 r2 ; END (ALU class) and BSWAP (ALU64 class)
    jeq r0, 0, +2 / jsgt32 r1, r2, label / ja label
    call 1 / exit
    ldxdw r2, [r1+0] / ldxsb r2, [r10-1]   ; LDX MEM / MEMSX
    stw [r10-4], 7 / stxdw [r10-8], r2     ; ST / STX MEM
    atomic_add64 [r0+0], r1 / atomic_fetch_or32 [r0+4], r1
    xchg64 [r0+0], r1 / cmpxchg64 [r0+0], r1
    lddw r1, 0x0123456789abcdef / lddw r1, map:counts / lddw r1, mapval:counts+8
    .raw 0x20 0 0 0 0              ; an arbitrary slot (for reject-corpus programs)
"""
from __future__ import annotations

import re
import struct

CLS = {"ld": 0x00, "ldx": 0x01, "st": 0x02, "stx": 0x03, "alu": 0x04,
       "jmp": 0x05, "jmp32": 0x06, "alu64": 0x07}
SZ = {"w": 0x00, "h": 0x08, "b": 0x10, "dw": 0x18}
MODE_IMM, MODE_MEM, MODE_MEMSX, MODE_ATOMIC = 0x00, 0x60, 0x80, 0xC0
SRC_K, SRC_X = 0x00, 0x08
ALU_OPS = {"add": 0x00, "sub": 0x10, "mul": 0x20, "div": 0x30, "or": 0x40,
           "and": 0x50, "lsh": 0x60, "rsh": 0x70, "neg": 0x80, "mod": 0x90,
           "xor": 0xA0, "mov": 0xB0, "arsh": 0xC0, "end": 0xD0}
JMP_OPS = {"ja": 0x00, "jeq": 0x10, "jgt": 0x20, "jge": 0x30, "jset": 0x40,
           "jne": 0x50, "jsgt": 0x60, "jsge": 0x70, "call": 0x80, "exit": 0x90,
           "jlt": 0xA0, "jle": 0xB0, "jslt": 0xC0, "jsle": 0xD0}
ATOMIC_OPS = {"add": 0x00, "or": 0x40, "and": 0x50, "xor": 0xA0}
FETCH, XCHG, CMPXCHG = 0x01, 0xE1, 0xF1

PSEUDO_MAP_FD, PSEUDO_MAP_VALUE = 1, 2


class AsmError(ValueError):
    pass


def encode(code: int, dst: int = 0, src: int = 0, off: int = 0, imm: int = 0) -> bytes:
    """One 8-byte slot (bpf.h:72-77)."""
    if not (0 <= dst <= 15 and 0 <= src <= 15):
        raise AsmError(f"register out of nibble range: {dst} {src}")
    if not -(1 << 15) <= off < (1 << 15):
        raise AsmError(f"off out of s16 range: {off}")
    imm = imm & 0xFFFFFFFF
    return struct.pack("<BBhI", code & 0xFF, (dst & 0xF) | ((src & 0xF) << 4), off, imm)


def decode(slots: bytes):
    """Yield (code, dst, src, off, imm) for every 8-byte slot."""
    if len(slots) % 8:
        raise AsmError("program length not a multiple of 8")
    for i in range(0, len(slots), 8):
        code, regs, off, imm = struct.unpack_from("<BBhi", slots, i)
        yield code, regs & 0xF, regs >> 4, off, imm


_REG = re.compile(r"^r(\d+)$")
_MEM = re.compile(r"^\[\s*r(\d+)\s*([+-]\s*(?:0x[0-9a-fA-F]+|\d+))?\s*\]$")


def _reg(tok: str) -> int:
    m = _REG.match(tok.strip())
    if not m:
        raise AsmError(f"expected register, got {tok!r}")
    return int(m.group(1))


def _int(tok: str) -> int:
    tok = tok.strip().replace(" ", "")
    try:
        return int(tok, 0)
    except ValueError as e:
        raise AsmError(f"expected integer, got {tok!r}") from e


def _mem(tok: str):
    m = _MEM.match(tok.strip())
    if not m:
        raise AsmError(f"expected [rN+off], got {tok!r}")
    off = _int(m.group(2).replace(" ", "")) if m.group(2) else 0
    return int(m.group(1)), off


def _split_operands(rest: str):
    out, depth, cur = [], 0, ""
    for ch in rest:
        if ch == "[":
            depth += 1
        elif ch == "]":
            depth -= 1
        if ch == "," and depth == 0:
            out.append(cur.strip())
            cur = ""
        else:
            cur += ch
    if cur.strip():
        out.append(cur.strip())
    return out


def assemble(text: str, maps: dict | None = None) -> bytes:
    """Assemble `text` into eBPF slots.  `maps` maps a name to its map fd."""
    maps = maps or {}
    lines = []
    for raw in text.splitlines():
        line = raw.split(";")[0].split("#")[0].strip()
        if line:
            lines.append(line)
    # pass 1: labels -> slot index
    labels, slot = {}, 0
    items = []
    for line in lines:
        while True:
            m = re.match(r"^([A-Za-z_]\w*):\s*(.*)$", line)
            if not m:
                break
            if m.group(1) in labels:
                raise AsmError(f"duplicate label {m.group(1)}")
            labels[m.group(1)] = slot
            line = m.group(2).strip()
        if not line:
            continue
        mnem = line.split(None, 1)[0].lower()
        items.append((slot, line))
        slot += 2 if mnem == "lddw" else 1
    out = bytearray()
    for pc, line in items:
        parts = line.split(None, 1)
        mnem = parts[0].lower()
        ops = _split_operands(parts[1]) if len(parts) > 1 else []
        out += _assemble_one(mnem, ops, pc, labels, maps)
    return bytes(out)


def _target(tok: str, pc: int, labels: dict) -> int:
    tok = tok.strip()
    if tok in labels:
        return labels[tok] - pc - 1
    return _int(tok)


def _assemble_one(mnem, ops, pc, labels, maps) -> bytes:
    if mnem == ".raw":
        vals = [int(x, 0) for x in " ".join(ops).replace(",", " ").split()]
        if len(vals) != 5:
            raise AsmError(".raw takes code dst src off imm")
        return encode(*vals)
    if mnem == "exit":
        return encode(CLS["jmp"] | JMP_OPS["exit"])
    if mnem == "call":
        return encode(CLS["jmp"] | JMP_OPS["call"], imm=_int(ops[0]))
    if mnem == "ja":
        return encode(CLS["jmp"] | JMP_OPS["ja"], off=_target(ops[0], pc, labels))
    if mnem == "lddw":
        dst = _reg(ops[0])
        arg = ops[1].strip()
        if arg.startswith("map:"):
            name = arg[4:]
            if name not in maps:
                raise AsmError(f"unknown map {name}")
            return encode(0x18, dst, PSEUDO_MAP_FD, 0, maps[name]) + encode(0, 0, 0, 0, 0)
        if arg.startswith("mapval:"):
            m = re.match(r"^mapval:([\w.]+)\s*(?:\+\s*(\S+))?$", arg)
            if not m or m.group(1) not in maps:
                raise AsmError(f"bad mapval operand {arg!r}")
            off = _int(m.group(2)) if m.group(2) else 0
            return encode(0x18, dst, PSEUDO_MAP_VALUE, 0, maps[m.group(1)]) + encode(0, 0, 0, 0, off)
        v = _int(arg) & 0xFFFFFFFFFFFFFFFF
        return encode(0x18, dst, 0, 0, v & 0xFFFFFFFF) + encode(0, 0, 0, 0, v >> 32)
    # jumps
    m = re.match(r"^(j[a-z]+?)(32)?$", mnem)
    if m and m.group(1) in JMP_OPS and m.group(1) not in ("call", "exit"):
        cls = CLS["jmp32"] if m.group(2) else CLS["jmp"]
        op = JMP_OPS[m.group(1)]
        dst = _reg(ops[0])
        off = _target(ops[2], pc, labels)
        if _REG.match(ops[1].strip()):
            return encode(cls | op | SRC_X, dst, _reg(ops[1]), off, 0)
        return encode(cls | op | SRC_K, dst, 0, off, _int(ops[1]))
    # loads / stores
    m = re.match(r"^ldx(s?)(dw|w|h|b)$", mnem)
    if m:
        mode = MODE_MEMSX if m.group(1) else MODE_MEM
        dst = _reg(ops[0])
        src, off = _mem(ops[1])
        return encode(CLS["ldx"] | SZ[m.group(2)] | mode, dst, src, off, 0)
    m = re.match(r"^st(dw|w|h|b)$", mnem)
    if m:
        dst, off = _mem(ops[0])
        return encode(CLS["st"] | SZ[m.group(1)] | MODE_MEM, dst, 0, off, _int(ops[1]))
    m = re.match(r"^stx(dw|w|h|b)$", mnem)
    if m:
        dst, off = _mem(ops[0])
        return encode(CLS["stx"] | SZ[m.group(1)] | MODE_MEM, dst, _reg(ops[1]), off, 0)
    m = re.match(r"^(atomic_fetch_|atomic_)(add|or|and|xor)(32|64)$", mnem)
    if m:
        imm = ATOMIC_OPS[m.group(2)] | (FETCH if m.group(1) == "atomic_fetch_" else 0)
        sz = SZ["dw"] if m.group(3) == "64" else SZ["w"]
        dst, off = _mem(ops[0])
        return encode(CLS["stx"] | sz | MODE_ATOMIC, dst, _reg(ops[1]), off, imm)
    m = re.match(r"^(xchg|cmpxchg)(32|64)$", mnem)
    if m:
        imm = XCHG if m.group(1) == "xchg" else CMPXCHG
        sz = SZ["dw"] if m.group(2) == "64" else SZ["w"]
        dst, off = _mem(ops[0])
        return encode(CLS["stx"] | sz | MODE_ATOMIC, dst, _reg(ops[1]), off, imm)
    # END / BSWAP
    m = re.match(r"^(le|be|bswap)(16|32|64)$", mnem)
    if m:
        dst = _reg(ops[0])
        width = int(m.group(2))
        if m.group(1) == "bswap":
            return encode(CLS["alu64"] | ALU_OPS["end"] | SRC_K, dst, 0, 0, width)
        src = SRC_X if m.group(1) == "be" else SRC_K
        return encode(CLS["alu"] | ALU_OPS["end"] | src, dst, 0, 0, width)
    # ALU
    m = re.match(r"^(add|sub|mul|div|sdiv|mod|smod|or|and|lsh|rsh|arsh|neg|xor|mov|movsx8|movsx16|movsx32)(64|32)$", mnem)
    if m:
        name, w = m.group(1), m.group(2)
        cls = CLS["alu64"] if w == "64" else CLS["alu"]
        off = 0
        if name in ("sdiv", "smod"):
            off, name = 1, name[1:]
        if name.startswith("movsx"):
            off, name = int(name[5:]), "mov"
        op = ALU_OPS[name]
        dst = _reg(ops[0])
        if name == "neg":
            return encode(cls | op | SRC_K, dst, 0, 0, 0)
        if _REG.match(ops[1].strip()):
            return encode(cls | op | SRC_X, dst, _reg(ops[1]), off, 0)
        if off and name == "mov":
            raise AsmError("movsx has only a register form")
        return encode(cls | op | SRC_K, dst, 0, off, _int(ops[1]))
    raise AsmError(f"unknown mnemonic {mnem!r}")


def n_slots(prog: bytes) -> int:
    return len(prog) // 8
