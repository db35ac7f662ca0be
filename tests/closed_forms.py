"""Closed forms used to PIN the oracle (and, through parity, the CUDA path).

These are the mathematical definitions written with Python's arbitrary-precision
integers and numpy reductions -- not a transcription of the oracle's C code:
    * ALU / JMP: RFC 9669 semantics as integer arithmetic mod 2^W;
    * configs: the numpy closed forms of SURVEY.md §8c c.5 (bincount, unique, searchsorted).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def signed(v: int, W: int) -> int:
    v &= (1 << W) - 1
    return v - (1 << W) if v >> (W - 1) else v


def trunc_div(a: int, b: int) -> int:
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


ALU_NAMES = ("add", "sub", "mul", "div", "sdiv", "mod", "smod", "or", "and", "xor",
             "lsh", "rsh", "arsh", "mov", "neg", "movsx8", "movsx16", "movsx32")


def alu(name: str, W: int, d: int, s: int) -> int:
    """Result register (64-bit view) of `name` on W-bit operands d (dst) and s (src)."""
    M = (1 << W) - 1
    d &= M
    s &= M
    sd, ss = signed(d, W), signed(s, W)
    if name == "add":
        r = d + s
    elif name == "sub":
        r = d - s
    elif name == "mul":
        r = d * s
    elif name == "div":
        r = 0 if s == 0 else d // s
    elif name == "sdiv":
        r = 0 if s == 0 else trunc_div(sd, ss)
    elif name == "mod":
        r = d if s == 0 else d % s
    elif name == "smod":
        r = d if s == 0 else sd - trunc_div(sd, ss) * ss
    elif name == "or":
        r = d | s
    elif name == "and":
        r = d & s
    elif name == "xor":
        r = d ^ s
    elif name == "lsh":
        r = d << (s % W)
    elif name == "rsh":
        r = d >> (s % W)
    elif name == "arsh":
        r = sd >> (s % W)
    elif name == "mov":
        r = s
    elif name == "neg":
        r = -d
    elif name.startswith("movsx"):
        b = int(name[5:])
        r = signed(s, b)
    else:
        raise KeyError(name)
    return r & M  # ALU32 results zero-extend into the 64-bit register


JMP_NAMES = ("jeq", "jne", "jgt", "jge", "jlt", "jle", "jsgt", "jsge", "jslt", "jsle", "jset")


def jmp(name: str, W: int, d: int, s: int) -> bool:
    M = (1 << W) - 1
    d &= M
    s &= M
    sd, ss = signed(d, W), signed(s, W)
    return {"jeq": d == s, "jne": d != s, "jgt": d > s, "jge": d >= s, "jlt": d < s, "jle": d <= s,
            "jsgt": sd > ss, "jsge": sd >= ss, "jslt": sd < ss, "jsle": sd <= ss,
            "jset": (d & s) != 0}[name]


def edge_grid(n_random: int = 40, seed: int = 7) -> list[int]:
    base = [0, 1, 2, 3, 7, 8, 31, 32, 33, 63, 64, 65, 127, 255, 256, 0x7FFF, 0x8000, 0xFFFF,
            (1 << 31) - 1, 1 << 31, (1 << 31) + 1, (1 << 32) - 1, 1 << 32, (1 << 32) + 1,
            (1 << 63) - 1, 1 << 63, (1 << 63) + 1, M64, M64 - 1, 0xFFFFFFFF80000000,
            0xFFFFFFFF00000007, 0x8000000000000001, 0x00000000DEADBEEF, 0x123456789ABCDEF0]
    rng = np.random.default_rng(seed)
    base += [int(x) for x in rng.integers(0, 1 << 63, n_random, dtype=np.uint64) * 2 + 1]
    base += [int(x) & 0xFFFFFFFF for x in rng.integers(0, 1 << 62, n_random // 2, dtype=np.uint64)]
    return base


# ---------------------------------------------------------------- config closed forms

def c1_counts(ev) -> np.ndarray:
    """P1/P1d: counts[(addr >> 12) & 255]."""
    return np.bincount(((ev["addr"] >> np.uint64(12)) & np.uint64(255)).astype(np.int64),
                       minlength=256).astype(np.uint64)


def c2_expected(ev):
    """P2: hist[sm*64+warp] and the per-thread fold {cnt, bytes} per lane_id."""
    key = ev["sm_id"].astype(np.int64) * 64 + ev["warp_id"].astype(np.int64)
    hist = np.bincount(key, minlength=148 * 64).astype(np.uint64)
    lane = ev["lane_id"].astype(np.int64)
    cnt = np.bincount(lane, minlength=32).astype(np.uint64)
    byt = np.bincount(lane, weights=ev["size"].astype(np.float64), minlength=32).astype(np.uint64)
    pt = np.stack([cnt, byt], axis=1).reshape(-1)
    return hist, pt


def c3_expected(ev, threshold=64, counts0=None):
    """P3 from an empty map: hash = page counts; ringbuf = {(page, T) : count >= T}."""
    pages = (ev["addr"] >> np.uint64(12)).astype(np.uint64)
    u, c = np.unique(pages, return_counts=True)
    table = {int(p): int(n) for p, n in zip(u, c)}
    rb = sorted(int(p).to_bytes(8, "little") + int(threshold).to_bytes(8, "little")
                for p, n in table.items() if n >= threshold)
    return table, rb


def c4_expected(ev, bounds):
    """P4: centroid events -> cstat[0]; else list = searchsorted(bounds, addr, 'right') - 1."""
    addr = ev["addr"]
    cent = addr < bounds[0]
    lst = np.searchsorted(bounds, addr, side="right").astype(np.int64) - 1
    lst = np.clip(lst, 0, 4095)
    scan = ~cent
    cstat = np.zeros(4, dtype=np.uint64)
    cstat[0] = int(cent.sum())
    hits_u, hits_c = np.unique(lst[scan], return_counts=True)
    hits = {int(k): int(v) for k, v in zip(hits_u, hits_c)}
    lbytes = np.bincount(lst[scan], weights=ev["size"][scan].astype(np.float64),
                         minlength=4096).astype(np.uint64)
    scan_pt = np.array([int(ev["size"][scan].astype(np.uint64).sum())], dtype=np.uint64)
    r0 = np.where(cent, 4096, lst).astype(np.uint64)
    return dict(cstat=cstat, hits=hits, list_bytes=lbytes, scan_pt=scan_pt, r0=r0)
