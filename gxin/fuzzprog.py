"""Seeded random eBPF policy programs + event batches for the GPU-vs-oracle differential fuzz.

INPUT-GENERATION module (gxin/__init__.py): it writes program TEXT for gxin.asm and builds
event records; it holds no execution semantics.  Used by tests/test_fuzz_*.py only.

The grammar covers the whole executed subset: every ALU/ALU32 op incl.
v4 SDIV/SMOD/MOVSX/BSWAP, END, JMP/JMP32 branches (forward, lane-varying -> divergence),
bounded loops (constant and lane-varying trip counts), LDX/LDX MEMSX/ST/STX of every size on
ctx / stack / map values, STX ATOMIC W/DW (ADD/OR/AND/XOR +-FETCH, XCHG, CMPXCHG) on stack,
ARRAY, HASH and per-thread values, map_lookup_elem / map_update_elem (ANY / NOEXIST / EXIST and
an invalid flag) on ARRAY and HASH, ringbuf_output, ldimm64 map values (src=2).

Determinism by construction: the batch result must not depend on the
order events run in, so that the GPU has ONE correct answer -- the oracle's:
  * "observe" maps (obs ARRAY, hobs HASH) are touched with event-UNIQUE keys (the low 13 bits of
    `addr` are a permutation of the event index), so any op may observe them: plain loads,
    FETCH atomics, XCHG, CMPXCHG, update flags, NULL-ness -- and the results flow anywhere
    (R0, branches, ringbuf payloads, other maps' operands);
  * "accumulate" maps (acc ARRAY, hacc/hacc4 HASH) take COLLIDING keys (record-uniform, lane-
    varying, constant) but are write-only: each 4- or 8-byte location has ONE fixed commutative
    op (ADD, OR, AND or XOR, never FETCH), the lookup-or-init idiom's update result is discarded;
  * the per-thread map (pt) is updated with 64-bit ADDs only (plain RMW or ATOMIC ADD): its SUM
    fold is shard-invariant (S4).
`tests/test_fuzz_oracle.py` checks these claims on the oracle itself (order and shard
invariance) before any GPU comparison relies on them.
"""
from __future__ import annotations

import numpy as np

from . import gen

HASH, ARRAY, PT, RINGBUF = 1, 2, 6, 27

MAPS = {
    "acc": (ARRAY, 4, 48, 64),
    "gacc": (ARRAY, 4, 64, 1),        # "global array" addressed by ldimm64 src=2 (ADD only)
    "hacc": (HASH, 8, 8, 4096),
    "hacc4": (HASH, 4, 8, 1024),
    "pt": (PT, 4, 16, 32),
    "obs": (ARRAY, 4, 16, 4096),
    "hobs": (HASH, 8, 8, 32768),
    "rb": (RINGBUF, 0, 0, 1 << 22),
}
UBITS = 13                       # addr & 0x1FFF is unique per event (a permutation)
UMASK = (1 << UBITS) - 1
MAX_EVENTS = 1 << UBITS

# accumulate-map layouts: (byte offset, width, op) -- one op per location, never FETCH
ACC_SLOTS = [(0, 64, "add"), (8, 64, "or"), (16, 64, "and"), (24, 64, "xor"),
             (32, 32, "add"), (36, 32, "or"), (40, 32, "and"), (44, 32, "xor")]
HACC_SLOTS = [(0, 32, "xor"), (4, 32, "add")]
HACC4_SLOTS = [(0, 64, "add")]

V = ("r6", "r7", "r8")           # live values; r9 = ctx; r0-r5 scratch
ALU_OPS = ("add", "sub", "mul", "div", "sdiv", "mod", "smod", "or", "and", "xor", "lsh", "rsh", "arsh", "mov")
JCC = ("jeq", "jne", "jgt", "jge", "jlt", "jle", "jsgt", "jsge", "jslt", "jsle", "jset")
CTX_FIELDS = [(0, 8), (8, 8), (16, 4), (20, 4), (24, 2), (26, 1), (27, 1), (28, 4)]
IMMS = (0, 1, 2, 3, 5, 7, 8, 31, 32, 63, 255, 0x7FFF, -1, -2, -128, 0x7FFFFFFF, -0x80000000, 12345)


class _Gen:
    def __init__(self, rng, n_snippets, allow=None):
        self.rng = rng
        self.lines = []
        self.lab = 0
        self.n = n_snippets
        self.allow = allow

    # -- helpers ---------------------------------------------------------------------------
    def r(self, xs):
        return xs[int(self.rng.integers(0, len(xs)))]

    def v(self):
        return self.r(V)

    def imm(self):
        return int(self.r(IMMS))

    def label(self):
        self.lab += 1
        return f"L{self.lab}"

    def emit(self, *ls):
        self.lines.extend(ls)

    # -- snippets --------------------------------------------------------------------------
    def alu(self):
        w = self.r(("64", "32"))
        d = self.v()
        k = int(self.rng.integers(0, 10))
        if k == 0:
            self.emit(f"neg{w} {d}")
        elif k == 1:
            self.emit(f"{self.r(('le', 'be'))}{self.r(('16', '32', '64'))} {d}")
        elif k == 2:
            self.emit(f"bswap{self.r(('16', '32', '64'))} {d}")
        elif k == 3:
            bits = self.r(("8", "16", "32")) if w == "64" else self.r(("8", "16"))
            self.emit(f"movsx{bits}{w} {d}, {self.v()}")
        else:
            op = self.r(ALU_OPS)
            if op in ("lsh", "rsh", "arsh") and self.rng.random() < 0.5:
                self.emit(f"{op}{w} {d}, {int(self.rng.integers(0, int(w)))}")
            elif self.rng.random() < 0.6:
                self.emit(f"{op}{w} {d}, {self.v()}")
            else:
                k_ = self.imm()
                if op in ("lsh", "rsh", "arsh"):
                    k_ &= int(w) - 1
                if op in ("div", "sdiv", "mod", "smod") and k_ == 0:
                    k_ = 7
                self.emit(f"{op}{w} {d}, {k_}")

    def ctx(self):
        off, sz = self.r(CTX_FIELDS)
        sub = {8: ["dw", "w", "h", "b"], 4: ["w", "h", "b"], 2: ["h", "b"], 1: ["b"]}[sz]
        s = self.r(sub)
        nb = {"dw": 8, "w": 4, "h": 2, "b": 1}[s]
        o = off + nb * int(self.rng.integers(0, sz // nb))
        sx = "s" if s != "dw" and self.rng.random() < 0.4 else ""
        self.emit(f"ldx{sx}{s} {self.v()}, [r9+{o}]")

    def _mem_op(self, base, offs):
        """One access at [base+off] (off from `offs`, 8-byte words), any size / kind."""
        word = self.r(offs)
        k = int(self.rng.integers(0, 6))
        if k == 0:
            s = self.r(("dw", "w", "h", "b"))
            nb = {"dw": 8, "w": 4, "h": 2, "b": 1}[s]
            o = word + nb * int(self.rng.integers(0, 8 // nb))
            sx = "s" if s != "dw" and self.rng.random() < 0.4 else ""
            self.emit(f"ldx{sx}{s} {self.v()}, [{base}{o:+d}]")
        elif k == 1:
            s = self.r(("dw", "w", "h", "b"))
            nb = {"dw": 8, "w": 4, "h": 2, "b": 1}[s]
            o = word + nb * int(self.rng.integers(0, 8 // nb))
            if self.rng.random() < 0.5:
                self.emit(f"stx{s} [{base}{o:+d}], {self.v()}")
            else:
                self.emit(f"st{s} [{base}{o:+d}], {self.imm()}")
        elif k in (2, 3):
            w = self.r(("64", "32"))
            o = word + (4 * int(self.rng.integers(0, 2)) if w == "32" else 0)
            op = self.r(("add", "or", "and", "xor"))
            f = "fetch_" if self.rng.random() < 0.6 else ""
            self.emit(f"atomic_{f}{op}{w} [{base}{o:+d}], {self.v()}")
        elif k == 4:
            w = self.r(("64", "32"))
            o = word + (4 * int(self.rng.integers(0, 2)) if w == "32" else 0)
            self.emit(f"xchg{w} [{base}{o:+d}], {self.v()}")
        else:
            w = self.r(("64", "32"))
            o = word + (4 * int(self.rng.integers(0, 2)) if w == "32" else 0)
            d = self.v()
            self.emit(f"mov64 r0, {self.v()}", f"cmpxchg{w} [{base}{o:+d}], {self.v()}", f"mov64 {d}, r0")

    def stack(self):
        self._mem_op("r10", [-64, -56, -48, -40, -32, -24, -16, -8])

    def branch(self, depth):
        L = self.label()
        cond = self.r(JCC)
        w = self.r(("", "32"))
        b = self.v() if self.rng.random() < 0.6 else str(self.imm())
        self.emit(f"{cond}{w} {self.v()}, {b}, {L}")
        for _ in range(int(self.rng.integers(1, 4))):
            self.snippet(depth + 1)
        self.emit(f"{L}:")

    def loop(self, depth):
        L = self.label()
        if self.rng.random() < 0.5:
            self.emit(f"mov64 r3, {int(self.rng.integers(1, 5))}")
        else:
            self.emit(f"mov64 r3, {self.v()}", "and64 r3, 7")
        self.emit(f"{L}:")
        for _ in range(int(self.rng.integers(1, 3))):
            self.r((self.alu, self.ctx, self.stack))()
        self.emit("sub64 r3, 1", f"jsgt{self.r(('', '32'))} r3, 0, {L}")

    def _key_to_stack(self, kind, nbytes):
        """Leaves the key at [r10-72] (nbytes wide)."""
        st = "stxdw" if nbytes == 8 else "stxw"
        if kind == "unique":
            self.emit("ldxdw r2, [r9+0]", f"and64 r2, {UMASK}")
        elif kind == "uniq_tag":       # unique key tagged per snippet class (hobs)
            self.emit("ldxdw r2, [r9+0]", f"and64 r2, {UMASK}", f"or64 r2, {int(self.rng.integers(0, 4)) << UBITS}")
        elif kind == "record":
            self.emit(f"ldx{self.r(('w', 'h'))} r2, [r9+{self.r((20, 24))}]")
        elif kind == "lane":
            self.emit("ldxb r2, [r9+27]")
        elif kind == "value":
            self.emit(f"mov64 r2, {self.v()}")
        else:
            self.emit(f"mov64 r2, {self.imm() & 0xFF}")
        return st

    def _lookup(self, m, keysz):
        self.emit(f"lddw r1, map:{m}", "mov64 r2, r10", "add64 r2, -72", "call 1")

    def acc(self):
        kind = self.r(("record", "lane", "value", "const"))
        st = self._key_to_stack(kind, 4)
        self.emit(f"and64 r2, {self.r((63, 127))}", f"{st} [r10-72], r2")
        L = self.label()
        self._lookup("acc", 4)
        self.emit(f"jeq r0, 0, {L}")
        for _ in range(int(self.rng.integers(1, 4))):
            off, w, op = self.r(ACC_SLOTS)
            self.emit(f"atomic_{op}{w} [r0+{off}], {self.v()}")
        self.emit(f"{L}:")

    def gacc(self):
        """ldimm64 src=2: a pointer into the global array's value; 8-aligned in-range offset."""
        self.emit(f"mov64 r2, {self.v()}", "and64 r2, 56", "lddw r1, mapval:gacc", "add64 r1, r2",
                  f"atomic_add64 [r1+0], {self.v()}")

    def hacc(self):
        m = self.r(("hacc", "hacc4"))
        ks = 8 if m == "hacc" else 4
        kind = self.r(("record", "lane", "value", "const"))
        st = self._key_to_stack(kind, ks)
        self.emit(f"and64 r2, {self.r((255, 1023))}", f"{st} [r10-72], r2")
        have, end = self.label(), self.label()
        self._lookup(m, ks)
        self.emit(f"jne r0, 0, {have}", "stdw [r10-80], 0", f"lddw r1, map:{m}", "mov64 r2, r10", "add64 r2, -72",
                  "mov64 r3, r10", "add64 r3, -80", "mov64 r4, 1", "call 2")
        self._lookup(m, ks)
        self.emit(f"jeq r0, 0, {end}", f"{have}:")
        for _ in range(int(self.rng.integers(1, 3))):
            off, w, op = self.r(HACC_SLOTS if m == "hacc" else HACC4_SLOTS)
            self.emit(f"atomic_{op}{w} [r0+{off}], {self.v()}")
        self.emit(f"{end}:")

    def pt(self):
        kind = self.r(("record", "lane", "value", "const"))
        st = self._key_to_stack(kind, 4)
        self.emit(f"and64 r2, {self.r((31, 63))}", f"{st} [r10-72], r2")
        L = self.label()
        self._lookup("pt", 4)
        self.emit(f"jeq r0, 0, {L}")
        for _ in range(int(self.rng.integers(1, 3))):
            off = self.r((0, 8))
            if self.rng.random() < 0.5:
                self.emit(f"ldxdw r3, [r0+{off}]", f"add64 r3, {self.v()}", f"stxdw [r0+{off}], r3")
            else:
                self.emit(f"atomic_add64 [r0+{off}], {self.v()}")
        self.emit(f"{L}:")

    def obs(self):
        self._key_to_stack("unique", 4)
        self.emit("stxw [r10-72], r2")
        if self.rng.random() < 0.3:
            self._update("obs", 16)
            return
        L = self.label()
        self._lookup("obs", 4)
        self.emit(f"jeq r0, 0, {L}", "mov64 r5, r0")
        for _ in range(int(self.rng.integers(1, 5))):
            self._mem_op("r5", [0, 8])
        self.emit(f"{L}:")

    def hobs(self):
        self._key_to_stack("uniq_tag", 8)
        self.emit("stxdw [r10-72], r2")
        if self.rng.random() < 0.4:
            self._update("hobs", 8)
            return
        L = self.label()
        self._lookup("hobs", 8)
        if self.rng.random() < 0.3:
            self.emit(f"mov64 {self.v()}, 0", f"jne r0, 0, {L}")  # NULL-ness observed
        self.emit(f"jeq r0, 0, {L}", "mov64 r5, r0")
        for _ in range(int(self.rng.integers(1, 4))):
            self._mem_op("r5", [0])
        self.emit(f"{L}:")

    def _update(self, m, vs):
        flags = self.r((0, 0, 1, 2, 2, 3))
        self.emit(f"stxdw [r10-96], {self.v()}")
        if vs > 8:
            self.emit(f"stxdw [r10-88], {self.v()}")
        self.emit(f"lddw r1, map:{m}", "mov64 r2, r10", "add64 r2, -72", "mov64 r3, r10", "add64 r3, -96",
                  f"mov64 r4, {flags}", "call 2", f"mov64 {self.v()}, r0")

    def rb(self):
        self.emit(f"stxdw [r10-96], {self.v()}", f"stxdw [r10-88], {self.v()}", f"stxdw [r10-80], {self.v()}")
        size = self.r((1, 4, 8, 12, 16, 20, 24))
        self.emit("lddw r1, map:rb", "mov64 r2, r10", "add64 r2, -96", f"mov64 r3, {size}",
                  f"mov64 r4, {self.r((0, 1, 2))}", "call 130", f"add64 {self.v()}, r0")

    def snippet(self, depth=0):
        kinds = ["alu", "alu", "ctx", "stack", "acc", "gacc", "hacc", "pt", "obs", "obs", "hobs", "hobs", "rb"]
        if depth < 2:
            kinds += ["branch", "branch", "loop"]
        if self.allow is not None:
            kinds = [k for k in kinds if k in self.allow or k in ("alu", "ctx", "branch", "loop")]
        k = self.r(kinds)
        if k == "branch":
            self.branch(depth)
        elif k == "loop":
            self.loop(depth)
        else:
            getattr(self, k)()

    def program(self):
        self.emit("mov64 r9, r1")
        for o in range(8, 104, 8):
            self.emit(f"stdw [r10-{o}], 0")
        self.emit("ldxdw r6, [r9+0]", "ldxdw r7, [r9+8]", "ldxw r8, [r9+20]")
        for _ in range(self.n):
            self.snippet()
        a, b = self.v(), self.v()
        self.emit(f"mov64 r0, {a}", f"{self.r(('xor', 'add', 'sub'))}64 r0, {b}", "exit")
        return "\n".join(self.lines)


def program(seed: int, n_snippets: int | None = None, allow=None) -> str:
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 14)) if n_snippets is None else n_snippets
    return _Gen(rng, n, allow).program()


def events(seed: int, n: int, n_tenants: int = 1, skip_tenant: bool = False, contract: bool = False) -> np.ndarray:
    """n <= 8192 events: the low 13 address bits are a permutation of [0, 8192) (unique keys);
    every other field is either record-uniform or lane-varying, per field and batch
    (`contract`: every field §8b tags UNIFORM is record-uniform, as a warp-level hook produces it)."""
    assert n <= MAX_EVENTS
    rng = np.random.default_rng(seed ^ 0xF022)
    rec = np.arange(n) >> 5

    def field(bits, uniform_p=0.5):
        hi = (1 << bits) - 1
        if contract and uniform_p != 0.3:
            uniform_p = 1.0
        if rng.random() < uniform_p:
            per_rec = rng.integers(0, hi, size=rec[-1] + 1 if n else 1, dtype=np.uint64, endpoint=True)
            return per_rec[rec] if n else per_rec[:0]
        return rng.integers(0, hi, size=n, dtype=np.uint64, endpoint=True)

    u = rng.permutation(MAX_EVENTS)[:n].astype(np.uint64)
    addr = (field(51, 0.3) << np.uint64(UBITS)) | u
    tenants = n_tenants + (1 if skip_tenant else 0)
    ten = rng.integers(0, tenants, size=n) if rng.random() < 0.5 and not contract else rng.integers(0, tenants, size=rec[-1] + 1 if n else 1)[rec]
    kind = np.where(rng.random(n) < 0.2, 2, 0) if n_tenants > 1 else np.zeros(n, dtype=np.int64)
    if contract and n and n_tenants > 1:
        kind = np.where(rng.random(rec[-1] + 1) < 0.2, 2, 0)[rec]
    hook = (kind | (ten.astype(np.int64) << 8)).astype(np.uint32) if n else np.zeros(0, dtype=np.uint32)
    return gen.records(n, addr=addr, ts=field(64), hook=hook, block_id=field(32).astype(np.uint32),
                       sm_id=field(16).astype(np.uint16), warp_id=field(8).astype(np.uint8),
                       size=field(32).astype(np.uint32))


def map_init(seed: int):
    """Host-written initial contents: (name, keys bytes, values bytes, n) for gx_update_map /
    the oracle's update, flags ANY.  obs: every entry random; hobs: a random half of the keys of
    every tag present; acc/hacc: random (so AND/OR/XOR have something to act on)."""
    rng = np.random.default_rng(seed ^ 0x1A17)
    out = []
    k = np.arange(4096, dtype=np.uint32)
    out.append(("obs", k.tobytes(), rng.integers(0, 1 << 64, size=4096 * 2, dtype=np.uint64).tobytes(), 4096))
    k = np.arange(64, dtype=np.uint32)
    out.append(("acc", k.tobytes(), rng.integers(0, 1 << 64, size=64 * 6, dtype=np.uint64).tobytes(), 64))
    keys = np.concatenate([(rng.permutation(MAX_EVENTS)[:MAX_EVENTS // 2].astype(np.uint64) | np.uint64(t << UBITS))
                           for t in range(4)])
    out.append(("hobs", keys.tobytes(), rng.integers(0, 1 << 64, size=len(keys), dtype=np.uint64).tobytes(), len(keys)))
    hk = rng.permutation(256)[:100].astype(np.uint64)
    out.append(("hacc", hk.tobytes(), rng.integers(0, 1 << 64, size=100, dtype=np.uint64).tobytes(), 100))
    return out
