/*
 * gx_verifier.cpp -- load-time verifier and pre-decoder for gx device programs.
 *
 * Stages:
 *   1. structural decode of every slot (bpf.h:72-77 encoding; BAD_INSN / BAD_REG / SHIFT_RANGE)
 *   2. CFG: jump targets, ldimm64 pairs, reachability (BAD_JUMP / UNREACHABLE)
 *   3. path-sensitive abstract interpretation (Linux-verifier style): register types CTX /
 *      STACK / CONST_MAP / MAP_VALUE(_OR_NULL) / SCALAR, scalars as tnum + u64/s64 intervals,
 *      per-byte stack initialisation with register spills, bounded loops proven by exploring
 *      every path with state pruning (UNBOUNDED_LOOP / COMPLEXITY), every access bounds- and
 *      alignment-checked (OOB_ACCESS / MISALIGNED / NULL_DEREF / UNINIT_READ / PTR_LEAK),
 *      helper prototypes (BAD_HELPER / FORBIDDEN_SYNC), worst-case budgets (BUDGET)
 *      -- PAPER.md:277, 310 ("standard memory safety, bounded loops, and type correctness")
 *   4. SIMT uniformity dataflow: UNINIT < UNIFORM < LANE_VARYING, join = max
 *      (SPEC.md:113, 141); strict-mode rules UNIFORM_BRANCH / UNIFORM_LOOP_BOUND /
 *      UNIFORM_MAP_KEY / NON_UNIFORM_ATOMIC
 *   5. facts for the executor (stack depth, per-map usage classes) and the pre-decoded image.
 * The GPU faults on misaligned accesses, so natural alignment is required everywhere (I-14).
 */
#include "gx_verifier.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

namespace {

/* --------------------------------------------------------------------------- encoding */
enum { CL_LD = 0, CL_LDX = 1, CL_ST = 2, CL_STX = 3, CL_ALU = 4, CL_JMP = 5, CL_JMP32 = 6, CL_ALU64 = 7 };
enum { HASH = 1, ARRAY = 2, PT = 6, RINGBUF = 27, PFQ = GX_MAP_TYPE_PFQ, REGION = GX_MAP_TYPE_REGION };

struct Raw {
    uint8_t code, dst, src;
    int16_t off;
    int32_t imm;
};

inline uint32_t size_of(uint8_t code) {
    static const uint32_t sz[4] = {4, 2, 1, 8};
    return sz[(code >> 3) & 3];
}

/* --------------------------------------------------------------------------- tnum
 * Tristate numbers (value v, unknown-bit mask m) with the published carry-propagation rules for
 * addition and subtraction: the Linux kernel verifier's kernel/bpf/tnum.c (tnum_add / tnum_sub,
 * whose sigma/chi/mu naming is kept here so the two can be compared), proved sound in Vishwanathan
 * et al., "Sound, Precise, and Fast Abstract Interpretation with Tristate Numbers" (CGO 2022). */
struct Tnum {
    uint64_t v, m;
};
inline Tnum tn_const(uint64_t x) { return {x, 0}; }
inline Tnum tn_unknown() { return {0, ~0ull}; }
inline bool tn_is_const(Tnum a) { return a.m == 0; }
inline Tnum tn_add(Tnum a, Tnum b) {
    uint64_t sm = a.m + b.m, sv = a.v + b.v, sigma = sm + sv, chi = sigma ^ sv, mu = chi | a.m | b.m;
    return {sv & ~mu, mu};
}
inline Tnum tn_sub(Tnum a, Tnum b) {
    uint64_t dv = a.v - b.v, alpha = dv + a.m, beta = dv - b.m, chi = alpha ^ beta, mu = chi | a.m | b.m;
    return {dv & ~mu, mu};
}
inline Tnum tn_and(Tnum a, Tnum b) {
    uint64_t alpha = a.v | a.m, beta = b.v | b.m, v = a.v & b.v;
    return {v, alpha & beta & ~v};
}
inline Tnum tn_or(Tnum a, Tnum b) {
    uint64_t v = a.v | b.v, mu = a.m | b.m;
    return {v, mu & ~v};
}
inline Tnum tn_xor(Tnum a, Tnum b) {
    uint64_t v = a.v ^ b.v, mu = a.m | b.m;
    return {v & ~mu, mu};
}
inline Tnum tn_lsh(Tnum a, unsigned k) { return {a.v << k, a.m << k}; }
inline Tnum tn_rsh(Tnum a, unsigned k) { return {a.v >> k, a.m >> k}; }
inline Tnum tn_arsh(Tnum a, unsigned k) {
    return {(uint64_t)((int64_t)a.v >> k), (uint64_t)((int64_t)a.m >> k)};
}
inline Tnum tn_range(uint64_t lo, uint64_t hi) {
    uint64_t chi = lo ^ hi;
    if (!chi) return tn_const(lo);
    int bits = 64 - __builtin_clzll(chi);
    if (bits > 63) return tn_unknown();
    uint64_t delta = (1ull << bits) - 1;
    return {lo & ~delta, delta};
}
inline Tnum tn_intersect(Tnum a, Tnum b) {
    uint64_t v = a.v | b.v, mu = a.m & b.m;
    return {v & ~mu, mu};
}
inline Tnum tn_cast(Tnum a, unsigned bytes) {
    if (bytes >= 8) return a;
    uint64_t msk = (1ull << (8 * bytes)) - 1;
    return {a.v & msk, a.m & msk};
}
inline bool tn_in(Tnum a, Tnum b) { /* b subset of a */
    if (b.m & ~a.m) return false;
    return (b.v & ~a.m) == a.v;
}

/* --------------------------------------------------------------------------- scalar domain */
struct Scalar {
    Tnum t;
    uint64_t umin, umax;
    int64_t smin, smax;
};
inline Scalar sc_const(uint64_t x) { return {tn_const(x), x, x, (int64_t)x, (int64_t)x}; }
inline Scalar sc_unknown() { return {tn_unknown(), 0, ~0ull, INT64_MIN, INT64_MAX}; }
inline Scalar sc_urange(uint64_t lo, uint64_t hi) {
    Scalar s = sc_unknown();
    s.umin = lo;
    s.umax = hi;
    return s;
}
inline bool sc_is_const(const Scalar &s) { return tn_is_const(s.t); }

/* keeps the five views consistent; returns false on contradiction (infeasible path) */
bool sc_sync(Scalar &s) {
    for (int it = 0; it < 3; it++) {
        s.umin = std::max(s.umin, s.t.v);
        s.umax = std::min(s.umax, s.t.v | s.t.m);
        s.smin = std::max(s.smin, (int64_t)(s.t.v | (s.t.m & 0x8000000000000000ull)));
        s.smax = std::min(s.smax, (int64_t)(s.t.v | (s.t.m & 0x7FFFFFFFFFFFFFFFull)));
        if (s.smin >= 0 || s.smax < 0) {
            s.umin = std::max(s.umin, (uint64_t)s.smin);
            s.umax = std::min(s.umax, (uint64_t)s.smax);
        }
        if ((int64_t)s.umax >= 0) { /* no sign crossing in the unsigned range */
            s.smin = std::max(s.smin, (int64_t)s.umin);
            s.smax = std::min(s.smax, (int64_t)s.umax);
        } else if ((int64_t)s.umin < 0) {
            s.smin = std::max(s.smin, (int64_t)s.umin);
            s.smax = std::min(s.smax, (int64_t)s.umax);
        }
        if (s.umin > s.umax || s.smin > s.smax) return false;
        s.t = tn_intersect(s.t, tn_range(s.umin, s.umax));
        if ((s.t.v & s.t.m) != 0) return false;
    }
    return !(s.umin > s.umax || s.smin > s.smax);
}

bool sc_in(const Scalar &a, const Scalar &b) { /* b subset of a */
    return tn_in(a.t, b.t) && b.umin >= a.umin && b.umax <= a.umax && b.smin >= a.smin && b.smax <= a.smax;
}
bool sc_eq(const Scalar &a, const Scalar &b) {
    return a.t.v == b.t.v && a.t.m == b.t.m && a.umin == b.umin && a.umax == b.umax && a.smin == b.smin &&
           a.smax == b.smax;
}

Scalar sc_add(const Scalar &a, const Scalar &b) {
    Scalar r = sc_unknown();
    r.t = tn_add(a.t, b.t);
    uint64_t lo, hi;
    if (!__builtin_add_overflow(a.umax, b.umax, &hi)) {
        lo = a.umin + b.umin;
        r.umin = lo;
        r.umax = hi;
    }
    int64_t slo, shi;
    if (!__builtin_add_overflow(a.smin, b.smin, &slo) && !__builtin_add_overflow(a.smax, b.smax, &shi)) {
        r.smin = slo;
        r.smax = shi;
    }
    sc_sync(r);
    return r;
}
Scalar sc_sub(const Scalar &a, const Scalar &b) {
    Scalar r = sc_unknown();
    r.t = tn_sub(a.t, b.t);
    if (a.umin >= b.umax) {
        r.umin = a.umin - b.umax;
        r.umax = a.umax - b.umin;
    }
    int64_t slo, shi;
    if (!__builtin_sub_overflow(a.smin, b.smax, &slo) && !__builtin_sub_overflow(a.smax, b.smin, &shi)) {
        r.smin = slo;
        r.smax = shi;
    }
    sc_sync(r);
    return r;
}

/* 64-bit ALU transfer on scalars. op = BPF_OP; off distinguishes SDIV/SMOD/MOVSX. */
Scalar sc_alu64(uint32_t op, int16_t off, const Scalar &a, const Scalar &b) {
    if (sc_is_const(a) && sc_is_const(b)) {
        uint64_t d = a.t.v, s = b.t.v, r;
        switch (op) {
        case 0x00: r = d + s; break;
        case 0x10: r = d - s; break;
        case 0x20: r = d * s; break;
        case 0x30:
            if (off == 0) r = s ? d / s : 0;
            else if (s == 0) r = 0;
            else if (d == 0x8000000000000000ull && s == ~0ull) r = d;
            else r = (uint64_t)((int64_t)d / (int64_t)s);
            break;
        case 0x90:
            if (off == 0) r = s ? d % s : d;
            else if (s == 0) r = d;
            else if (s == ~0ull) r = 0;
            else r = (uint64_t)((int64_t)d % (int64_t)s);
            break;
        case 0x40: r = d | s; break;
        case 0x50: r = d & s; break;
        case 0xA0: r = d ^ s; break;
        case 0x60: r = d << (s & 63); break;
        case 0x70: r = d >> (s & 63); break;
        case 0xC0: r = (uint64_t)((int64_t)d >> (s & 63)); break;
        case 0x80: r = 0 - d; break;
        case 0xB0:
            if (off == 0) r = s;
            else {
                uint64_t m = 1ull << (off - 1);
                r = off == 64 ? s : (((s & ((1ull << off) - 1)) ^ m) - m);
            }
            break;
        default: r = 0; return sc_unknown();
        }
        return sc_const(r);
    }
    Scalar r = sc_unknown();
    switch (op) {
    case 0x00: return sc_add(a, b);
    case 0x10: return sc_sub(a, b);
    case 0x80: return sc_sub(sc_const(0), a);
    case 0x20:
        if (a.umax <= 0xFFFFFFFFull && b.umax <= 0xFFFFFFFFull) {
            r.umin = a.umin * b.umin;
            r.umax = a.umax * b.umax;
        }
        break;
    case 0x30:
        if (off == 0) {
            if (sc_is_const(b) && b.t.v) {
                r.umin = a.umin / b.t.v;
                r.umax = a.umax / b.t.v;
            } else {
                r.umin = 0;
                r.umax = a.umax;
            }
        }
        break;
    case 0x90:
        if (off == 0) {
            r.umin = 0;
            r.umax = (sc_is_const(b) && b.t.v) ? std::min(a.umax, b.t.v - 1) : a.umax;
        }
        break;
    case 0x50:
        r.t = tn_and(a.t, b.t);
        r.umax = std::min(a.umax, b.umax);
        if ((int64_t)a.umax >= 0 || (int64_t)b.umax >= 0) r.smin = 0;
        break;
    case 0x40:
        r.t = tn_or(a.t, b.t);
        r.umin = std::max(a.umin, b.umin);
        break;
    case 0xA0: r.t = tn_xor(a.t, b.t); break;
    case 0x60:
        if (sc_is_const(b)) {
            unsigned k = b.t.v & 63;
            r.t = tn_lsh(a.t, k);
            if (k == 0 || a.umax <= (~0ull >> k)) {
                r.umin = a.umin << k;
                r.umax = a.umax << k;
            }
        }
        break;
    case 0x70:
        if (sc_is_const(b)) {
            unsigned k = b.t.v & 63;
            r.t = tn_rsh(a.t, k);
            r.umin = a.umin >> k;
            r.umax = a.umax >> k;
        } else {
            r.umax = a.umax;
            r.umin = 0;
        }
        break;
    case 0xC0:
        if (sc_is_const(b)) {
            unsigned k = b.t.v & 63;
            r.t = tn_arsh(a.t, k);
            r.smin = a.smin >> k;
            r.smax = a.smax >> k;
        }
        break;
    case 0xB0:
        if (off == 0) return b;
        {
            int64_t lo = -(int64_t)(1ull << (off - 1)), hi = (int64_t)(1ull << (off - 1)) - 1;
            if (b.smin >= lo && b.smax <= hi) return b;  /* value already sign-extended */
            if (b.umax <= (uint64_t)hi) return b;
            r.smin = lo;
            r.smax = hi;
        }
        break;
    default: break;
    }
    sc_sync(r);
    return r;
}

Scalar sc_trunc32(const Scalar &a) {
    if (a.umax <= 0xFFFFFFFFull) return a;
    Scalar r = sc_unknown();
    r.t = tn_cast(a.t, 4);
    r.umin = 0;
    r.umax = 0xFFFFFFFFull;
    sc_sync(r);
    return r;
}
Scalar sc_sext32(const Scalar &a32) { /* a32 is a zero-extended 32-bit value */
    if (sc_is_const(a32)) return sc_const((uint64_t)(int64_t)(int32_t)(uint32_t)a32.t.v);
    if (a32.umax <= 0x7FFFFFFFull) return a32;
    Scalar r = sc_unknown();
    r.smin = INT32_MIN;
    r.smax = INT32_MAX;
    sc_sync(r);
    return r;
}

/* 32-bit ALU: operate on the zero-extended low halves, result zero-extended (I-6). */
Scalar sc_alu32(uint32_t op, int16_t off, const Scalar &a64, const Scalar &b64) {
    Scalar a = sc_trunc32(a64), b = sc_trunc32(b64);
    if (sc_is_const(a) && sc_is_const(b)) {
        uint32_t d = (uint32_t)a.t.v, s = (uint32_t)b.t.v, r;
        switch (op) {
        case 0x00: r = d + s; break;
        case 0x10: r = d - s; break;
        case 0x20: r = d * s; break;
        case 0x30:
            if (off == 0) r = s ? d / s : 0;
            else if (s == 0) r = 0;
            else if (d == 0x80000000u && s == 0xFFFFFFFFu) r = d;
            else r = (uint32_t)((int32_t)d / (int32_t)s);
            break;
        case 0x90:
            if (off == 0) r = s ? d % s : d;
            else if (s == 0) r = d;
            else if (s == 0xFFFFFFFFu) r = 0;
            else r = (uint32_t)((int32_t)d % (int32_t)s);
            break;
        case 0x40: r = d | s; break;
        case 0x50: r = d & s; break;
        case 0xA0: r = d ^ s; break;
        case 0x60: r = d << (s & 31); break;
        case 0x70: r = d >> (s & 31); break;
        case 0xC0: r = (uint32_t)((int32_t)d >> (s & 31)); break;
        case 0x80: r = 0u - d; break;
        case 0xB0:
            if (off == 0) r = s;
            else if (off == 8) r = (uint32_t)(int32_t)(int8_t)s;
            else r = (uint32_t)(int32_t)(int16_t)s;
            break;
        default: return sc_urange(0, 0xFFFFFFFFull);
        }
        return sc_const(r);
    }
    Scalar r;
    switch (op) {
    case 0x00: case 0x10: case 0x20: case 0x40: case 0x50: case 0xA0: case 0x60:
        r = sc_alu64(op, 0, a, b);
        break;
    case 0x80: r = sc_sub(sc_const(0), a); break;
    case 0x30: case 0x90:
        r = off == 0 ? sc_alu64(op, 0, a, b) : sc_urange(0, 0xFFFFFFFFull);
        break;
    case 0x70:
        r = sc_alu64(op, 0, a, sc_is_const(b) ? sc_const(b.t.v & 31) : b);
        break;
    case 0xC0:
        if (sc_is_const(b)) {
            r = sc_alu64(0xC0, 0, sc_sext32(a), sc_const(b.t.v & 31));
        } else {
            r = sc_unknown();
        }
        break;
    case 0xB0:
        if (off == 0) r = b;
        else r = sc_alu64(0xB0, off, sc_unknown(), b);
        break;
    default: r = sc_unknown();
    }
    return sc_trunc32(r);
}

/* --------------------------------------------------------------------------- registers */
enum RType : uint8_t { NOT_INIT = 0, SCALAR, PTR_CTX, PTR_STACK, CONST_MAP, PTR_MAPV, PTR_MAPV_OR_NULL };

struct Reg {
    RType type = NOT_INIT;
    int16_t map = -1;
    uint32_t id = 0;     /* MAPV_OR_NULL identity */
    int64_t off = 0;     /* fixed pointer offset */
    Scalar var{};        /* SCALAR value, or the variable part of a pointer offset */
};

inline Reg reg_scalar(const Scalar &s) {
    Reg r;
    r.type = SCALAR;
    r.var = s;
    return r;
}
inline bool is_ptr(const Reg &r) { return r.type >= PTR_CTX; }

struct Slot {
    uint8_t init = 0;   /* bit k: byte k initialised */
    bool spill = false; /* a full 8-byte register spill */
    Reg reg;
    /* 4-byte scalar stores (e.g. a map key written with stxw): bit h = half h holds a value known
     * to be <= nmax[h].  Lets a lookup with a provably in-range key return a non-NULL pointer. */
    uint8_t nok = 0;
    uint64_t nmax[2] = {0, 0};
};

struct State {
    Reg r[11];
    Slot s[GX_STACK_SIZE / 8];
};

bool reg_in(const Reg &a, const Reg &b, std::vector<std::pair<uint32_t, uint32_t>> &idmap) {
    /* does old register a subsume current register b? */
    if (a.type == NOT_INIT) return true;
    if (a.type != b.type) return false;
    switch (a.type) {
    case SCALAR: return sc_in(a.var, b.var);
    case PTR_CTX: case PTR_STACK: return a.off == b.off && sc_in(a.var, b.var);
    case CONST_MAP: return a.map == b.map;
    case PTR_MAPV: return a.map == b.map && a.off == b.off && sc_in(a.var, b.var);
    case PTR_MAPV_OR_NULL:
        if (a.map != b.map || a.off != b.off || !sc_in(a.var, b.var)) return false;
        for (auto &p : idmap) {
            if (p.first == a.id) return p.second == b.id;
            if (p.second == b.id) return false;
        }
        idmap.push_back({a.id, b.id});
        return true;
    default: return false;
    }
}
bool reg_eq(const Reg &a, const Reg &b) {
    if (a.type != b.type) return false;
    if (a.type == NOT_INIT) return true;
    if (a.type == CONST_MAP) return a.map == b.map;
    return a.map == b.map && a.off == b.off && sc_eq(a.var, b.var);
}

bool state_in(const State &a, const State &b) {
    std::vector<std::pair<uint32_t, uint32_t>> idmap;
    for (int i = 0; i < 11; i++)
        if (!reg_in(a.r[i], b.r[i], idmap)) return false;
    for (int k = 0; k < GX_STACK_SIZE / 8; k++) {
        const Slot &x = a.s[k], &y = b.s[k];
        if (!x.init) continue;
        if ((x.init & y.init) != x.init) return false;
        if (x.spill) {
            if (!y.spill) {
                if (x.reg.type == SCALAR && sc_eq(x.reg.var, sc_unknown())) continue;
                return false;
            }
            if (!reg_in(x.reg, y.reg, idmap)) return false;
        } else if (y.spill && y.reg.type != SCALAR) {
            return false; /* old read these bytes as plain bytes; a pointer there would leak */
        }
        for (int h = 0; h < 2; h++) /* an old bound must still hold */
            if (((x.nok >> h) & 1) && (!((y.nok >> h) & 1) || y.nmax[h] > x.nmax[h])) return false;
    }
    return true;
}
bool state_eq(const State &a, const State &b) {
    for (int i = 0; i < 11; i++)
        if (!reg_eq(a.r[i], b.r[i])) return false;
    for (int k = 0; k < GX_STACK_SIZE / 8; k++) {
        const Slot &x = a.s[k], &y = b.s[k];
        if (x.init != y.init || x.spill != y.spill || x.nok != y.nok) return false;
        if (x.spill && !reg_eq(x.reg, y.reg)) return false;
        for (int h = 0; h < 2; h++)
            if (((x.nok >> h) & 1) && x.nmax[h] != y.nmax[h]) return false;
    }
    return true;
}

/* --------------------------------------------------------------------------- per-insn facts */
enum MemKind : uint8_t { MK_NONE = 0, MK_CTX, MK_STACK, MK_MAPV, MK_PTV };

struct Fact {
    bool seen = false;
    MemKind kind = MK_NONE;      /* memory insns: pointer kind of the base register */
    int16_t map = -1;            /* MAPV / PTV / helper map */
    int32_t stack_addr = 0;      /* STACK: byte address in [0,512) */
    /* helper args */
    MemKind key_kind = MK_NONE, val_kind = MK_NONE;
    int32_t key_addr = 0, val_addr = 0;
    int64_t rb_size = -1, rb_flags = -1;
    uint8_t br = 0;              /* conditional jumps: 1 = taken on some path, 2 = fell through on some path */
    bool pt_vstart = false;      /* PTV memory insns: the base register is a value start (no offset) on every path */
    uint8_t narrow = 0;          /* scalar ALU64: 1 = operands and result below 2^32 on every path, 2 = not */
    uint8_t inrange = 0;         /* ARRAY / PERTHREAD lookups: 1 = key below max_entries on every path, 2 = not */
    bool nin_seen = false;
    uint16_t nin = 0;            /* registers r0..r9 that are scalars below 2^32 on entry, every path */
};

struct Checkpoint {
    State st;
    Checkpoint *parent = nullptr;
    int branches = 0;
    uint64_t ci = 0, ch = 0, cm = 0;            /* counts when the path reached this checkpoint */
    uint64_t ri = 0, rh = 0, rm = 0;            /* max remaining counts to an exit */
};

struct Path {
    State st;
    uint32_t pc = 0;
    Checkpoint *parent = nullptr;
    uint64_t ci = 0, ch = 0, cm = 0;
};

struct Violation {
    uint32_t insn, rule;
    std::string msg;
};

const char *kRuleNames[GX_NUM_RULES] = {
    "OK", "BAD_INSN", "BAD_REG", "BAD_JUMP", "FALLTHROUGH", "UNREACHABLE", "UNINIT_READ", "OOB_ACCESS",
    "NULL_DEREF", "MISALIGNED", "PTR_LEAK", "SHIFT_RANGE", "BAD_HELPER", "FORBIDDEN_SYNC", "UNBOUNDED_LOOP",
    "COMPLEXITY", "BUDGET", "UNIFORM_BRANCH", "UNIFORM_LOOP_BOUND", "UNIFORM_MAP_KEY", "NON_UNIFORM_ATOMIC",
    "MIXED_PTR"};

struct Verifier {
    const uint8_t *slots;
    uint32_t n;
    const GxMapInfo *maps;
    gx_verify_opts opts;
    GxVerifyResult &out;
    std::vector<Raw> ins;
    std::vector<uint8_t> is_second;  /* second slot of an ldimm64 */
    std::vector<uint8_t> prune_pt;
    std::vector<Fact> facts;
    std::vector<std::vector<Checkpoint *>> visited;
    std::vector<std::unique_ptr<Checkpoint>> pool;
    std::vector<Violation> viol;
    uint64_t processed = 0;
    uint64_t worst_i = 0, worst_h = 0, worst_m = 0;
    uint32_t next_id = 1;
    uint32_t max_stack = 0;          /* deepest stack byte touched (bytes below fp) */

    Verifier(const uint8_t *s, uint32_t n_, const GxMapInfo *m, const gx_verify_opts &o, GxVerifyResult &r)
        : slots(s), n(n_), maps(m), opts(o), out(r) {}

    bool fail(uint32_t pc, uint32_t rule, const std::string &msg) {
        viol.push_back({pc, rule, msg});
        return false;
    }

    /* ---------------------------------------------------------------- stage 1+2 */
    bool structural() {
        if (n == 0) return fail(0, GX_BAD_INSN, "empty program");
        if (n > 4096) return fail(0, GX_BAD_INSN, "more than BPF_MAXINSNS (4096) slots");
        ins.resize(n);
        is_second.assign(n, 0);
        for (uint32_t i = 0; i < n; i++) {
            const uint8_t *b = slots + 8 * i;
            Raw &r = ins[i];
            r.code = b[0];
            r.dst = b[1] & 0xF;
            r.src = b[1] >> 4;
            memcpy(&r.off, b + 2, 2);
            memcpy(&r.imm, b + 4, 4);
        }
        for (uint32_t i = 0; i < n; i++) {
            const Raw &r = ins[i];
            if (is_second[i]) continue;
            uint32_t cls = r.code & 7;
            char msg[96];
            if (r.dst > 10 || r.src > 10) return fail(i, GX_BAD_REG, "register number > 10");
            if (cls == CL_LD) {
                if (r.code != 0x18) return fail(i, GX_BAD_INSN, "LD ABS/IND and non-ldimm64 LD are not supported");
                if (i + 1 >= n) return fail(i, GX_BAD_INSN, "ldimm64 truncated");
                const Raw &r2 = ins[i + 1];
                if (r2.code || r2.dst || r2.src || r2.off) return fail(i, GX_BAD_INSN, "ldimm64 second slot not zero");
                if (r.off) return fail(i, GX_BAD_INSN, "ldimm64 off != 0");
                if (r.src > 2) return fail(i, GX_BAD_INSN, "unsupported ldimm64 pseudo source");
                if (r.dst == 10) return fail(i, GX_BAD_REG, "write to r10");
                if (r.src != 0) {
                    if (r.imm < 0 || r.imm >= GX_MAX_MAPS || !maps[r.imm].valid)
                        return fail(i, GX_BAD_INSN, "ldimm64 references an unknown map fd");
                    const GxMapInfo &mi = maps[r.imm];
                    if (r.src == 2) {
                        if (mi.type != ARRAY || mi.max_entries != 1)
                            return fail(i, GX_BAD_INSN, "BPF_PSEUDO_MAP_VALUE needs a 1-entry ARRAY");
                        if ((uint32_t)r2.imm >= mi.value_size)
                            return fail(i, GX_BAD_INSN, "map_value offset outside the value");
                    } else if (r2.imm) {
                        return fail(i, GX_BAD_INSN, "map fd ldimm64 with nonzero upper imm");
                    }
                }
                is_second[i + 1] = 1;
                continue;
            }
            if (cls == CL_ALU || cls == CL_ALU64) {
                uint32_t op = r.code & 0xF0;
                bool x = r.code & 0x08;
                if (op > 0xD0) return fail(i, GX_BAD_INSN, "unknown ALU op");
                if (r.dst == 10) return fail(i, GX_BAD_REG, "write to r10");
                if (op == 0xD0) {
                    if (r.src || r.off || (r.imm != 16 && r.imm != 32 && r.imm != 64))
                        return fail(i, GX_BAD_INSN, "bad END/BSWAP");
                    if (cls == CL_ALU64 && x) return fail(i, GX_BAD_INSN, "BSWAP has no X form");
                    continue;
                }
                if (op == 0x80) {
                    if (x || r.src || r.off || r.imm) return fail(i, GX_BAD_INSN, "bad NEG");
                    continue;
                }
                if (x) {
                    if (r.imm) return fail(i, GX_BAD_INSN, "X-form ALU with nonzero imm");
                } else if (r.src) {
                    return fail(i, GX_BAD_INSN, "K-form ALU with nonzero src");
                }
                if (op == 0x30 || op == 0x90) {
                    if (r.off != 0 && r.off != 1) return fail(i, GX_BAD_INSN, "bad SDIV/SMOD off");
                    if (!x && r.imm == 0) return fail(i, GX_BAD_INSN, "division by zero immediate");
                } else if (op == 0xB0) {
                    if (r.off) {
                        if (!x) return fail(i, GX_BAD_INSN, "MOVSX has no K form");
                        bool ok = cls == CL_ALU64 ? (r.off == 8 || r.off == 16 || r.off == 32)
                                                  : (r.off == 8 || r.off == 16);
                        if (!ok) return fail(i, GX_BAD_INSN, "bad MOVSX width");
                    }
                } else if (r.off) {
                    return fail(i, GX_BAD_INSN, "nonzero off in ALU");
                }
                if ((op == 0x60 || op == 0x70 || op == 0xC0) && !x) {
                    int W = cls == CL_ALU64 ? 64 : 32;
                    if (r.imm < 0 || r.imm >= W) {
                        snprintf(msg, sizeof msg, "immediate shift %d >= %d", r.imm, W);
                        return fail(i, GX_SHIFT_RANGE, msg);
                    }
                }
                continue;
            }
            if (cls == CL_JMP || cls == CL_JMP32) {
                uint32_t op = r.code & 0xF0;
                bool x = r.code & 0x08;
                if (op == 0xE0 || op == 0xF0) return fail(i, GX_BAD_INSN, "unknown jump op");
                if (op == 0x80) {
                    if (cls != CL_JMP || x || r.dst || r.off) return fail(i, GX_BAD_INSN, "bad CALL");
                    if (r.src == 1 || r.src == 2) return fail(i, GX_BAD_INSN, "bpf-to-bpf and kfunc calls are not supported");
                    if (r.src) return fail(i, GX_BAD_INSN, "bad CALL src");
                    continue;
                }
                if (op == 0x90) {
                    if (cls != CL_JMP || x || r.dst || r.src || r.off || r.imm) return fail(i, GX_BAD_INSN, "bad EXIT");
                    continue;
                }
                if (op == 0x00) {
                    if (cls != CL_JMP) return fail(i, GX_BAD_INSN, "gotol (JMP32 JA) is not supported");
                    if (x || r.dst || r.src || r.imm) return fail(i, GX_BAD_INSN, "bad JA");
                } else if (x ? r.imm != 0 : r.src != 0) {
                    return fail(i, GX_BAD_INSN, "reserved field set in jump");
                }
                int64_t t = (int64_t)i + 1 + r.off;
                if (t < 0 || t >= (int64_t)n) return fail(i, GX_BAD_JUMP, "jump target outside the program");
                continue;
            }
            if (cls == CL_LDX) {
                uint32_t mode = r.code & 0xE0;
                if (mode != 0x60 && mode != 0x80) return fail(i, GX_BAD_INSN, "bad LDX mode");
                if (mode == 0x80 && size_of(r.code) == 8) return fail(i, GX_BAD_INSN, "MEMSX DW does not exist");
                if (r.imm) return fail(i, GX_BAD_INSN, "LDX with nonzero imm");
                if (r.dst == 10) return fail(i, GX_BAD_REG, "write to r10");
                continue;
            }
            if (cls == CL_ST) {
                if ((r.code & 0xE0) != 0x60) return fail(i, GX_BAD_INSN, "bad ST mode");
                if (r.src) return fail(i, GX_BAD_INSN, "ST with nonzero src");
                continue;
            }
            if (cls == CL_STX) {
                uint32_t mode = r.code & 0xE0;
                if (mode == 0x60) {
                    if (r.imm) return fail(i, GX_BAD_INSN, "STX with nonzero imm");
                    continue;
                }
                if (mode == 0xC0) {
                    uint32_t sz = size_of(r.code);
                    if (sz != 4 && sz != 8) return fail(i, GX_BAD_INSN, "B/H atomics are not supported");
                    switch (r.imm) {
                    case 0x00: case 0x01: case 0x40: case 0x41: case 0x50: case 0x51: case 0xA0: case 0xA1:
                    case 0xE1: case 0xF1: break;
                    default: return fail(i, GX_BAD_INSN, "unknown atomic op");
                    }
                    continue;
                }
                return fail(i, GX_BAD_INSN, "bad STX mode");
            }
            return fail(i, GX_BAD_INSN, "unknown instruction class");
        }
        /* jumps into the second slot of ldimm64; CFG reachability; prune points */
        prune_pt.assign(n, 0);
        std::vector<uint8_t> reach(n, 0);
        std::vector<uint32_t> work{0};
        reach[0] = 1;
        while (!work.empty()) {
            uint32_t i = work.back();
            work.pop_back();
            const Raw &r = ins[i];
            uint32_t cls = r.code & 7, op = r.code & 0xF0;
            std::vector<uint32_t> succ;
            if (cls == CL_JMP || cls == CL_JMP32) {
                if (op == 0x90) continue;
                if (op == 0x80) succ.push_back(i + 1);
                else {
                    uint32_t t = i + 1 + r.off;
                    if (is_second[t]) return fail(i, GX_BAD_JUMP, "jump into the middle of ldimm64");
                    prune_pt[t] = 1;
                    succ.push_back(t);
                    if (op != 0x00) {
                        succ.push_back(i + 1);
                        if (i + 1 < n) prune_pt[i + 1] = 1;
                    }
                }
            } else if (cls == CL_LD) {
                succ.push_back(i + 2);
            } else {
                succ.push_back(i + 1);
            }
            for (uint32_t s : succ) {
                if (s >= n) return fail(i, GX_FALLTHROUGH, "control falls off the end of the program");
                if (!reach[s]) {
                    reach[s] = 1;
                    work.push_back(s);
                }
            }
        }
        for (uint32_t i = 0; i < n; i++)
            if (!reach[i] && !is_second[i]) return fail(i, GX_UNREACHABLE, "unreachable instruction");
        return true;
    }

    /* ---------------------------------------------------------------- stage 3 helpers */
    bool last_vstart = false;    /* set by check_access: the map value pointer has no offset */
    bool record_mem(uint32_t pc, MemKind k, int map, int32_t saddr) {
        Fact &f = facts[pc];
        if (!f.seen) {
            f.seen = true;
            f.kind = k;
            f.map = (int16_t)map;
            f.stack_addr = saddr;
            f.pt_vstart = k == MK_PTV && last_vstart;
            return true;
        }
        if (k == MK_PTV && !last_vstart) f.pt_vstart = false;
        if (f.kind != k || f.map != map || (k == MK_STACK && f.stack_addr != saddr))
            return fail(pc, GX_MIXED_PTR, "the same instruction accesses different pointer kinds/maps/stack offsets on different paths");
        return true;
    }

    /* checks an access of `size` bytes at reg + off; returns the memory kind */
    bool check_access(uint32_t pc, const Reg &p, int64_t off, uint32_t size, bool write, MemKind &kind,
                      int32_t &saddr, int &map) {
        char msg[128];
        saddr = 0;
        map = -1;
        switch (p.type) {
        case NOT_INIT: return fail(pc, GX_UNINIT_READ, "base register is not initialised");
        case SCALAR: return fail(pc, GX_OOB_ACCESS, "memory access through a scalar");
        case CONST_MAP: return fail(pc, GX_OOB_ACCESS, "memory access through a map handle");
        case PTR_MAPV_OR_NULL: return fail(pc, GX_NULL_DEREF, "map value pointer used before the NULL check");
        case PTR_CTX: {
            if (write) return fail(pc, GX_OOB_ACCESS, "write to the read-only ctx");
            if (p.off != 0 || !sc_is_const(p.var) || p.var.t.v != 0)
                return fail(pc, GX_OOB_ACCESS, "dereference of a modified ctx pointer");
            if (off < 0 || off + size > 32) {
                snprintf(msg, sizeof msg, "ctx access [%lld,+%u) outside [0,32)", (long long)off, size);
                return fail(pc, GX_OOB_ACCESS, msg);
            }
            if (off % size) return fail(pc, GX_MISALIGNED, "misaligned ctx access");
            kind = MK_CTX;
            saddr = (int32_t)off;
            return true;
        }
        case PTR_STACK: {
            if (!sc_is_const(p.var)) return fail(pc, GX_OOB_ACCESS, "variable-offset stack access");
            int64_t a = p.off + (int64_t)p.var.t.v + off; /* relative to fp */
            if (a < -GX_STACK_SIZE || a + (int64_t)size > 0) {
                snprintf(msg, sizeof msg, "stack access at fp%+lld size %u outside [-512,0)", (long long)a, size);
                return fail(pc, GX_OOB_ACCESS, msg);
            }
            if (a % (int64_t)size) return fail(pc, GX_MISALIGNED, "misaligned stack access");
            kind = MK_STACK;
            saddr = (int32_t)(a + GX_STACK_SIZE);
            max_stack = std::max<uint32_t>(max_stack, (uint32_t)(-a));
            return true;
        }
        case PTR_MAPV: {
            const GxMapInfo &mi = maps[p.map];
            int64_t lo = p.off + off + p.var.smin, hi = p.off + off + p.var.smax;
            if (p.var.smin < -(1ll << 30) || p.var.smax > (1ll << 30) || lo < 0 || hi + (int64_t)size > (int64_t)mi.value_size) {
                snprintf(msg, sizeof msg, "map value access [%lld,%lld]+%u outside [0,%u)", (long long)lo, (long long)hi,
                         size, mi.value_size);
                return fail(pc, GX_OOB_ACCESS, msg);
            }
            Tnum t = tn_add(tn_const((uint64_t)(p.off + off)), p.var.t);
            if ((t.v | t.m) & (size - 1)) return fail(pc, GX_MISALIGNED, "map value access not naturally aligned");
            kind = mi.type == PT ? MK_PTV : MK_MAPV;
            map = p.map;
            last_vstart = p.off == 0 && sc_is_const(p.var) && p.var.t.v == 0;
            return true;
        }
        default: return fail(pc, GX_OOB_ACCESS, "bad pointer");
        }
    }

    /* stack byte range [a, a+len) (fp-relative) must be initialised plain bytes (helper reads) */
    bool check_stack_read_bytes(uint32_t pc, State &st, int64_t a, uint32_t len, const char *what) {
        char msg[128];
        if (a < -GX_STACK_SIZE || a + (int64_t)len > 0) {
            snprintf(msg, sizeof msg, "%s at fp%+lld (%u bytes) outside the stack", what, (long long)a, len);
            return fail(pc, GX_OOB_ACCESS, msg);
        }
        max_stack = std::max<uint32_t>(max_stack, (uint32_t)(-a));
        for (int64_t b = a; b < a + (int64_t)len; b++) {
            int64_t x = b + GX_STACK_SIZE;
            Slot &s = st.s[x / 8];
            if (!(s.init >> (x % 8) & 1)) {
                snprintf(msg, sizeof msg, "%s reads uninitialised stack at fp%+lld", what, (long long)b);
                return fail(pc, GX_UNINIT_READ, msg);
            }
            if (s.spill && is_ptr(s.reg)) {
                snprintf(msg, sizeof msg, "%s would read a spilled pointer (leak)", what);
                return fail(pc, GX_PTR_LEAK, msg);
            }
        }
        return true;
    }

    /* helper memory argument: pointer to `len` readable bytes */
    bool check_arg_mem(uint32_t pc, State &st, const Reg &p, uint32_t len, uint32_t align, const char *what,
                       MemKind &kind, int32_t &addr) {
        char msg[128];
        if (p.type == PTR_STACK) {
            if (!sc_is_const(p.var)) return fail(pc, GX_OOB_ACCESS, "variable-offset stack helper argument");
            int64_t a = p.off + (int64_t)p.var.t.v;
            if (a % align) {
                snprintf(msg, sizeof msg, "%s must be %u-byte aligned on the stack", what, align);
                return fail(pc, GX_MISALIGNED, msg);
            }
            if (!check_stack_read_bytes(pc, st, a, len, what)) return false;
            kind = MK_STACK;
            addr = (int32_t)(a + GX_STACK_SIZE);
            return true;
        }
        if (p.type == PTR_MAPV) {
            const GxMapInfo &mi = maps[p.map];
            if (mi.type == PT) {
                snprintf(msg, sizeof msg, "%s pointing into a per-thread map is not supported", what);
                return fail(pc, GX_BAD_HELPER, msg);
            }
            int64_t lo = p.off + p.var.smin, hi = p.off + p.var.smax;
            if (lo < 0 || hi + (int64_t)len > (int64_t)mi.value_size) {
                snprintf(msg, sizeof msg, "%s outside the map value", what);
                return fail(pc, GX_OOB_ACCESS, msg);
            }
            Tnum t = tn_add(tn_const((uint64_t)p.off), p.var.t);
            if ((t.v | t.m) & (align - 1)) return fail(pc, GX_MISALIGNED, "helper argument not naturally aligned");
            kind = MK_MAPV;
            addr = 0;
            return true;
        }
        if (p.type == PTR_MAPV_OR_NULL) return fail(pc, GX_NULL_DEREF, "possibly-NULL pointer passed to a helper");
        if (p.type == NOT_INIT) return fail(pc, GX_UNINIT_READ, "helper argument register not initialised");
        snprintf(msg, sizeof msg, "%s must point to the stack or a map value", what);
        return fail(pc, GX_BAD_HELPER, msg);
    }

    /* upper bound of the u32 key at stack byte address ka (0..511), if one is known */
    static bool key_bound(const State &st, int32_t ka, uint64_t &kmax) {
        if (ka < 0 || ka + 4 > GX_STACK_SIZE || ka % 4) return false;
        const Slot &s = st.s[ka / 8];
        const int h = (ka % 8) / 4;
        if (s.spill) {
            if (is_ptr(s.reg) || s.reg.var.umax > 0xFFFFFFFFull) return false;
            kmax = h == 0 ? s.reg.var.umax : 0;
            return true;
        }
        if (!((s.nok >> h) & 1)) return false;
        kmax = s.nmax[h];
        return true;
    }

    bool record_call(uint32_t pc, int map, MemKind kk, int32_t ka, MemKind vk, int32_t va, int64_t rbs, int64_t rbf) {
        Fact &f = facts[pc];
        if (!f.seen) {
            f.seen = true;
            f.map = (int16_t)map;
            f.key_kind = kk;
            f.key_addr = ka;
            f.val_kind = vk;
            f.val_addr = va;
            f.rb_size = rbs;
            f.rb_flags = rbf;
            return true;
        }
        if (f.map != map || f.key_kind != kk || f.key_addr != ka || f.val_kind != vk || f.val_addr != va ||
            f.rb_size != rbs || f.rb_flags != rbf)
            return fail(pc, GX_MIXED_PTR, "helper call site sees different maps/argument locations on different paths");
        return true;
    }

    void stack_write(State &st, int64_t a, uint32_t size, const Reg *val) {
        int64_t x = a + GX_STACK_SIZE;
        Slot &s = st.s[x / 8];
        if (size == 8 && val) {
            s.spill = true;
            s.reg = *val;
            s.init = 0xFF;
            s.nok = 0;
            return;
        }
        uint8_t bits = (uint8_t)(((1u << size) - 1) << (x % 8));
        if (s.spill && is_ptr(s.reg)) s.init = 0;  /* the rest of a clobbered pointer is garbage */
        if (s.spill && !is_ptr(s.reg) && s.reg.var.umax <= 0xFFFFFFFFull) {
            /* the untouched half of a small spilled scalar keeps its bound */
            s.nok = 3;
            s.nmax[0] = s.reg.var.umax;
            s.nmax[1] = 0;
        } else if (s.spill) {
            s.nok = 0;
        }
        s.spill = false;
        s.init |= bits;
        const int h0 = (int)(x % 8) / 4, h1 = (int)((x % 8) + size - 1) / 4;
        for (int h = h0; h <= h1; h++) s.nok &= (uint8_t)~(1u << h);
        if (size == 4 && x % 4 == 0 && val && val->type == SCALAR && val->var.umax <= 0xFFFFFFFFull) {
            s.nok |= (uint8_t)(1u << h0);
            s.nmax[h0] = val->var.umax;
        }
    }

    Reg stack_read(State &st, int64_t a, uint32_t size, bool sx, uint32_t pc, bool &ok) {
        ok = true;
        int64_t x = a + GX_STACK_SIZE;
        Slot &s = st.s[x / 8];
        uint8_t bits = (uint8_t)(((1u << size) - 1) << (x % 8));
        if ((s.init & bits) != bits) {
            ok = fail(pc, GX_UNINIT_READ, "read of uninitialised stack");
            return Reg{};
        }
        if (s.spill) {
            if (size == 8 && !sx) return s.reg;
            if (is_ptr(s.reg)) {
                ok = fail(pc, GX_PTR_LEAK, "partial read of a spilled pointer");
                return Reg{};
            }
            if (sc_is_const(s.reg.var)) {
                uint64_t v = s.reg.var.t.v >> (8 * (x % 8));
                if (size < 8) v &= (1ull << (8 * size)) - 1;
                if (sx) {
                    uint64_t m = 1ull << (8 * size - 1);
                    v = (v ^ m) - m;
                }
                return reg_scalar(sc_const(v));
            }
        }
        if (!sx && size == 4 && x % 4 == 0 && !s.spill && ((s.nok >> ((x % 8) / 4)) & 1))
            return reg_scalar(sc_urange(0, s.nmax[(x % 8) / 4]));
        if (sx) {
            Scalar r = sc_unknown();
            r.smin = -(int64_t)(1ull << (8 * size - 1));
            r.smax = (int64_t)(1ull << (8 * size - 1)) - 1;
            sc_sync(r);
            return reg_scalar(r);
        }
        return reg_scalar(size == 8 ? sc_unknown() : sc_urange(0, (1ull << (8 * size)) - 1));
    }

    /* ---------------------------------------------------------------- one instruction
     * Returns: 0 continue at pc (updated), 1 path ended (exit), -1 violation.
     * For conditional jumps it may push the other branch onto `pending`. */
    int step(Path &P, std::vector<Path> &pending) {
        uint32_t pc = P.pc;
        State &st = P.st;
        {
            uint16_t m = 0;
            for (int k = 0; k < 10; k++)
                if (st.r[k].type == SCALAR && st.r[k].var.umax < (1ull << 32)) m |= (uint16_t)(1u << k);
            Fact &fn = facts[pc];
            fn.nin = fn.nin_seen ? (uint16_t)(fn.nin & m) : m;
            fn.nin_seen = true;
        }
        const Raw &r = ins[pc];
        uint32_t cls = r.code & 7, op = r.code & 0xF0;
        bool x = r.code & 0x08;
        Reg &D = st.r[r.dst];
        Reg &S = st.r[r.src];
        char msg[160];

        if (cls == CL_ALU || cls == CL_ALU64) {
            bool is64 = cls == CL_ALU64;
            if (op == 0xD0) {
                if (D.type != SCALAR) return fail(pc, D.type == NOT_INIT ? GX_UNINIT_READ : GX_PTR_LEAK, "END on a non-scalar") ? 0 : -1;
                uint32_t w = (uint32_t)r.imm;
                bool swap = is64 || x;
                if (sc_is_const(D.var)) {
                    uint64_t v = D.var.t.v, o = 0;
                    if (swap) for (uint32_t k = 0; k < w / 8; k++) o |= ((v >> (8 * k)) & 0xFF) << (w - 8 - 8 * k);
                    else o = w == 64 ? v : v & ((1ull << w) - 1);
                    D.var = sc_const(o);
                } else if (!swap) {
                    D.var = sc_alu64(0x50, 0, D.var, sc_const(w == 64 ? ~0ull : (1ull << w) - 1));
                } else {
                    D.var = w == 64 ? sc_unknown() : sc_urange(0, (1ull << w) - 1);
                }
                P.pc++;
                return 0;
            }
            Reg src;
            if (op == 0x80) src = reg_scalar(sc_const(0));
            else if (x) {
                src = S;
                if (src.type == NOT_INIT) return fail(pc, GX_UNINIT_READ, "source register not initialised") ? 0 : -1;
            } else {
                src = reg_scalar(sc_const(is64 ? (uint64_t)(int64_t)r.imm : (uint64_t)(uint32_t)r.imm));
            }
            if (op == 0xB0 && r.off == 0) { /* MOV */
                if (!is64 && is_ptr(src)) return fail(pc, GX_PTR_LEAK, "32-bit move of a pointer") ? 0 : -1;
                if (is64) { /* narrow: a scalar below 2^32 (the JIT zero-extends explicitly) */
                    Fact &f = facts[pc];
                    f.narrow = (f.narrow != 2 && src.type == SCALAR && src.var.umax < (1ull << 32)) ? 1 : 2;
                }
                D = src;
                if (!is64) D.var = sc_trunc32(D.var);
                P.pc++;
                return 0;
            }
            if (op != 0x80 && D.type == NOT_INIT) return fail(pc, GX_UNINIT_READ, "destination register not initialised") ? 0 : -1;
            if (op == 0x80 && D.type == NOT_INIT) return fail(pc, GX_UNINIT_READ, "NEG of an uninitialised register") ? 0 : -1;
            bool dp = is_ptr(D), sp = is_ptr(src);
            if (dp || sp) {
                if (!is64) return fail(pc, GX_PTR_LEAK, "32-bit ALU on a pointer") ? 0 : -1;
                if ((dp && D.type == PTR_MAPV_OR_NULL) || (sp && src.type == PTR_MAPV_OR_NULL))
                    return fail(pc, GX_NULL_DEREF, "arithmetic on a possibly-NULL map value pointer") ? 0 : -1;
                if ((dp && D.type == CONST_MAP) || (sp && src.type == CONST_MAP))
                    return fail(pc, GX_PTR_LEAK, "arithmetic on a map handle") ? 0 : -1;
                if (op == 0x00 && dp != sp) {
                    Reg p = dp ? D : src;
                    const Scalar &k = dp ? src.var : D.var;
                    if (sc_is_const(k)) p.off += (int64_t)k.t.v;
                    else p.var = sc_add(p.var, k);
                    if (p.off < -(1ll << 30) || p.off > (1ll << 30)) return fail(pc, GX_OOB_ACCESS, "pointer offset out of range") ? 0 : -1;
                    D = p;
                } else if (op == 0x10 && dp && !sp) {
                    if (sc_is_const(src.var)) D.off -= (int64_t)src.var.t.v;
                    else D.var = sc_sub(D.var, src.var);
                    if (D.off < -(1ll << 30) || D.off > (1ll << 30)) return fail(pc, GX_OOB_ACCESS, "pointer offset out of range") ? 0 : -1;
                } else if (op == 0x10 && dp && sp && D.type == src.type && (D.type == PTR_STACK || (D.type == PTR_MAPV && D.map == src.map))) {
                    Scalar a = sc_add(sc_const((uint64_t)D.off), D.var), b = sc_add(sc_const((uint64_t)src.off), src.var);
                    D = reg_scalar(sc_sub(a, b));
                } else {
                    return fail(pc, GX_PTR_LEAK, "illegal arithmetic on a pointer") ? 0 : -1;
                }
                P.pc++;
                return 0;
            }
            const Scalar before = D.var;
            D.var = is64 ? sc_alu64(op, r.off, D.var, src.var) : sc_alu32(op, r.off, D.var, src.var);
            D.type = SCALAR;
            if (is64) {
                /* narrow: the 64-bit result equals the zero-extended 32-bit operation (ADD / SUB /
                 * MUL / unsigned DIV, MOD / OR / AND / XOR, RSH by a count below 32) */
                const bool kind_ok = op == 0x00 || op == 0x10 || op == 0x20 || op == 0x40 || op == 0x50 || op == 0xA0 ||
                                     ((op == 0x30 || op == 0x90) && r.off == 0) || (op == 0x70 && src.var.umax < 32);
                const bool nar = kind_ok && before.umax < (1ull << 32) && src.var.umax < (1ull << 32) &&
                                 D.var.umax < (1ull << 32) && (op != 0x10 || before.umin >= src.var.umax);
                Fact &f = facts[pc];
                f.narrow = (f.narrow != 2 && nar) ? 1 : 2;
            }
            P.pc++;
            return 0;
        }

        if (cls == CL_LD) { /* ldimm64 */
            uint64_t lo = (uint32_t)r.imm, hi = (uint32_t)ins[pc + 1].imm;
            Reg v;
            if (r.src == 0) v = reg_scalar(sc_const(lo | (hi << 32)));
            else if (r.src == 1) {
                v.type = CONST_MAP;
                v.map = (int16_t)r.imm;
            } else {
                v.type = PTR_MAPV;
                v.map = (int16_t)r.imm;
                v.off = (int64_t)hi;
                v.var = sc_const(0);
            }
            D = v;
            P.pc += 2;
            return 0;
        }

        if (cls == CL_LDX) {
            uint32_t size = size_of(r.code);
            bool sx = (r.code & 0xE0) == 0x80;
            MemKind k;
            int32_t sa;
            int map;
            if (!check_access(pc, S, r.off, size, false, k, sa, map)) return -1;
            if (!record_mem(pc, k, map, sa)) return -1;
            P.cm++;
            if (k == MK_STACK) {
                bool ok;
                Reg v = stack_read(st, sa - GX_STACK_SIZE, size, sx, pc, ok);
                if (!ok) return -1;
                D = v;
            } else {
                Scalar v;
                if (sx) {
                    v = sc_unknown();
                    v.smin = -(int64_t)(1ull << (8 * size - 1));
                    v.smax = (int64_t)(1ull << (8 * size - 1)) - 1;
                    sc_sync(v);
                } else {
                    v = size == 8 ? sc_unknown() : sc_urange(0, (1ull << (8 * size)) - 1);
                }
                D = reg_scalar(v);
                if (map >= 0) {
                    out.use[map].used = true;
                    out.use[map].reads = true;
                }
            }
            P.pc++;
            return 0;
        }

        if (cls == CL_ST || (cls == CL_STX && (r.code & 0xE0) == 0x60)) {
            uint32_t size = size_of(r.code);
            Reg val = cls == CL_ST ? reg_scalar(sc_const((uint64_t)(int64_t)r.imm)) : S;
            if (val.type == NOT_INIT) return fail(pc, GX_UNINIT_READ, "stored register not initialised") ? 0 : -1;
            MemKind k;
            int32_t sa;
            int map;
            if (!check_access(pc, D, r.off, size, true, k, sa, map)) return -1;
            if (!record_mem(pc, k, map, sa)) return -1;
            P.cm++;
            if (is_ptr(val)) {
                if (k != MK_STACK || size != 8) return fail(pc, GX_PTR_LEAK, "pointer stored outside an 8-byte stack slot") ? 0 : -1;
            }
            if (k == MK_STACK) {
                Reg v = val;
                if (size < 8 && v.type == SCALAR) v.var = sc_unknown();
                stack_write(st, sa - GX_STACK_SIZE, size, size == 8 ? &v : &val); /* narrow: bound only */
            } else if (map >= 0) {
                out.use[map].used = out.use[map].writes = out.use[map].non_add_write = out.use[map].store = true;
            }
            P.pc++;
            return 0;
        }

        if (cls == CL_STX) { /* atomics */
            uint32_t size = size_of(r.code);
            if (S.type != SCALAR) return fail(pc, S.type == NOT_INIT ? GX_UNINIT_READ : GX_PTR_LEAK, "atomic operand is not a scalar") ? 0 : -1;
            MemKind k;
            int32_t sa;
            int map;
            if (!check_access(pc, D, r.off, size, true, k, sa, map)) return -1;
            if (!record_mem(pc, k, map, sa)) return -1;
            P.cm++;
            if (k == MK_STACK) {
                if (!check_stack_read_bytes(pc, st, sa - GX_STACK_SIZE, size, "atomic")) return -1;
                Slot &s = st.s[sa / 8];
                if (s.spill) {
                    s.spill = false; /* value now unknown */
                }
                s.nok = 0;
            } else if (map >= 0) {
                GxMapUse &u = out.use[map];
                u.used = u.writes = true;
                bool add = (r.imm & ~1) == 0x00;
                if (!add) u.non_add_write = u.store = true;
                if (size != 8) u.non_dw_atomic = true;
                if (r.imm & 1) {
                    u.reads = true;
                    if (add) u.fetch_add = true;
                }
            }
            if (r.imm == 0xF1) {
                Reg &R0 = st.r[0];
                if (R0.type != SCALAR) return fail(pc, R0.type == NOT_INIT ? GX_UNINIT_READ : GX_PTR_LEAK, "CMPXCHG needs a scalar r0") ? 0 : -1;
                R0 = reg_scalar(size == 8 ? sc_unknown() : sc_urange(0, 0xFFFFFFFFull));
            } else if (r.imm & 1) {
                S = reg_scalar(size == 8 ? sc_unknown() : sc_urange(0, 0xFFFFFFFFull));
            }
            P.pc++;
            return 0;
        }

        /* jumps */
        if (op == 0x00) {
            P.pc = pc + 1 + r.off;
            return 0;
        }
        if (op == 0x90) {
            Reg &R0 = st.r[0];
            if (R0.type == NOT_INIT) return fail(pc, GX_UNINIT_READ, "r0 not initialised at exit") ? 0 : -1;
            if (R0.type != SCALAR) return fail(pc, GX_PTR_LEAK, "returning a pointer in r0") ? 0 : -1;
            return 1;
        }
        if (op == 0x80) return call(P) ? 0 : -1;

        /* conditional: every outcome seen on some path is recorded (facts[pc].br) so the pre-decoder
         * can drop a branch the verifier proved one-sided on all paths (e.g. the NULL test after a
         * lookup whose key is provably in range) */
        int rc = cond_branch(P, pc, r, D, S, x, cls, pending);
        if (rc == 0) {
            const uint32_t tgt = pc + 1 + r.off;
            if (P.pc == tgt) facts[pc].br |= 1;
            if (P.pc == pc + 1) facts[pc].br |= 2;
        }
        return rc;
    }

    int cond_branch(Path &P, uint32_t pc, const Raw &r, Reg &D, Reg &S, bool x, uint32_t cls, std::vector<Path> &pending) {
        const uint32_t op = r.code & 0xF0;
        bool is64 = cls == CL_JMP;
        if (D.type == NOT_INIT || (x && S.type == NOT_INIT)) return fail(pc, GX_UNINIT_READ, "comparison of an uninitialised register") ? 0 : -1;
        uint32_t tgt = pc + 1 + r.off;
        Reg srcv = x ? S : reg_scalar(sc_const(is64 ? (uint64_t)(int64_t)r.imm : (uint64_t)(uint32_t)r.imm));
        if (is_ptr(D) || is_ptr(srcv)) {
            /* only JEQ/JNE ptr, 0 */
            if (!is64 || x || r.imm != 0 || (op != 0x10 && op != 0x50))
                return fail(pc, GX_PTR_LEAK, "pointer comparison") ? 0 : -1;
            if (D.type == PTR_MAPV_OR_NULL) {
                Path other = P;
                uint32_t id = D.id;
                /* null branch: every copy with this id becomes scalar 0; other: PTR_MAPV */
                auto mark = [id](State &s, bool null) {
                    auto fix = [&](Reg &rg) {
                        if (rg.type == PTR_MAPV_OR_NULL && rg.id == id) {
                            if (null) rg = reg_scalar(sc_const(0));
                            else {
                                rg.type = PTR_MAPV;
                                rg.id = 0;
                            }
                        }
                    };
                    for (auto &rg : s.r) fix(rg);
                    for (auto &sl : s.s)
                        if (sl.spill) fix(sl.reg);
                };
                bool taken_is_null = op == 0x10;
                mark(P.st, !taken_is_null);  /* fall-through */
                P.pc = pc + 1;
                mark(other.st, taken_is_null);
                other.pc = tgt;
                push_branch(other, pending);
                facts[pc].br |= other.pc == tgt ? 1 : 2;
                return 0;
            }
            /* non-null pointer vs 0: JEQ never taken, JNE always */
            P.pc = op == 0x50 ? tgt : pc + 1;
            return 0;
        }
        /* scalar comparison with refinement */
        Scalar d = D.var, s = srcv.var;
        if (!is64) {
            if (d.umax > 0xFFFFFFFFull || s.umax > 0xFFFFFFFFull) {
                /* compare low halves; only decide statically when both are constants */
                if (sc_is_const(d) && sc_is_const(s)) {
                    bool t = eval_cond(op, (uint32_t)d.t.v, (uint32_t)s.t.v, false);
                    P.pc = t ? tgt : pc + 1;
                    return 0;
                }
                Path other = P;
                other.pc = tgt;
                P.pc = pc + 1;
                push_branch(other, pending);
                facts[pc].br |= other.pc == tgt ? 1 : 2;
                return 0;
            }
        }
        int known = static_cond(op, d, s, is64);
        if (known == 1) {
            P.pc = tgt;
            return 0;
        }
        if (known == 0) {
            P.pc = pc + 1;
            return 0;
        }
        Path other = P;
        bool okT = refine(op, other.st.r[r.dst].var, x ? &other.st.r[r.src].var : nullptr, s, true, is64);
        bool okF = refine(op, P.st.r[r.dst].var, x ? &P.st.r[r.src].var : nullptr, s, false, is64);
        other.pc = tgt;
        P.pc = pc + 1;
        if (okT && okF) {
            push_branch(other, pending);
                facts[pc].br |= other.pc == tgt ? 1 : 2;
            return 0;
        }
        if (okT) {
            P = other;
            return 0;
        }
        return 0; /* only fall-through feasible (or neither: keep fall-through, sound) */
    }

    static bool eval_cond(uint32_t op, uint64_t d, uint64_t s, bool is64) {
        int64_t sd = is64 ? (int64_t)d : (int64_t)(int32_t)(uint32_t)d;
        int64_t ss = is64 ? (int64_t)s : (int64_t)(int32_t)(uint32_t)s;
        switch (op) {
        case 0x10: return d == s;
        case 0x50: return d != s;
        case 0x20: return d > s;
        case 0x30: return d >= s;
        case 0xA0: return d < s;
        case 0xB0: return d <= s;
        case 0x60: return sd > ss;
        case 0x70: return sd >= ss;
        case 0xC0: return sd < ss;
        case 0xD0: return sd <= ss;
        case 0x40: return (d & s) != 0;
        }
        return false;
    }

    /* 1 always taken, 0 never, -1 unknown (values already in 64-bit form; JMP32 only reaches
     * here with both operands < 2^32, where the 32- and 64-bit unsigned orders agree) */
    static int static_cond(uint32_t op, const Scalar &d, const Scalar &s, bool is64) {
        if (sc_is_const(d) && sc_is_const(s)) return eval_cond(op, d.t.v, s.t.v, is64);
        if (!is64) {
            /* signed 32-bit compares of values < 2^32 need the bit-31 view; stay unknown */
            if (op == 0x60 || op == 0x70 || op == 0xC0 || op == 0xD0) return -1;
        }
        switch (op) {
        case 0x10: if (d.umax < s.umin || d.umin > s.umax) return 0; break;
        case 0x50: if (d.umax < s.umin || d.umin > s.umax) return 1; break;
        case 0x20: if (d.umin > s.umax) return 1; if (d.umax <= s.umin) return 0; break;
        case 0x30: if (d.umin >= s.umax) return 1; if (d.umax < s.umin) return 0; break;
        case 0xA0: if (d.umax < s.umin) return 1; if (d.umin >= s.umax) return 0; break;
        case 0xB0: if (d.umax <= s.umin) return 1; if (d.umin > s.umax) return 0; break;
        case 0x60: if (d.smin > s.smax) return 1; if (d.smax <= s.smin) return 0; break;
        case 0x70: if (d.smin >= s.smax) return 1; if (d.smax < s.smin) return 0; break;
        case 0xC0: if (d.smax < s.smin) return 1; if (d.smin >= s.smax) return 0; break;
        case 0xD0: if (d.smax <= s.smin) return 1; if (d.smin > s.smax) return 0; break;
        case 0x40:
            if (sc_is_const(s) && ((d.t.v & s.t.v) != 0)) return 1;
            if (((d.t.v | d.t.m) & (s.t.v | s.t.m)) == 0) return 0;
            break;
        }
        return -1;
    }

    /* refine dst (and src if a register) for the branch outcome `taken` */
    static bool refine(uint32_t op, Scalar &d, Scalar *sreg, const Scalar &s, bool taken, bool is64) {
        if (!is64 && (op == 0x60 || op == 0x70 || op == 0xC0 || op == 0xD0)) return true;
        /* normalise to a predicate that holds on this branch */
        uint32_t p = op;
        if (!taken) {
            switch (op) {
            case 0x10: p = 0x50; break;
            case 0x50: p = 0x10; break;
            case 0x20: p = 0xB0; break;  /* !(d > s)  -> d <= s */
            case 0x30: p = 0xA0; break;
            case 0xA0: p = 0x30; break;
            case 0xB0: p = 0x20; break;
            case 0x60: p = 0xD0; break;
            case 0x70: p = 0xC0; break;
            case 0xC0: p = 0x70; break;
            case 0xD0: p = 0x60; break;
            case 0x40: p = 0x140; break; /* (d & s) == 0 */
            }
        }
        Scalar sv = sreg ? *sreg : s;
        switch (p) {
        case 0x10: {
            Scalar m = d;
            m.t = tn_intersect(d.t, sv.t);
            m.umin = std::max(d.umin, sv.umin);
            m.umax = std::min(d.umax, sv.umax);
            m.smin = std::max(d.smin, sv.smin);
            m.smax = std::min(d.smax, sv.smax);
            if (!sc_sync(m)) return false;
            d = m;
            if (sreg) *sreg = m;
            return true;
        }
        case 0x50:
            if (sc_is_const(sv)) {
                if (sc_is_const(d) && d.t.v == sv.t.v) return false;
                if (d.umin == sv.t.v) d.umin++;
                else if (d.umax == sv.t.v) d.umax--;
                return sc_sync(d);
            }
            return true;
        case 0x20: /* d > s */
            if (sv.umin == ~0ull) return false;
            d.umin = std::max(d.umin, sv.umin + 1);
            if (sreg && d.umax > 0) sreg->umax = std::min(sreg->umax, d.umax - 1);
            break;
        case 0x30:
            d.umin = std::max(d.umin, sv.umin);
            if (sreg) sreg->umax = std::min(sreg->umax, d.umax);
            break;
        case 0xA0: /* d < s */
            if (sv.umax == 0) return false;
            d.umax = std::min(d.umax, sv.umax - 1);
            if (sreg && d.umin < ~0ull) sreg->umin = std::max(sreg->umin, d.umin + 1);
            break;
        case 0xB0:
            d.umax = std::min(d.umax, sv.umax);
            if (sreg) sreg->umin = std::max(sreg->umin, d.umin);
            break;
        case 0x60:
            if (sv.smin == INT64_MAX) return false;
            d.smin = std::max(d.smin, sv.smin + 1);
            if (sreg && d.smax > INT64_MIN) sreg->smax = std::min(sreg->smax, d.smax - 1);
            break;
        case 0x70:
            d.smin = std::max(d.smin, sv.smin);
            if (sreg) sreg->smax = std::min(sreg->smax, d.smax);
            break;
        case 0xC0:
            if (sv.smax == INT64_MIN) return false;
            d.smax = std::min(d.smax, sv.smax - 1);
            if (sreg && d.smin < INT64_MAX) sreg->smin = std::max(sreg->smin, d.smin + 1);
            break;
        case 0xD0:
            d.smax = std::min(d.smax, sv.smax);
            if (sreg) sreg->smin = std::max(sreg->smin, d.smin);
            break;
        case 0x140:
            if (sc_is_const(sv)) {
                d.t.v &= ~sv.t.v;
                d.t.m &= ~sv.t.v;
            }
            break;
        default: break;
        }
        if (!sc_sync(d)) return false;
        if (sreg && !sc_sync(*sreg)) return false;
        return true;
    }

    void push_branch(Path &other, std::vector<Path> &pending) {
        if (other.parent) other.parent->branches++;
        pending.push_back(other);
    }

    /* helper calls (bpf.h:1753-1776, 4407-4422) */
    bool call(Path &P) {
        uint32_t pc = P.pc;
        State &st = P.st;
        int32_t id = ins[pc].imm;
        char msg[128];
        if (id == 93 || id == 94) return fail(pc, GX_FORBIDDEN_SYNC, "bpf_spin_lock/unlock: GPU-wide synchronisation is forbidden on device hooks");
        if (id != 1 && id != 2 && id != 130 && id != GX_FN_MEM_PREFETCH && id != GX_FN_PREFETCH_L2) {
            snprintf(msg, sizeof msg, "helper %d is not available to device programs", id);
            return fail(pc, GX_BAD_HELPER, msg);
        }
        Reg &R1 = st.r[1];
        if (R1.type != CONST_MAP) return fail(pc, R1.type == NOT_INIT ? GX_UNINIT_READ : GX_BAD_HELPER, "r1 must be a map handle");
        const GxMapInfo &mi = maps[R1.map];
        int m = R1.map;
        MemKind kk = MK_NONE, vk = MK_NONE;
        int32_t ka = 0, va = 0;
        int64_t rbs = -1, rbf = -1;
        GxMapUse &u = out.use[m];
        u.used = true;
        if (id == 1 || id == 2) {
            if (mi.type == RINGBUF || mi.type == PFQ || mi.type == REGION)
                return fail(pc, GX_BAD_HELPER, "map lookup/update on a ring buffer / prefetch queue / region");
            if (!check_arg_mem(pc, st, st.r[2], mi.key_size, mi.key_size, "key", kk, ka)) return false;
            if (kk == MK_MAPV) out.use[st.r[2].map].reads = out.use[st.r[2].map].used = true;
            if (id == 2) {
                if (!check_arg_mem(pc, st, st.r[3], mi.value_size, 8, "value", vk, va)) return false;
                if (vk == MK_MAPV) out.use[st.r[3].map].reads = out.use[st.r[3].map].used = true;
                Reg &R4 = st.r[4];
                if (R4.type != SCALAR) return fail(pc, R4.type == NOT_INIT ? GX_UNINIT_READ : GX_BAD_HELPER, "flags must be a scalar");
                u.writes = u.non_add_write = u.update_call = true;
                if (!sc_is_const(R4.var) || R4.var.t.v != 1) u.upd_overwrite = true; /* not BPF_NOEXIST */
                P.ch += 2;
            } else {
                P.ch += 1;
            }
        } else if (id == GX_FN_PREFETCH_L2) {
            /* gdev_prefetch_l2(region, addr, len) (F-7): addr and len are plain
             * scalars checked against the region at run time (-EFAULT / -EINVAL); nothing is written */
            if (mi.type != REGION) return fail(pc, GX_BAD_HELPER, "gdev_prefetch_l2 needs a device-region map");
            for (int a = 2; a <= 3; a++)
                if (st.r[a].type != SCALAR)
                    return fail(pc, st.r[a].type == NOT_INIT ? GX_UNINIT_READ : GX_BAD_HELPER,
                                a == 2 ? "prefetch address must be a scalar" : "prefetch length must be a scalar");
            P.ch += 1;
        } else if (id == GX_FN_MEM_PREFETCH) {
            /* gdev_mem_prefetch(queue, addr, len) (F-1): addr and len are
             * plain scalars (no memory is touched), range errors are run-time -EINVAL */
            if (mi.type != PFQ) return fail(pc, GX_BAD_HELPER, "gdev_mem_prefetch needs a prefetch-queue map");
            for (int a = 2; a <= 3; a++)
                if (st.r[a].type != SCALAR)
                    return fail(pc, st.r[a].type == NOT_INIT ? GX_UNINIT_READ : GX_BAD_HELPER,
                                a == 2 ? "prefetch address must be a scalar" : "prefetch length must be a scalar");
            u.writes = true;
            P.ch += 1;
        } else {
            if (mi.type != RINGBUF) return fail(pc, GX_BAD_HELPER, "bpf_ringbuf_output needs a ring buffer map");
            Reg &R3 = st.r[3], &R4 = st.r[4];
            if (R3.type != SCALAR || !sc_is_const(R3.var) || R3.var.t.v < 1 || R3.var.t.v > 256)
                return fail(pc, GX_BAD_HELPER, "ringbuf size must be a constant in [1,256]");
            if (R4.type != SCALAR || !sc_is_const(R4.var))
                return fail(pc, GX_BAD_HELPER, "ringbuf flags must be a constant");
            rbs = (int64_t)R3.var.t.v;
            rbf = (int64_t)R4.var.t.v;
            if (!check_arg_mem(pc, st, st.r[2], (uint32_t)rbs, 8, "ringbuf data", vk, va)) return false;
            if (vk == MK_MAPV) out.use[st.r[2].map].reads = out.use[st.r[2].map].used = true;
            u.writes = true;
            P.ch += 1;
        }
        if (!record_call(pc, m, kk, ka, vk, va, rbs, rbf)) return false;
        for (int i = 1; i <= 5; i++) st.r[i] = Reg{};
        Reg r0;
        if (id == 1) {
            r0.type = PTR_MAPV_OR_NULL;
            r0.map = (int16_t)m;
            r0.id = next_id++;
            r0.off = 0;
            r0.var = sc_const(0);
            /* an ARRAY lookup whose key is provably below max_entries cannot return NULL */
            uint64_t kmax = 0;
            const bool inr = (mi.type == ARRAY || mi.type == PT) && kk == MK_STACK && key_bound(st, ka, kmax) &&
                             kmax < mi.max_entries;
            if (inr && mi.type == ARRAY) {
                r0.type = PTR_MAPV;
                r0.id = 0;
            }
            facts[pc].inrange = (facts[pc].inrange != 2 && inr) ? 1 : 2;
        } else {
            Scalar s = sc_unknown();
            s.smin = -4095;
            s.smax = 0;
            sc_sync(s);
            r0 = reg_scalar(s);
        }
        st.r[0] = r0;
        P.pc++;
        return true;
    }

    /* ---------------------------------------------------------------- path bookkeeping */
    void path_end(Path &P, uint64_t ti, uint64_t th, uint64_t tm) {
        worst_i = std::max(worst_i, ti);
        worst_h = std::max(worst_h, th);
        worst_m = std::max(worst_m, tm);
        for (Checkpoint *c = P.parent; c; c = c->parent) {
            c->ri = std::max(c->ri, ti - c->ci);
            c->rh = std::max(c->rh, th - c->ch);
            c->rm = std::max(c->rm, tm - c->cm);
        }
        for (Checkpoint *c = P.parent; c;) {
            if (--c->branches > 0) break;
            c = c->parent;
        }
    }

    bool explore() {
        facts.assign(n, Fact{});
        visited.assign(n, {});
        std::vector<Path> pending;
        Path init;
        for (auto &rg : init.st.r) rg = Reg{};
        init.st.r[1].type = PTR_CTX;
        init.st.r[1].var = sc_const(0);
        init.st.r[10].type = PTR_STACK;
        init.st.r[10].var = sc_const(0);
        pending.push_back(init);
        uint32_t limit = opts.complexity_limit;
        uint64_t bi = opts.max_insns, bh = opts.max_helpers, bm = opts.max_memops;
        while (!pending.empty()) {
            Path P = std::move(pending.back());
            pending.pop_back();
            for (;;) {
                uint32_t pc = P.pc;
                if (++processed > limit) return fail(pc, GX_COMPLEXITY, "verifier complexity limit exceeded");
                if (prune_pt[pc]) {
                    bool pruned = false;
                    for (Checkpoint *c : visited[pc]) {
                        if (c->branches == 0) {
                            if (state_in(c->st, P.st)) {
                                path_end(P, P.ci + c->ri, P.ch + c->rh, P.cm + c->rm);
                                pruned = true;
                                break;
                            }
                        } else if (state_eq(c->st, P.st)) {
                            for (Checkpoint *a = P.parent; a; a = a->parent)
                                if (a == c) return fail(pc, GX_UNBOUNDED_LOOP, "infinite loop: the same state repeats");
                        }
                    }
                    if (pruned) break;
                    pool.emplace_back(new Checkpoint());
                    Checkpoint *cp = pool.back().get();
                    cp->st = P.st;
                    cp->parent = P.parent;
                    cp->branches = 1;
                    cp->ci = P.ci;
                    cp->ch = P.ch;
                    cp->cm = P.cm;
                    visited[pc].push_back(cp);
                    P.parent = cp;
                }
                P.ci++;
                if (P.ci > bi || P.ch > bh || P.cm > bm) {
                    char msg[128];
                    snprintf(msg, sizeof msg, "budget exceeded on a path (insns %llu/%llu, helpers %llu/%llu, memops %llu/%llu)",
                             (unsigned long long)P.ci, (unsigned long long)bi, (unsigned long long)P.ch,
                             (unsigned long long)bh, (unsigned long long)P.cm, (unsigned long long)bm);
                    return fail(pc, GX_BUDGET, msg);
                }
                int rc = step(P, pending);
                if (rc < 0) return false;
                if (rc == 1) {
                    path_end(P, P.ci, P.ch, P.cm);
                    break;
                }
            }
        }
        return true;
    }

    /* ---------------------------------------------------------------- stage 4: SIMT pass */
    enum U : uint8_t { U_UNINIT = 0, U_UNI = 1, U_VAR = 2 };
    struct UState {
        uint8_t r[11];
        uint8_t s[GX_STACK_SIZE / 8];
    };
    static uint8_t ctx_tag(int off, int size) {
        /* §8b: addr [0,8) and lane_id [27,28) are LANE_VARYING; all other fields UNIFORM */
        for (int b = off; b < off + size; b++)
            if (b < 8 || b == 27) return U_VAR;
        return U_UNI;
    }

    /* ---------------------------------------------------------------- stage 4b: divergence analysis
     * Sound warp-uniformity of each conditional branch, for the JIT's ballot-free branches
     * (GXF_UNIFORM).  Data flow as in simt(), except that EVERY ctx field is LANE_VARYING (§8b's
     * UNIFORM tags are a performance contract, not a guarantee), plus control dependence: at the
     * immediate post-dominator of a branch whose condition is LANE_VARYING, everything written
     * between the branch and that join is LANE_VARYING -- lanes arrive there from different paths
     * or after different iteration counts.  A branch whose operands stay UNIFORM is taken the same
     * way by every lane that reaches it together (a counted loop's exit, C4's 12 binary-search
     * steps), so it needs no ballot. */
    void divergence() {
        const uint32_t N = n, X = n; /* X: virtual exit */
        std::vector<std::vector<uint32_t>> succ(N);
        std::vector<uint8_t> is_insn(N, 0), is_jcc(N, 0);
        for (uint32_t pc = 0; pc < N; pc++) {
            if (pc > 0 && is_insn[pc - 1] && (ins[pc - 1].code & 7) == CL_LD) continue; /* 2nd ldimm64 slot */
            is_insn[pc] = 1;
            const Raw &r = ins[pc];
            const uint32_t cls = r.code & 7, op = r.code & 0xF0;
            if (cls == CL_LD) succ[pc].push_back(pc + 2);
            else if (cls == CL_JMP || cls == CL_JMP32) {
                if (op == 0x90) { /* exit */
                } else if (op == 0x80) succ[pc].push_back(pc + 1);
                else if (op == 0x00) succ[pc].push_back(pc + 1 + r.off);
                else {
                    is_jcc[pc] = 1;
                    succ[pc].push_back(pc + 1 + r.off);
                    succ[pc].push_back(pc + 1);
                }
            } else succ[pc].push_back(pc + 1);
            for (uint32_t &s : succ[pc])
                if (s >= N) s = X;
        }
        /* post-dominators (bit sets over N + 1 nodes) */
        const uint32_t W = (N + 1 + 63) / 64;
        std::vector<uint64_t> pd((uint64_t)(N + 1) * W, ~0ull);
        auto row = [&](uint32_t v) { return pd.data() + (uint64_t)v * W; };
        std::fill(row(X), row(X) + W, 0ull);
        row(X)[X / 64] |= 1ull << (X % 64);
        for (bool ch = true; ch;) {
            ch = false;
            for (int64_t p = (int64_t)N - 1; p >= 0; p--) {
                if (!is_insn[p]) continue;
                std::vector<uint64_t> t(W, ~0ull);
                if (succ[p].empty()) { /* exit */
                    std::fill(t.begin(), t.end(), 0ull);
                    t[X / 64] |= 1ull << (X % 64);
                } else {
                    for (uint32_t s : succ[p])
                        for (uint32_t w = 0; w < W; w++) t[w] &= row(s)[w];
                }
                t[p / 64] |= 1ull << (p % 64);
                for (uint32_t w = 0; w < W; w++)
                    if (row((uint32_t)p)[w] != t[w]) {
                        std::copy(t.begin(), t.end(), row((uint32_t)p));
                        ch = true;
                        break;
                    }
            }
        }
        auto popc = [&](uint32_t v) {
            uint32_t c = 0;
            for (uint32_t w = 0; w < W; w++) c += (uint32_t)__builtin_popcountll(row(v)[w]);
            return c;
        };
        auto ipdom = [&](uint32_t b) -> uint32_t { /* the strict post-dominator with the most post-dominators */
            const uint32_t want = popc(b) - 1;
            for (uint32_t v = 0; v <= N; v++)
                if (v != b && ((row(b)[v / 64] >> (v % 64)) & 1) && (v == X || is_insn[v]) && popc(v) == want) return v;
            return X;
        };
        /* written variables of one instruction: registers 0..10, stack slots 11.. */
        auto defs = [&](uint32_t pc, std::vector<uint32_t> &out) {
            const Raw &r = ins[pc];
            const Fact &f = facts[pc];
            const uint32_t cls = r.code & 7, op = r.code & 0xF0;
            if (cls == CL_ALU || cls == CL_ALU64 || cls == CL_LD || cls == CL_LDX) out.push_back(r.dst);
            else if (cls == CL_ST || cls == CL_STX) {
                if (f.kind == MK_STACK) out.push_back(11 + f.stack_addr / 8);
                if (cls == CL_STX && (r.code & 0xE0) == 0xC0 && (r.imm & 1)) out.push_back(r.imm == 0xF1 ? 0 : r.src);
            } else if ((cls == CL_JMP || cls == CL_JMP32) && op == 0x80) out.push_back(0);
        };
        std::vector<UState> in(N);
        std::vector<uint8_t> has(N, 0), var_br(N, 0);
        std::vector<UState> inject(N);
        std::vector<uint8_t> has_inj(N, 0);
        auto join = [](UState &a, const UState &b) {
            bool c = false;
            for (int i = 0; i < 11; i++)
                if (b.r[i] > a.r[i]) a.r[i] = b.r[i], c = true;
            for (int i = 0; i < GX_STACK_SIZE / 8; i++)
                if (b.s[i] > a.s[i]) a.s[i] = b.s[i], c = true;
            return c;
        };
        for (int round = 0; round < 64; round++) {
            std::fill(has.begin(), has.end(), 0);
            UState e{};
            e.r[1] = U_VAR; /* the ctx pointer differs per lane; its loads are LANE_VARYING below anyway */
            e.r[10] = U_UNI;
            in[0] = e;
            has[0] = 1;
            if (has_inj[0]) join(in[0], inject[0]);
            std::vector<uint32_t> work{0};
            while (!work.empty()) {
                const uint32_t pc = work.back();
                work.pop_back();
                UState u = in[pc];
                const Raw &r = ins[pc];
                const Fact &f = facts[pc];
                const uint32_t cls = r.code & 7, op = r.code & 0xF0;
                const bool x = r.code & 0x08;
                if (cls == CL_ALU || cls == CL_ALU64) {
                    if (op == 0xB0 && r.off == 0) u.r[r.dst] = x ? u.r[r.src] : U_UNI;
                    else if (x) u.r[r.dst] = std::max(u.r[r.dst], u.r[r.src]);
                } else if (cls == CL_LD) {
                    u.r[r.dst] = U_UNI;
                } else if (cls == CL_LDX) {
                    if (f.kind == MK_STACK) u.r[r.dst] = std::max(u.s[f.stack_addr / 8], u.r[r.src]);
                    else u.r[r.dst] = U_VAR; /* ctx (every field) and map values */
                } else if (cls == CL_ST || cls == CL_STX) {
                    if ((r.code & 0xE0) == 0xC0) {
                        if (r.imm & 1) u.r[r.imm == 0xF1 ? 0 : r.src] = U_VAR;
                        if (f.kind == MK_STACK) u.s[f.stack_addr / 8] = U_VAR;
                    } else if (f.kind == MK_STACK) {
                        const uint8_t v = std::max(cls == CL_ST ? (uint8_t)U_UNI : u.r[r.src], u.r[r.dst]);
                        const uint32_t sz = size_of(r.code);
                        u.s[f.stack_addr / 8] = sz == 8 ? v : std::max(u.s[f.stack_addr / 8], v);
                    }
                } else if ((cls == CL_JMP || cls == CL_JMP32) && op == 0x80) {
                    uint8_t keyu = U_UNI;
                    if (f.key_kind == MK_STACK) {
                        const GxMapInfo &mi = maps[f.map];
                        for (uint32_t b = 0; b < mi.key_size; b += 8) keyu = std::max(keyu, u.s[(f.key_addr + b) / 8]);
                    } else if (f.key_kind == MK_MAPV) {
                        keyu = U_VAR;
                    }
                    const bool shared = f.map >= 0 && maps[f.map].type != PT;
                    for (int i = 1; i <= 5; i++) u.r[i] = U_UNINIT;
                    u.r[0] = (r.imm == 1 && shared && keyu == U_UNI) ? U_UNI : U_VAR;
                } else if (is_jcc[pc]) {
                    const uint8_t c = std::max(u.r[r.dst], x ? u.r[r.src] : (uint8_t)U_UNI);
                    if (c == U_VAR) var_br[pc] = 1;
                }
                for (uint32_t s : succ[pc]) {
                    if (s >= N) continue;
                    if (!has[s]) {
                        in[s] = u;
                        if (has_inj[s]) join(in[s], inject[s]);
                        has[s] = 1;
                        work.push_back(s);
                    } else if (join(in[s], u)) {
                        work.push_back(s);
                    }
                }
            }
            /* control dependence ("sync dependence"): lanes that split at a LANE_VARYING branch meet
             * again at every node reachable from both of its sides (up to the immediate post-
             * dominator, which both reach); everything written on the way is LANE_VARYING there */
            bool grew = false;
            for (uint32_t b = 0; b < N; b++) {
                if (!var_br[b] || succ[b].size() != 2 || succ[b][0] == succ[b][1]) continue;
                const uint32_t j = ipdom(b);
                std::vector<uint8_t> side[2] = {std::vector<uint8_t>(N, 0), std::vector<uint8_t>(N, 0)};
                for (int k = 0; k < 2; k++) {
                    std::vector<uint32_t> st2;
                    const uint32_t s0 = succ[b][k];
                    if (s0 < N && s0 != j) side[k][s0] = 1, st2.push_back(s0);
                    while (!st2.empty()) {
                        const uint32_t p = st2.back();
                        st2.pop_back();
                        for (uint32_t q : succ[p])
                            if (q < N && q != j && !side[k][q]) side[k][q] = 1, st2.push_back(q);
                    }
                }
                std::vector<uint32_t> dv;
                for (uint32_t p = 0; p < N; p++)
                    if (side[0][p] || side[1][p]) defs(p, dv);
                if (dv.empty()) continue;
                UState add{};
                for (uint32_t v : dv) {
                    if (v < 11) add.r[v] = U_VAR;
                    else add.s[v - 11] = U_VAR;
                }
                auto put = [&](uint32_t v) {
                    if (!has_inj[v]) {
                        inject[v] = add;
                        has_inj[v] = 1;
                        grew = true;
                    } else if (join(inject[v], add)) {
                        grew = true;
                    }
                };
                if (j < N) put(j);
                for (uint32_t p = 0; p < N; p++)
                    if (side[0][p] && side[1][p]) put(p);
            }
            if (!grew) break;
        }
        for (uint32_t pc = 0; pc < N; pc++)
            if (is_jcc[pc]) hint_uniform[pc] = (has[pc] && !var_br[pc]) ? 1 : 0;
        if (getenv("GX_VERIFY_DEBUG"))
            for (uint32_t pc = 0; pc < N; pc++)
                if (is_jcc[pc])
                    fprintf(stderr, "divergence: pc %u %s (dst %u: %d, src %u: %d)\n", pc, hint_uniform[pc] ? "UNIFORM" : "varying",
                            ins[pc].dst, has[pc] ? in[pc].r[ins[pc].dst] : -1, ins[pc].src, has[pc] ? in[pc].r[ins[pc].src] : -1);
    }

    bool simt(bool strict, uint32_t &all_uniform) {
        std::vector<UState> in(n);
        std::vector<uint8_t> has(n, 0);
        UState e{};
        e.r[1] = U_UNI;
        e.r[10] = U_UNI;
        in[0] = e;
        has[0] = 1;
        std::vector<uint32_t> work{0};
        std::vector<uint8_t> branch_var(n, 0), key_var(n, 0), atom_var(n, 0);
        auto join = [](UState &a, const UState &b) {
            bool ch = false;
            for (int i = 0; i < 11; i++)
                if (b.r[i] > a.r[i]) { a.r[i] = b.r[i]; ch = true; }
            for (int i = 0; i < GX_STACK_SIZE / 8; i++)
                if (b.s[i] > a.s[i]) { a.s[i] = b.s[i]; ch = true; }
            return ch;
        };
        while (!work.empty()) {
            uint32_t pc = work.back();
            work.pop_back();
            UState u = in[pc];
            const Raw &r = ins[pc];
            const Fact &f = facts[pc];
            uint32_t cls = r.code & 7, op = r.code & 0xF0;
            bool x = r.code & 0x08;
            std::vector<uint32_t> succ;
            if (cls == CL_ALU || cls == CL_ALU64) {
                if (op == 0xB0 && r.off == 0) u.r[r.dst] = x ? u.r[r.src] : U_UNI;
                else if (x) u.r[r.dst] = std::max(u.r[r.dst], u.r[r.src]);
                succ.push_back(pc + 1);
            } else if (cls == CL_LD) {
                u.r[r.dst] = U_UNI;
                succ.push_back(pc + 2);
            } else if (cls == CL_LDX) {
                uint32_t sz = size_of(r.code);
                if (f.kind == MK_CTX) u.r[r.dst] = ctx_tag(f.stack_addr, (int)sz);
                else if (f.kind == MK_STACK) u.r[r.dst] = std::max(u.s[f.stack_addr / 8], u.r[r.src]);
                else u.r[r.dst] = U_VAR; /* map values are LANE_VARYING by default (I-11) */
                succ.push_back(pc + 1);
            } else if (cls == CL_ST || cls == CL_STX) {
                if ((r.code & 0xE0) == 0xC0) {
                    if ((f.kind == MK_MAPV) && u.r[r.dst] == U_VAR) atom_var[pc] = 1;
                    if (r.imm & 1) {
                        if (r.imm == 0xF1) u.r[0] = U_VAR;
                        else u.r[r.src] = U_VAR;
                    }
                    if (f.kind == MK_STACK) u.s[f.stack_addr / 8] = U_VAR;
                } else if (f.kind == MK_STACK) {
                    uint8_t v = cls == CL_ST ? U_UNI : u.r[r.src];
                    uint32_t sz = size_of(r.code);
                    u.s[f.stack_addr / 8] = sz == 8 ? v : std::max(u.s[f.stack_addr / 8], v);
                }
                succ.push_back(pc + 1);
            } else if (op == 0x90) {
            } else if (op == 0x80) {
                int id = r.imm;
                uint8_t keyu = U_UNI;
                if (f.key_kind == MK_STACK) {
                    const GxMapInfo &mi = maps[f.map];
                    for (uint32_t b = 0; b < mi.key_size; b += 8) keyu = std::max(keyu, u.s[(f.key_addr + b) / 8]);
                } else if (f.key_kind == MK_MAPV) {
                    keyu = U_VAR;
                }
                bool shared = f.map >= 0 && maps[f.map].type != PT;
                if (id == 2 && shared && keyu == U_VAR) key_var[pc] = 1;
                for (int i = 1; i <= 5; i++) u.r[i] = U_UNINIT;
                u.r[0] = (id == 1 && shared && keyu == U_UNI) ? U_UNI : U_VAR;
                succ.push_back(pc + 1);
            } else if (op == 0x00) {
                succ.push_back(pc + 1 + r.off);
            } else {
                uint8_t c = std::max(u.r[r.dst], x ? u.r[r.src] : (uint8_t)U_UNI);
                if (c == U_VAR) branch_var[pc] = 1;
                succ.push_back(pc + 1 + r.off);
                succ.push_back(pc + 1);
            }
            for (uint32_t s : succ) {
                if (s >= n) continue;
                if (!has[s]) {
                    in[s] = u;
                    has[s] = 1;
                    work.push_back(s);
                } else if (join(in[s], u)) {
                    work.push_back(s);
                }
            }
        }
        /* loops: a branch inside a cycle (it can reach itself) */
        all_uniform = 1;
        for (uint32_t i = 0; i < n; i++) {
            if (branch_var[i]) all_uniform = 0;
        }
        for (uint32_t i = 0; i < n; i++)
            if (branch_var[i]) hint_uniform[i] = 0;
        if (!strict) return true;
        for (uint32_t i = 0; i < n; i++) {
            if (!has[i]) continue;
            if (branch_var[i]) {
                if (in_cycle(i)) fail(i, GX_UNIFORM_LOOP_BOUND, "loop bound / back-edge condition depends on a LANE_VARYING value");
                else fail(i, GX_UNIFORM_BRANCH, "branch condition depends on a LANE_VARYING value");
            }
            if (key_var[i]) fail(i, GX_UNIFORM_MAP_KEY, "map update key is LANE_VARYING on a shared map");
            if (atom_var[i]) fail(i, GX_NON_UNIFORM_ATOMIC, "atomic target address is LANE_VARYING on a shared map");
        }
        return viol.empty();
    }

    bool in_cycle(uint32_t start) {
        std::vector<uint8_t> seen(n, 0);
        std::vector<uint32_t> work;
        auto push_succ = [&](uint32_t i) {
            const Raw &r = ins[i];
            uint32_t cls = r.code & 7, op = r.code & 0xF0;
            auto add = [&](uint32_t s) {
                if (s < n && !seen[s]) { seen[s] = 1; work.push_back(s); }
            };
            if (cls == CL_JMP || cls == CL_JMP32) {
                if (op == 0x90) return;
                if (op == 0x80) { add(i + 1); return; }
                add(i + 1 + r.off);
                if (op != 0x00) add(i + 1);
            } else if (cls == CL_LD) add(i + 2);
            else add(i + 1);
        };
        push_succ(start);
        while (!work.empty()) {
            uint32_t i = work.back();
            work.pop_back();
            if (i == start) return true;
            push_succ(i);
        }
        return false;
    }

    /* ---------------------------------------------------------------- stage 5: pre-decode */
    void predecode() {
        out.image.assign(n, GxInsn{});
        static const uint8_t alu64[14] = {GX_ADD64, GX_SUB64, GX_MUL64, GX_DIV64, GX_OR64, GX_AND64, GX_LSH64,
                                          GX_RSH64, GX_NEG64, GX_MOD64, GX_XOR64, GX_MOV64, GX_ARSH64, 0};
        static const uint8_t alu32[14] = {GX_ADD32, GX_SUB32, GX_MUL32, GX_DIV32, GX_OR32, GX_AND32, GX_LSH32,
                                          GX_RSH32, GX_NEG32, GX_MOD32, GX_XOR32, GX_MOV32, GX_ARSH32, 0};
        auto jop = [](uint32_t op, bool is64) -> uint8_t {
            uint8_t b = 0;
            switch (op) {
            case 0x10: b = GX_JEQ; break;
            case 0x50: b = GX_JNE; break;
            case 0x20: b = GX_JGT; break;
            case 0x30: b = GX_JGE; break;
            case 0xA0: b = GX_JLT; break;
            case 0xB0: b = GX_JLE; break;
            case 0x60: b = GX_JSGT; break;
            case 0x70: b = GX_JSGE; break;
            case 0xC0: b = GX_JSLT; break;
            case 0xD0: b = GX_JSLE; break;
            case 0x40: b = GX_JSET; break;
            }
            return is64 ? b : (uint8_t)(b + (GX_JEQ32 - GX_JEQ));
        };
        auto lg = [](uint32_t sz) -> uint16_t { return sz == 1 ? 0 : sz == 2 ? 1 : sz == 4 ? 2 : 3; };
        for (uint32_t i = 0; i < n; i++) {
            if (is_second[i]) continue;
            const Raw &r = ins[i];
            const Fact &f = facts[i];
            GxInsn g{};
            g.dst = r.dst;
            g.src = r.src;
            uint32_t cls = r.code & 7, op = r.code & 0xF0;
            bool x = r.code & 0x08;
            if (x) g.flags |= GXF_X;
            if (cls == CL_ALU || cls == CL_ALU64) {
                bool is64 = cls == CL_ALU64;
                if (op == 0xD0) {
                    g.op = (is64 || x) ? GX_BE : GX_LE;
                    g.aux = (uint16_t)r.imm;
                } else {
                    g.op = (is64 ? alu64 : alu32)[op >> 4];
                    if ((op == 0x30 || op == 0x90) && r.off == 1) g.op = (uint8_t)(g.op + 1); /* SDIV/SMOD follow DIV/MOD */
                    if (op == 0xB0 && r.off) {
                        g.op = is64 ? GX_MOVSX64 : GX_MOVSX32;
                        g.aux = (uint16_t)r.off;
                    }
                    g.imm = is64 ? (uint64_t)(int64_t)r.imm : (uint64_t)(uint32_t)r.imm;
                    if (is64 && f.narrow == 1) g.flags |= GXF_NARROW;
                }
            } else if (cls == CL_LD) {
                g.op = GX_LDIMM;
                uint64_t lo = (uint32_t)r.imm, hi = (uint32_t)ins[i + 1].imm;
                if (r.src == 0) g.imm = lo | (hi << 32);
                else if (r.src == 1) g.imm = (uint64_t)r.imm; /* map handle = fd (never dereferenced) */
                else {
                    g.imm = hi;                  /* byte offset; relocated to an address at launch */
                    g.aux = (uint16_t)r.imm;     /* map fd */
                    g.flags |= GXF_VAL_MAPV;     /* marks "relocate imm += map data address" */
                }
            } else if (cls == CL_JMP || cls == CL_JMP32) {
                bool is64 = cls == CL_JMP;
                if (op == 0x00) {
                    g.op = GX_JA;
                    g.aux = (uint16_t)(i + 1 + r.off);
                } else if (op == 0x90) {
                    g.op = GX_EXIT;
                } else if (op == 0x80) {
                    int id = r.imm;
                    const GxMapInfo &mi = maps[f.map < 0 ? 0 : f.map];
                    g.aux = (uint16_t)f.map;
                    if (f.key_kind == MK_MAPV) g.flags |= GXF_KEY_MAPV;
                    if (f.val_kind == MK_MAPV) g.flags |= GXF_VAL_MAPV;
                    g.off = (int16_t)f.key_addr;
                    if (id == 1) {
                        g.op = mi.type == ARRAY ? GX_CALL_LOOKUP_ARRAY : mi.type == PT ? GX_CALL_LOOKUP_PT : GX_CALL_LOOKUP_HASH;
                        if (g.op != GX_CALL_LOOKUP_HASH && f.inrange == 1) g.flags |= GXF_SX; /* key always in range */
                    }
                    else if (id == 2) {
                        g.op = mi.type == ARRAY ? GX_CALL_UPDATE_ARRAY : mi.type == PT ? GX_CALL_UPDATE_PT : GX_CALL_UPDATE_HASH;
                        g.imm = (uint64_t)(uint32_t)f.val_addr;
                    } else if (id == GX_FN_MEM_PREFETCH) {
                        g.op = GX_CALL_MEM_PREFETCH;
                    } else if (id == GX_FN_PREFETCH_L2) {
                        g.op = GX_CALL_PREFETCH_L2;
                    } else {
                        g.op = GX_CALL_RINGBUF_OUTPUT;
                        g.off = (int16_t)f.val_addr;
                        g.imm = (uint64_t)f.rb_size | ((uint64_t)(uint32_t)f.rb_flags << 32);
                    }
                } else {
                    g.op = jop(op, is64);
                    g.aux = (uint16_t)(i + 1 + r.off);
                    g.imm = is64 ? (uint64_t)(int64_t)r.imm : (uint64_t)(uint32_t)r.imm;
                    if (hint_uniform.size() == n && hint_uniform[i]) g.flags |= GXF_UNIFORM;
                    /* one-sided on every explored path: an unconditional jump (no ballot, no split) */
                    if (f.br == 1) g.op = GX_JA, g.flags = 0, g.imm = 0;
                    else if (f.br == 2) g.op = GX_JA, g.aux = (uint16_t)(i + 1), g.flags = 0, g.imm = 0;
                }
            } else if (cls == CL_LDX) {
                uint32_t sz = size_of(r.code);
                g.aux = lg(sz);
                if ((r.code & 0xE0) == 0x80) g.flags |= GXF_SX;
                switch (f.kind) {
                case MK_CTX: g.op = GX_LDX_CTX; g.off = (int16_t)f.stack_addr; break;
                case MK_STACK: g.op = GX_LDX_STACK; g.off = (int16_t)f.stack_addr; break;
                case MK_MAPV: g.op = GX_LDX_MAP; g.off = r.off; g.imm = (uint64_t)f.map; break;
                case MK_PTV: g.op = GX_LDX_PT; g.off = r.off; g.imm = (uint64_t)f.map;
                    if (f.pt_vstart) g.flags |= GXF_PT_VSTART;
                    break;
                default: g.op = GX_OP_NOP;
                }
            } else if (cls == CL_ST || (cls == CL_STX && (r.code & 0xE0) == 0x60)) {
                uint32_t sz = size_of(r.code);
                g.aux = lg(sz);
                if (cls == CL_ST) {
                    g.flags &= ~GXF_X;
                    g.imm = (uint64_t)(int64_t)r.imm;
                } else {
                    g.flags |= GXF_X;
                }
                switch (f.kind) {
                case MK_STACK: g.op = GX_ST_STACK; g.off = (int16_t)f.stack_addr; break;
                case MK_MAPV: g.op = GX_ST_MAP; g.off = r.off; break;
                case MK_PTV: g.op = GX_ST_PT; g.off = r.off;
                    if (f.pt_vstart) g.flags |= GXF_PT_VSTART;
                    break;
                default: g.op = GX_OP_NOP;
                }
                if (f.kind == MK_PTV) g.aux = (uint16_t)(lg(sz) | (f.map << 4));
            } else if (cls == CL_STX) {
                uint32_t sz = size_of(r.code);
                g.aux = (uint16_t)(lg(sz) | ((f.map < 0 ? 0 : f.map) << 4));
                g.imm = (uint64_t)(uint32_t)r.imm;
                if (r.imm & 1) g.flags |= GXF_FETCH;
                switch (f.kind) {
                case MK_STACK: g.op = GX_ATOM_STACK; g.off = (int16_t)f.stack_addr; break;
                case MK_MAPV: g.op = GX_ATOM_MAP; g.off = r.off; break;
                case MK_PTV: g.op = GX_ATOM_PT; g.off = r.off;
                    if (f.pt_vstart) g.flags |= GXF_PT_VSTART;
                    break;
                default: g.op = GX_OP_NOP;
                }
            }
            if (!f.seen && (cls == CL_LDX || cls == CL_ST || cls == CL_STX || (cls == CL_JMP && op == 0x80)))
                g.op = GX_OP_NOP; /* never reached on any feasible path */
            out.image[i] = g;
        }
    }
    std::vector<uint8_t> hint_uniform;

    /* ---------------------------------------------------------------- stage 6: image optimisation
     * Liveness-based removal of instructions whose only effect is a register nobody reads (the
     * helper-argument set-up `lddw r1, map; mov r2, r10; add r2, -k` that the pre-decoded call
     * resolved statically), three superinstructions, and compaction (ldimm64 second slots go).
     * Pure re-encoding of the verified program: same per-event semantics (tests compare with the
     * oracle). */
    struct UD {
        uint16_t use = 0, def = 0;
        bool effect = false;
    };
    static UD ud_of(const GxInsn &g) {
        UD u;
        auto R = [](int r) { return (uint16_t)(1u << r); };
        const bool x = g.flags & GXF_X;
        switch (g.op) {
        case GX_MOV64: case GX_MOV32:
            u.use = x ? R(g.src) : 0;
            u.def = R(g.dst);
            break;
        case GX_MOVSX64: case GX_MOVSX32:
            u.use = R(g.src);
            u.def = R(g.dst);
            break;
        case GX_NEG64: case GX_NEG32: case GX_LE: case GX_BE:
            u.use = R(g.dst);
            u.def = R(g.dst);
            break;
        case GX_LDIMM: u.def = R(g.dst); break;
        case GX_JA: break;
        case GX_EXIT: u.use = R(0); u.effect = true; break;
        case GX_LDX_CTX: case GX_LDX_STACK: u.def = R(g.dst); break;
        case GX_LDX_MAP: case GX_LDX_PT: u.use = R(g.src); u.def = R(g.dst); break;
        case GX_ST_STACK: u.use = x ? R(g.src) : 0; u.effect = true; break;
        case GX_ST_MAP: case GX_ST_PT: u.use = R(g.dst) | (x ? R(g.src) : 0); u.effect = true; break;
        case GX_ATOM_STACK: case GX_ATOM_MAP: case GX_ATOM_PT: {
            const uint32_t op = (uint32_t)(g.imm & 0xFF);
            u.use = R(g.src) | (g.op != GX_ATOM_STACK ? R(g.dst) : 0) | (op == 0xF1 ? R(0) : 0);
            if (op == 0xF1) u.def = R(0);
            else if (op & 1) u.def = R(g.src);
            u.effect = true;
            break;
        }
        case GX_CALL_LOOKUP_ARRAY: case GX_CALL_LOOKUP_PT: case GX_CALL_LOOKUP_HASH:
            u.use = (g.flags & GXF_KEY_MAPV) ? R(2) : 0;
            u.def = 0x3F;
            u.effect = true;
            break;
        case GX_CALL_UPDATE_ARRAY: case GX_CALL_UPDATE_PT: case GX_CALL_UPDATE_HASH:
            u.use = R(4) | ((g.flags & GXF_KEY_MAPV) ? R(2) : 0) | ((g.flags & GXF_VAL_MAPV) ? R(3) : 0);
            u.def = 0x3F;
            u.effect = true;
            break;
        case GX_CALL_RINGBUF_OUTPUT:
            u.use = (g.flags & GXF_VAL_MAPV) ? R(2) : 0;
            u.def = 0x3F;
            u.effect = true;
            break;
        case GX_CALL_MEM_PREFETCH:
        case GX_CALL_PREFETCH_L2:
            u.use = R(2) | R(3);
            u.def = 0x3F;
            u.effect = true;
            break;
        case GX_OP_NOP: u.effect = true; break;
        default:
            if (g.op >= GX_JEQ && g.op <= GX_JSET32) {
                u.use = R(g.dst) | (x ? R(g.src) : 0);
            } else { /* binary ALU */
                u.use = R(g.dst) | (x ? R(g.src) : 0);
                u.def = R(g.dst);
            }
        }
        return u;
    }
    static bool is_jcc(uint8_t op) { return op >= GX_JEQ && op <= GX_JSET32; }

    void optimize(bool full) {
        std::vector<GxInsn> &im = out.image;
        const uint32_t N = (uint32_t)im.size();
        std::vector<uint8_t> removed(N, 0), target(N, 0);
        for (uint32_t i = 0; i < N; i++)
            if (is_second[i]) removed[i] = 1;
        auto succs = [&](uint32_t i, uint32_t *s) -> int {
            const GxInsn &g = im[i];
            if (g.op == GX_EXIT || g.op == GX_OP_NOP) return 0;
            uint32_t nx = i + (g.op == GX_LDIMM ? 2 : 1);
            if (g.op == GX_JA) { s[0] = g.aux; return 1; }
            if (is_jcc(g.op)) { s[0] = g.aux; s[1] = nx; return 2; }
            s[0] = nx;
            return 1;
        };
        for (uint32_t i = 0; i < N; i++)
            if (!removed[i] && (im[i].op == GX_JA || is_jcc(im[i].op))) target[im[i].aux] = 1;
        /* dead-definition elimination to a fixpoint (removed insns become pass-throughs) */
        for (int round = 0; round < (full ? 16 : 0); round++) {
            std::vector<uint16_t> live_in(N, 0), live_out(N, 0);
            bool ch = true;
            while (ch) {
                ch = false;
                for (int i = (int)N - 1; i >= 0; i--) {
                    if (is_second[i]) continue;
                    uint32_t sv[2];
                    int ns = succs(i, sv);
                    uint16_t lo = 0;
                    for (int k = 0; k < ns; k++)
                        if (sv[k] < N) lo |= live_in[sv[k]];
                    uint16_t li;
                    if (removed[i]) li = lo;
                    else {
                        UD u = ud_of(im[i]);
                        li = (uint16_t)(u.use | (lo & ~u.def));
                    }
                    if (lo != live_out[i] || li != live_in[i]) {
                        live_out[i] = lo;
                        live_in[i] = li;
                        ch = true;
                    }
                }
            }
            bool any = false;
            for (uint32_t i = 0; i < N; i++) {
                if (removed[i] || is_second[i]) continue;
                UD u = ud_of(im[i]);
                if (!u.effect && u.def && !(u.def & live_out[i]) && im[i].op != GX_JA && !is_jcc(im[i].op)) {
                    removed[i] = 1;
                    any = true;
                }
            }
            if (!any) {
                live = live_out;
                break;
            }
        }
        if (live.size() != N) live.assign(N, 0x7FF);
        /* superinstructions over adjacent surviving instructions */
        auto next_kept = [&](uint32_t i) {
            uint32_t j = i + 1;
            while (j < N && removed[j]) j++;
            return j;
        };
        for (uint32_t i = 0; i < N && full; i++) {
            if (removed[i]) continue;
            GxInsn &a = im[i];
            uint32_t j = next_kept(i);
            if (j >= N || target[j]) continue;
            /* all removed insns between i and j must not be jump targets either */
            bool clean = true;
            for (uint32_t k = i + 1; k < j; k++)
                if (target[k]) clean = false;
            if (!clean) continue;
            GxInsn &b = im[j];
            if (a.op == GX_MOV64 && !(a.flags & GXF_X) && a.dst == 0 && b.op == GX_EXIT) {
                b = a;
                b.op = GX_EXIT;
                b.flags = GXF_SX; /* exit with r0 = imm */
                std::swap(a, b);
                removed[j] = 1;
            } else if ((a.op == GX_CALL_LOOKUP_ARRAY || a.op == GX_CALL_LOOKUP_PT || a.op == GX_CALL_LOOKUP_HASH) &&
                       (b.op == GX_JEQ || b.op == GX_JNE) && b.dst == 0 && !(b.flags & GXF_X) && b.imm == 0) {
                a.flags |= b.op == GX_JEQ ? GXF_FETCH /* jump if NULL */ : GXF_W32 /* jump if not NULL */;
                a.flags |= b.flags & GXF_UNIFORM; /* a warp-uniform key: every lane finds the same entry */
                a.imm = b.aux;
                removed[j] = 1;
            } else if (a.op == GX_MOV64 && !(a.flags & GXF_X) &&
                       (b.op == GX_ATOM_MAP || b.op == GX_ATOM_PT || b.op == GX_ATOM_STACK) && b.src == a.dst &&
                       !(b.imm & 1) && (b.imm & 0xFF) != 0xE1 && !(live[j] & (1u << a.dst))) {
                /* non-FETCH only: on C3 the folded FETCH-ADD measured 25 % slower than the register
                 * form (8.1 vs 6.2 ms, same box, interleaved; profiles/r2_c3.md) */
                GxInsn f = b;
                f.flags |= GXF_PRIV; /* constant operand in imm[63:32] */
                f.imm = (b.imm & 0xFF) | ((uint64_t)(uint32_t)(int32_t)(int64_t)a.imm << 32);
                a = f;
                removed[j] = 1;
            }
        }
        /* compaction */
        std::vector<uint32_t> map(N + 1, 0);
        uint32_t np = 0;
        for (uint32_t i = 0; i < N; i++) {
            map[i] = np;
            if (!removed[i]) np++;
        }
        map[N] = np;
        std::vector<GxInsn> c;
        c.reserve(np);
        /* the narrow-register set of a compacted slot: the entry state of its surviving original
         * slot.  (Not that of a removed slot mapped onto it: one removed from the end of the
         * preceding block lies on the fall-through path only -- the fuzz caught a join taking a
         * predecessor's narrower state.  Removed slots define dead registers only, so the survivor's
         * state holds for every live register on every way in.) */
        std::vector<uint16_t> nin(np + 1, 0);
        for (uint32_t i = 0; i < N; i++)
            if (!removed[i]) nin[map[i]] = facts[i].nin_seen ? facts[i].nin : 0;
        out.narrow_in.assign(nin.begin(), nin.begin() + np);
        for (uint32_t i = 0; i < N; i++) {
            if (removed[i]) continue;
            GxInsn g = im[i];
            if (g.op == GX_JA || is_jcc(g.op)) g.aux = (uint16_t)map[g.aux];
            if ((g.op == GX_CALL_LOOKUP_ARRAY || g.op == GX_CALL_LOOKUP_PT || g.op == GX_CALL_LOOKUP_HASH) &&
                (g.flags & (GXF_FETCH | GXF_W32)))
                g.imm = map[g.imm];
            c.push_back(g);
        }
        im.swap(c);
    }
    std::vector<uint16_t> live;
};

}  // namespace

const char *gx_rule_name(uint32_t rule) { return rule < GX_NUM_RULES ? kRuleNames[rule] : "?"; }

int gx_verify_program(const uint8_t *slots, uint32_t n, const GxMapInfo *maps, const gx_verify_opts &o,
                      GxVerifyResult &out) {
    gx_verify_opts opts = o;
    if (!opts.max_insns) opts.max_insns = 4096;
    if (!opts.max_helpers) opts.max_helpers = 64;
    if (!opts.max_memops) opts.max_memops = 1024;
    if (!opts.complexity_limit) opts.complexity_limit = 1000000;
    out = GxVerifyResult{};
    Verifier v(slots, n, maps, opts, out);
    bool st_ok = v.structural();
    bool ok = st_ok && v.explore();
    uint32_t all_uniform = 0;
    if (ok) {
        v.hint_uniform.assign(n, 1);
        ok = v.simt(opts.simt_strict != 0, all_uniform);
        if (ok) v.divergence(); /* the sound GXF_UNIFORM branch hints the JIT relies on */
    } else if (st_ok && opts.simt_strict && !v.viol.empty() &&
               (v.viol[0].rule == GX_BUDGET || v.viol[0].rule == GX_COMPLEXITY || v.viol[0].rule == GX_UNBOUNDED_LOOP)) {
        /* strict mode: a loop that never terminates in exploration is usually a lane-varying loop
         * bound; report the SIMT rule first when the uniformity pass finds one */
        std::vector<Violation> first = v.viol;
        v.viol.clear();
        v.hint_uniform.assign(n, 1);
        v.simt(true, all_uniform);
        for (auto &x : first) v.viol.push_back(x);
    }
    gx_verify_report &rep = out.report;
    rep.n_insns = n;
    rep.processed_insns = v.processed;
    rep.n_violations = (uint32_t)v.viol.size();
    if (!v.viol.empty()) {
        const Violation &f = v.viol.front();
        rep.first_insn = f.insn;
        rep.first_rule = f.rule;
        rep.verdict = (f.rule == GX_COMPLEXITY || f.rule == GX_BUDGET) ? -7 /* -E2BIG */
                      : (f.rule == GX_BAD_INSN || f.rule == GX_BAD_REG || f.rule == GX_BAD_JUMP) ? -22 /* -EINVAL */
                                                                                                   : -13; /* -EACCES */
        for (auto &vv : v.viol) {
            char line[256];
            snprintf(line, sizeof line, "insn %u: %s: %s\n", vv.insn, gx_rule_name(vv.rule), vv.msg.c_str());
            out.log += line;
        }
        return rep.verdict;
    }
    if (v.worst_i > opts.max_insns || v.worst_h > opts.max_helpers || v.worst_m > opts.max_memops) {
        rep.verdict = -7;
        rep.first_rule = GX_BUDGET;
        rep.n_violations = 1;
        out.log += "insn 0: BUDGET: worst-case path exceeds the per-hook budget\n";
        return rep.verdict;
    }
    rep.worst_insns = v.worst_i;
    rep.worst_helpers = v.worst_h;
    rep.worst_memops = v.worst_m;
    rep.stack_depth = (v.max_stack + 7) & ~7u;
    rep.all_uniform = all_uniform;
    /* commutative (S1 sufficient flag, simplified): shared maps change only via ATOMIC ADD /
     * update(NOEXIST)-style inserts, and no shared map value is read */
    uint32_t comm = 1;
    for (int m = 0; m < GX_MAX_MAPS; m++) {
        const GxMapUse &u = out.use[m];
        if (!u.used || !maps[m].valid || maps[m].type == PT || maps[m].type == RINGBUF || maps[m].type == PFQ ||
            maps[m].type == REGION)
            continue;
        if (u.writes && (u.non_add_write && !u.update_call)) comm = 0;
        if (u.reads && u.writes) comm = 0;
    }
    rep.commutative = comm;
    out.stack_depth = rep.stack_depth;
    v.predecode();
    v.optimize(getenv("GX_NO_OPT") == nullptr);
    rep.image_insns = (uint32_t)out.image.size();
    rep.verdict = 0;
    return 0;
}
