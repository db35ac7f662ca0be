/*
 * gx_exec.cu -- the warp-cooperative eBPF executor for B200 (sm_100a).
 *
 * What it computes: for every event of the batch, the attached verified program runs to EXIT
 * on ctx = &event against the persistent maps ("preserving
 * eBPF's scalar semantics").  How:
 *   a1  a warp takes a 32-event record (1 KiB): two 16-B non-allocating vector loads per lane,
 *       prefetched one record ahead, staged into a per-warp SoA ctx area in shared memory;
 *   a2  the pre-decoded programs (16-B GxInsn) and the map descriptors are staged in shared
 *       memory once per block;
 *   a3  interpretation: the 11 eBPF registers live in shared memory as [reg][lane] u64 rows
 *       (conflict-free), the stack as [slot][lane]; while all active lanes share a PC the warp
 *       runs the UNIFORM-PC FAST PATH: one broadcast LDS.128 fetch + one uniform dispatch per
 *       instruction for all 32 events.  A split branch switches to the MIN-PC path:
 *       pc* = __reduce_min_sync over the active lanes' PCs and only lanes at pc* execute, until
 *       all PCs meet again (then back to the fast path);
 *   a4-a6  ARRAY / per-thread ARRAY / HASH helpers;
 *   a7  ATOMIC ops on shared map values are warp-aggregated: lanes are grouped by address
 *       (__all_sync fast check, else __match_any_sync), the group's operands reduced with
 *       __reduce_*_sync, and the group leader issues one L2 atomic ("executing
 *       policy logic once per warp using a designated warp leader", 312 "__ballot_sync and
 *       __shfl_sync"); FETCH lanes get old + their exclusive group prefix (a valid
 *       linearisation).  Write-only ADD accumulator ARRAYs are privatised in shared memory per
 *       block and flushed at the end ("aggregate them per warp, and store results
 *       into GPU-local shards");
 *   a8  ringbuf output: one atomicAdd per warp reserves the whole warp's records;
 *   a9  epilogue: privatised shards flushed, stats accumulated;
 *   a10 multi-program dispatch: a record runs one masked sub-pass per distinct attached program.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "gx_device.cuh"
#include "gx_internal.h"

using gxd::E_2BIG;
using gxd::E_AGAIN;
using gxd::E_EXIST;
using gxd::E_INVAL;
using gxd::E_NOENT;

#define GX_BLOCK 256
#define GX_WARPS (GX_BLOCK / 32)

namespace {

/* the event stream is read once: L1 no-allocate, L2 evict-first (keeps the maps resident) */
__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
    uint4 r;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ uint64_t sext(uint64_t v, unsigned bits) {
    if (bits >= 64) return v;
    uint64_t m = 1ull << (bits - 1);
    v &= (1ull << bits) - 1;
    return (v ^ m) - m;
}

__device__ __forceinline__ uint64_t bswap_w(uint64_t v, unsigned w) {
    uint64_t r = __byte_perm((uint32_t)(v >> 32), 0, 0x0123) | ((uint64_t)__byte_perm((uint32_t)v, 0, 0x0123) << 32);
    return w == 64 ? r : (r >> (64 - w));
}

/* sized global load / store of a naturally aligned access */
__device__ __forceinline__ uint64_t gload(uint64_t a, unsigned lg, bool coherent) {
    switch (lg) {
    case 0: return *reinterpret_cast<const volatile uint8_t *>(a);
    case 1: return *reinterpret_cast<const volatile uint16_t *>(a);
    case 2: return coherent ? *reinterpret_cast<const volatile uint32_t *>(a) : *reinterpret_cast<const uint32_t *>(a);
    default: return coherent ? gxd::ld_relaxed(reinterpret_cast<const uint64_t *>(a)) : *reinterpret_cast<const uint64_t *>(a);
    }
}
__device__ __forceinline__ void gstore(uint64_t a, unsigned lg, uint64_t v) {
    switch (lg) {
    case 0: *reinterpret_cast<uint8_t *>(a) = (uint8_t)v; break;
    case 1: *reinterpret_cast<uint16_t *>(a) = (uint16_t)v; break;
    case 2: *reinterpret_cast<uint32_t *>(a) = (uint32_t)v; break;
    default: *reinterpret_cast<uint64_t *>(a) = v; break;
    }
}
/* little-endian sized store into a (private) 8-byte word */
__device__ __forceinline__ void word_store(uint64_t *w, unsigned byte, unsigned lg, uint64_t v) {
    if (lg == 3) {
        *w = v;
        return;
    }
    unsigned bits = 8u << lg;
    uint64_t msk = ((1ull << bits) - 1) << (8 * byte);
    *w = (*w & ~msk) | ((v << (8 * byte)) & msk);
}

/* plain (non-atomic) RMW of a private word: stack slots and per-thread shards */
__device__ __forceinline__ uint64_t rmw_private(uint64_t *w, unsigned byte, bool w32, uint32_t op, uint64_t s,
                                                uint64_t r0, uint64_t &newv) {
    uint64_t full = *w;
    uint64_t old = w32 ? (full >> (8 * byte)) & 0xFFFFFFFFull : full;
    uint64_t m = w32 ? 0xFFFFFFFFull : ~0ull;
    s &= m;
    uint64_t nv;
    switch (op) {
    case 0x00: case 0x01: nv = old + s; break;
    case 0x40: case 0x41: nv = old | s; break;
    case 0x50: case 0x51: nv = old & s; break;
    case 0xA0: case 0xA1: nv = old ^ s; break;
    case 0xE1: nv = s; break;
    default: nv = (old == (r0 & m)) ? s : old; break; /* 0xF1 CMPXCHG */
    }
    nv &= m;
    if (w32) full = (full & ~(0xFFFFFFFFull << (8 * byte))) | (nv << (8 * byte));
    else full = nv;
    *w = full;
    newv = nv;
    return old;
}

/* 64-bit sum over the lanes of `mask` (all lanes of mask call it) */
__device__ __forceinline__ uint64_t group_sum64(unsigned mask, uint64_t v) {
    if (__all_sync(mask, v < (1ull << 27))) return __reduce_add_sync(mask, (uint32_t)v);
    uint64_t s0 = __reduce_add_sync(mask, (uint32_t)(v & 0xFFFF));
    uint64_t s1 = __reduce_add_sync(mask, (uint32_t)((v >> 16) & 0xFFFF));
    uint64_t s2 = __reduce_add_sync(mask, (uint32_t)((v >> 32) & 0xFFFF));
    uint64_t s3 = __reduce_add_sync(mask, (uint32_t)(v >> 48));
    return s0 + (s1 << 16) + (s2 << 32) + (s3 << 48);
}
__device__ __forceinline__ uint64_t group_reduce(unsigned mask, uint32_t op, uint64_t v, bool w32) {
    if (w32) {
        uint32_t x = (uint32_t)v;
        switch (op & 0xF0) {
        case 0x00: return __reduce_add_sync(mask, x);
        case 0x40: return __reduce_or_sync(mask, x);
        case 0x50: return __reduce_and_sync(mask, x);
        default: return __reduce_xor_sync(mask, x);
        }
    }
    uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    switch (op & 0xF0) {
    case 0x00: return group_sum64(mask, v);
    case 0x40: return __reduce_or_sync(mask, lo) | ((uint64_t)__reduce_or_sync(mask, hi) << 32);
    case 0x50: return __reduce_and_sync(mask, lo) | ((uint64_t)__reduce_and_sync(mask, hi) << 32);
    default: return __reduce_xor_sync(mask, lo) | ((uint64_t)__reduce_xor_sync(mask, hi) << 32);
    }
}
__device__ __forceinline__ uint64_t apply_op(uint32_t op, uint64_t a, uint64_t b) {
    switch (op & 0xF0) {
    case 0x00: return a + b;
    case 0x40: return a | b;
    case 0x50: return a & b;
    default: return a ^ b;
    }
}
__device__ __forceinline__ uint64_t global_atomic(uint32_t op, uint64_t addr, uint64_t v, bool w32, bool fetch) {
    if (w32) {
        unsigned *p = reinterpret_cast<unsigned *>(addr);
        uint32_t x = (uint32_t)v;
        switch (op & 0xF0) {
        case 0x00: if (!fetch) { atomicAdd(p, x); return 0; } return atomicAdd(p, x);
        case 0x40: return atomicOr(p, x);
        case 0x50: return atomicAnd(p, x);
        default: return atomicXor(p, x);
        }
    }
    unsigned long long *p = reinterpret_cast<unsigned long long *>(addr);
    switch (op & 0xF0) {
    case 0x00: if (!fetch) { atomicAdd(p, v); return 0; } return atomicAdd(p, v);
    case 0x40: return atomicOr(p, v);
    case 0x50: return atomicAnd(p, v);
    default: return atomicXor(p, v);
    }
}

/* XCHG on a shared map value, called by the lanes of `mask`: lanes on one address take the group's
 * sequential result in lane order (the first gets the old value, each later lane the value of the
 * lane before it; the word keeps the last lane's value) with one atomicExch per address. */
__device__ __forceinline__ uint64_t group_xchg(unsigned mask, uint64_t addr, uint64_t v, bool w32) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(mask, addr);
    const int last = 31 - __clz(peers);
    const unsigned below = peers & ((1u << lane) - 1);
    const int prev = below ? 31 - __clz(below) : (int)lane;
    uint64_t old = 0;
    if ((int)lane == last)
        old = w32 ? (uint64_t)atomicExch(reinterpret_cast<unsigned *>(addr), (uint32_t)v)
                  : (uint64_t)atomicExch(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)v);
    old = __shfl_sync(peers, old, last);
    const uint64_t pv = __shfl_sync(peers, v, prev);
    const uint64_t r = below ? pv : old;
    return w32 ? (uint32_t)r : r;
}
/* CMPXCHG (cmp = r0): the group's sequential outcome in lane order from one read of the word,
 * committed with one CAS old -> final (recomputed from the returned value if another warp changed
 * the word).  W: 32-bit compare and result, zero-extended. */
__device__ __forceinline__ uint64_t group_cmpxchg(unsigned mask, uint64_t addr, uint64_t cmp, uint64_t v, bool w32) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(mask, addr);
    const int gl = __ffs(peers) - 1;
    const uint64_t M = w32 ? 0xFFFFFFFFull : ~0ull;
    cmp &= M;
    v &= M;
    uint64_t cur = 0;
    if ((int)lane == gl) {
        if (w32) {
            uint32_t t;
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(t) : "l"(addr) : "memory");
            cur = t;
        } else {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(addr) : "memory");
        }
    }
    cur = __shfl_sync(peers, cur, gl);
    for (;;) {
        uint64_t c = cur, mine = 0;
        for (unsigned m = peers; m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            const uint64_t cj = __shfl_sync(peers, cmp, j), vj = __shfl_sync(peers, v, j);
            if (j == (int)lane) mine = c;
            if (c == cj) c = vj;
        }
        uint64_t got = 0;
        if ((int)lane == gl)
            got = w32 ? (uint64_t)atomicCAS(reinterpret_cast<unsigned *>(addr), (uint32_t)cur, (uint32_t)c)
                      : (uint64_t)atomicCAS(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)cur,
                                            (unsigned long long)c);
        got = __shfl_sync(peers, got, gl);
        if (got == cur) return mine;
        cur = got;
    }
}

struct Smem {
    GxInsn *prog;
    GxMapDesc *maps;
    int8_t *attach;
    uint32_t *priv;
    unsigned long long *stats;
};

}  // namespace

extern "C" __global__ void __launch_bounds__(GX_BLOCK) gx_exec_kernel(const GxLaunch *__restrict__ L,
                                                                        const uint4 *__restrict__ events,
                                                                        uint64_t n_events, uint64_t *__restrict__ ret) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;

    /* ---------------- shared-memory carve-up (must match gx_runtime.cpp smem_bytes()) */
    const uint32_t staged = L->staged_insns, sslots = L->stack_slots, priv_bytes = L->priv_bytes;
    unsigned char *p = smem_raw;
    GxInsn *sprog = reinterpret_cast<GxInsn *>(p);
    p += staged * sizeof(GxInsn);
    GxMapDesc *M = reinterpret_cast<GxMapDesc *>(p);
    p += GX_MAX_MAPS * sizeof(GxMapDesc);
    int8_t *sattach = reinterpret_cast<int8_t *>(p);
    p += GX_MAX_KINDS * 256;
    uint32_t *spriv = reinterpret_cast<uint32_t *>(p);
    p += priv_bytes;
    unsigned long long *sstats = reinterpret_cast<unsigned long long *>(p);
    p += 8 * sizeof(unsigned long long);
    const uint32_t per_warp = (GX_NREGS + 4 + sslots) * 32; /* u64 words */
    uint64_t *R = reinterpret_cast<uint64_t *>(p) + wib * per_warp;
    uint64_t *C = R + GX_NREGS * 32;
    uint64_t *K = C + 4 * 32 - (int64_t)(GX_STACK_SIZE / 8 - sslots) * 32; /* K[(addr>>3)*32+lane] */

    /* ---------------- a2: stage programs, map descriptors, attach table; zero shards/stats */
    for (uint32_t q = 0; q < L->n_progs; q++) {
        const GxInsn *src = reinterpret_cast<const GxInsn *>(L->progs[q].image);
        const uint32_t off = L->progs[q].smem_off, cnt = L->progs[q].n;
        for (uint32_t i = tid; i < cnt; i += GX_BLOCK) sprog[off + i] = src[i];
    }
    for (uint32_t i = tid; i < GX_MAX_MAPS * sizeof(GxMapDesc) / 4; i += GX_BLOCK)
        reinterpret_cast<uint32_t *>(M)[i] = reinterpret_cast<const uint32_t *>(L->maps)[i];
    for (uint32_t i = tid; i < GX_MAX_KINDS * 256 / 4; i += GX_BLOCK)
        reinterpret_cast<uint32_t *>(sattach)[i] = reinterpret_cast<const uint32_t *>(L->attach)[i];
    for (uint32_t i = tid; i < priv_bytes / 4; i += GX_BLOCK) spriv[i] = 0;
    if (tid < 8) sstats[tid] = 0;
    R[10 * 32 + lane] = GX_STACK_SIZE; /* r10 = frame pointer (stack addresses are [0,512)) */
    __syncthreads();

    const int32_t single = L->single;
    const uint32_t shard = blockIdx.x * GX_BLOCK + tid;
    const uint64_t nrec = (n_events + 31) >> 5;
    const uint64_t total_warps = (uint64_t)gridDim.x * GX_WARPS;
    uint64_t c_run = 0, c_skip = 0, c_div = 0, c_herr = 0, c_rbb = 0, c_drop = 0, c_hfull = 0, c_steps = 0;

    /* ---------------- a1: event ingest, one record (32 events) per warp, prefetched */
    uint64_t rec = (uint64_t)blockIdx.x * GX_WARPS + wib;
    uint4 na = make_uint4(0, 0, 0, 0), nb = na;
    if (rec < nrec) {
        uint64_t idx = rec * 32 + lane;
        if (idx < n_events) {
            na = ldg_stream(events + 2 * idx);
            nb = ldg_stream(events + 2 * idx + 1);
        }
    }
    for (; rec < nrec; rec += total_warps) {
        const uint64_t idx = rec * 32 + lane;
        const bool valid = idx < n_events;
        const uint4 ca = na, cb = nb;
        {
            const uint64_t nrec2 = rec + total_warps;
            if (nrec2 < nrec) {
                uint64_t nidx = nrec2 * 32 + lane;
                if (nidx < n_events) {
                    na = ldg_stream(events + 2 * nidx);
                    nb = ldg_stream(events + 2 * nidx + 1);
                }
            }
        }
        C[0 * 32 + lane] = (uint64_t)ca.x | ((uint64_t)ca.y << 32);
        C[1 * 32 + lane] = (uint64_t)ca.z | ((uint64_t)ca.w << 32);
        C[2 * 32 + lane] = (uint64_t)cb.x | ((uint64_t)cb.y << 32);
        C[3 * 32 + lane] = (uint64_t)cb.z | ((uint64_t)cb.w << 32);

        /* a10: program selection */
        int myp = -1;
        if (valid) {
            if (single >= 0) myp = single;
            else {
                uint32_t hook = cb.x, kind = hook & 0xFF, tenant = (hook >> 8) & 0xFF;
                if (kind < GX_MAX_KINDS) myp = sattach[kind * 256 + tenant];
            }
        }
        const unsigned vmask = __ballot_sync(GX_FULL, valid);
        unsigned todo = __ballot_sync(GX_FULL, myp >= 0);
        if (lane == 0) c_skip += __popc(vmask & ~todo);
        if (ret && valid && myp < 0) ret[idx] = 0;
        __syncwarp();

        while (todo) {
            const int leader = __ffs(todo) - 1;
            const int pq = __shfl_sync(GX_FULL, myp, leader);
            const unsigned mask = __ballot_sync(GX_FULL, myp == pq) & todo;
            todo &= ~mask;
            const GxInsn *P = sprog + L->progs[pq].smem_off;
            if (lane == 0) c_run += __popc(mask);
            R[1 * 32 + lane] = 0; /* r1 = ctx */

            /* ---------------- a3: the interpreter */
            unsigned active = mask;
            uint32_t pc = 0, mypc = 0;
            bool uni = true;
            for (;;) {
                unsigned exec;
                if (uni) {
                    exec = active;
                } else {
                    const uint32_t v = ((active >> lane) & 1) ? mypc : 0xFFFFFFFFu;
                    pc = __reduce_min_sync(GX_FULL, v);
                    exec = __ballot_sync(GX_FULL, v == pc);
                    if (exec == active) uni = true;
                    c_div++;
                }
                c_steps++;
                const bool me = (exec >> lane) & 1;
                GxInsn in;
                {   /* one 16-B broadcast LDS per instruction */
                    const uint4 w = reinterpret_cast<const uint4 *>(P)[pc];
                    in = *reinterpret_cast<const GxInsn *>(&w);
                }
                uint32_t npc = pc + 1, tgt = 0;
                bool taken = false;
                uint64_t *const RD = &R[in.dst * 32 + lane];
                const uint64_t S = (in.flags & GXF_X) ? R[in.src * 32 + lane] : in.imm;
                switch (in.op) {
                /* ---------------- ALU64 */
                case GX_ADD64: if (me) *RD = *RD + S; break;
                case GX_SUB64: if (me) *RD = *RD - S; break;
                case GX_MUL64: if (me) *RD = *RD * S; break;
                case GX_DIV64: if (me) *RD = S ? *RD / S : 0; break;
                case GX_SDIV64:
                    if (me) {
                        int64_t d = (int64_t)*RD, s = (int64_t)S;
                        *RD = s == 0 ? 0 : (d == INT64_MIN && s == -1) ? (uint64_t)d : (uint64_t)(d / s);
                    }
                    break;
                case GX_MOD64: if (me) *RD = S ? *RD % S : *RD; break;
                case GX_SMOD64:
                    if (me) {
                        int64_t d = (int64_t)*RD, s = (int64_t)S;
                        *RD = s == 0 ? (uint64_t)d : s == -1 ? 0 : (uint64_t)(d % s);
                    }
                    break;
                case GX_OR64: if (me) *RD = *RD | S; break;
                case GX_AND64: if (me) *RD = *RD & S; break;
                case GX_XOR64: if (me) *RD = *RD ^ S; break;
                case GX_LSH64: if (me) *RD = *RD << (S & 63); break;
                case GX_RSH64: if (me) *RD = *RD >> (S & 63); break;
                case GX_ARSH64: if (me) *RD = (uint64_t)((int64_t)*RD >> (S & 63)); break;
                case GX_NEG64: if (me) *RD = 0 - *RD; break;
                case GX_MOV64: if (me) *RD = S; break;
                case GX_MOVSX64: if (me) *RD = sext(S, in.aux); break;
                /* ---------------- ALU32 (results zero-extended) */
                case GX_ADD32: if (me) *RD = (uint32_t)((uint32_t)*RD + (uint32_t)S); break;
                case GX_SUB32: if (me) *RD = (uint32_t)((uint32_t)*RD - (uint32_t)S); break;
                case GX_MUL32: if (me) *RD = (uint32_t)((uint32_t)*RD * (uint32_t)S); break;
                case GX_DIV32: if (me) { uint32_t s = (uint32_t)S; *RD = s ? (uint32_t)*RD / s : 0; } break;
                case GX_SDIV32:
                    if (me) {
                        int32_t d = (int32_t)*RD, s = (int32_t)S;
                        *RD = (uint32_t)(s == 0 ? 0 : (d == INT32_MIN && s == -1) ? d : d / s);
                    }
                    break;
                case GX_MOD32: if (me) { uint32_t s = (uint32_t)S; *RD = s ? (uint32_t)*RD % s : (uint32_t)*RD; } break;
                case GX_SMOD32:
                    if (me) {
                        int32_t d = (int32_t)*RD, s = (int32_t)S;
                        *RD = (uint32_t)(s == 0 ? d : s == -1 ? 0 : d % s);
                    }
                    break;
                case GX_OR32: if (me) *RD = (uint32_t)*RD | (uint32_t)S; break;
                case GX_AND32: if (me) *RD = (uint32_t)*RD & (uint32_t)S; break;
                case GX_XOR32: if (me) *RD = (uint32_t)*RD ^ (uint32_t)S; break;
                case GX_LSH32: if (me) *RD = (uint32_t)((uint32_t)*RD << (S & 31)); break;
                case GX_RSH32: if (me) *RD = (uint32_t)*RD >> (S & 31); break;
                case GX_ARSH32: if (me) *RD = (uint32_t)((int32_t)*RD >> (S & 31)); break;
                case GX_NEG32: if (me) *RD = (uint32_t)(0u - (uint32_t)*RD); break;
                case GX_MOV32: if (me) *RD = (uint32_t)S; break;
                case GX_MOVSX32: if (me) *RD = (uint32_t)sext(S, in.aux); break;
                case GX_LE: if (me && in.aux < 64) *RD = *RD & ((1ull << in.aux) - 1); break;
                case GX_BE: if (me) *RD = bswap_w(*RD, in.aux); break;
                case GX_LDIMM: /* the pre-decoder dropped the second slot */
                    if (me) *RD = (in.flags & GXF_VAL_MAPV) ? M[in.aux].data + in.imm : in.imm;
                    break;

                /* ---------------- memory */
                case GX_LDX_CTX:
                    if (me) {
                        uint64_t v = C[(in.off >> 3) * 32 + lane] >> (8 * (in.off & 7));
                        if (in.aux < 3) v &= (1ull << (8u << in.aux)) - 1;
                        if (in.flags & GXF_SX) v = sext(v, 8u << in.aux);
                        *RD = v;
                    }
                    break;
                case GX_LDX_STACK:
                    if (me) {
                        uint64_t v = K[(in.off >> 3) * 32 + lane] >> (8 * (in.off & 7));
                        if (in.aux < 3) v &= (1ull << (8u << in.aux)) - 1;
                        if (in.flags & GXF_SX) v = sext(v, 8u << in.aux);
                        *RD = v;
                    }
                    break;
                case GX_LDX_MAP:
                    if (me) {
                        uint64_t v = gload(R[in.src * 32 + lane] + in.off, in.aux, M[in.imm].coherent);
                        if (in.flags & GXF_SX) v = sext(v, 8u << in.aux);
                        *RD = v;
                    }
                    break;
                case GX_LDX_PT:
                    if (me) {
                        uint64_t a = (uint64_t)gxd::pt_phys(M[in.imm], R[in.src * 32 + lane] + in.off, shard);
                        uint64_t v = gload(a, in.aux, false);
                        if (in.flags & GXF_SX) v = sext(v, 8u << in.aux);
                        *RD = v;
                    }
                    break;
                case GX_ST_STACK:
                    if (me) word_store(&K[(in.off >> 3) * 32 + lane], in.off & 7, in.aux, S);
                    break;
                case GX_ST_MAP:
                    if (me) gstore(R[in.dst * 32 + lane] + in.off, in.aux, S);
                    break;
                case GX_ST_PT:
                    if (me) gstore((uint64_t)gxd::pt_phys(M[in.aux >> 4], R[in.dst * 32 + lane] + in.off, shard), in.aux & 15, S);
                    break;
                case GX_ATOM_STACK:
                    if (me) {
                        const uint32_t op = (uint32_t)(in.imm & 0xFF);
                        uint64_t nv, s = (in.flags & GXF_PRIV) ? (uint64_t)(int64_t)(int32_t)(in.imm >> 32) : R[in.src * 32 + lane];
                        uint64_t old = rmw_private(&K[(in.off >> 3) * 32 + lane], in.off & 7, (in.aux & 15) == 2,
                                                   op, s, R[lane], nv);
                        if (op == 0xF1) R[lane] = old;
                        else if (in.flags & GXF_FETCH) R[in.src * 32 + lane] = old;
                    }
                    break;
                case GX_ATOM_PT:
                    if (me) {
                        const uint64_t a = (uint64_t)gxd::pt_phys(M[in.aux >> 4], R[in.dst * 32 + lane] + in.off, shard);
                        const bool w32 = (in.aux & 15) == 2;
                        const uint32_t op = (uint32_t)(in.imm & 0xFF);
                        uint64_t nv, s = (in.flags & GXF_PRIV) ? (uint64_t)(int64_t)(int32_t)(in.imm >> 32) : R[in.src * 32 + lane];
                        uint64_t *w = reinterpret_cast<uint64_t *>(a & ~7ull);
                        uint64_t old = rmw_private(w, a & 7, w32, op, s, R[lane], nv);
                        if (op == 0xF1) R[lane] = old;
                        else if (in.flags & GXF_FETCH) R[in.src * 32 + lane] = old;
                    }
                    break;
                case GX_ATOM_MAP: {
                    /* a7: warp-aggregated atomics on shared map values */
                    const uint32_t op = (uint32_t)(in.imm & 0xFF);
                    const bool w32 = (in.aux & 15) == 2;
                    const GxMapDesc &md = M[in.aux >> 4];
                    const uint64_t addr = me ? R[in.dst * 32 + lane] + in.off : 0;
                    const uint64_t sv = !me ? 0 : (in.flags & GXF_PRIV) ? (uint64_t)(int64_t)(int32_t)(in.imm >> 32)
                                                                       : R[in.src * 32 + lane];
                    if (op == 0xE1 || op == 0xF1) { /* XCHG / CMPXCHG: the sequential result in lane order */
                        if (me) {
                            if (op == 0xE1) R[in.src * 32 + lane] = group_xchg(exec, addr, sv, w32);
                            else R[lane] = group_cmpxchg(exec, addr, R[lane], sv, w32);
                        }
                        break;
                    }
                    const bool fetch = op & 1;
                    if (md.priv_off != 0xFFFFFFFFu) {
                        /* privatised write-only ADD accumulator (verifier fact): shared-memory
                         * lo/hi u32 counters, flushed once per block */
                        const uint32_t nw = md.max_entries * md.value_size / 8;
                        uint32_t *lo = spriv + md.priv_off / 4, *hi = lo + nw;
                        const uint32_t leader = __ffs(exec) - 1;
                        const uint64_t a0 = __shfl_sync(GX_FULL, addr, leader);
                        uint64_t v = sv, a = addr;
                        bool doit = me;
                        if (__all_sync(GX_FULL, !me || addr == a0)) {
                            v = group_sum64(GX_FULL, sv);
                            a = a0;
                            doit = lane == leader;
                        }
                        if (doit) {
                            const uint32_t w = (uint32_t)((a - md.data) >> 3);
                            const uint32_t old = atomicAdd(&lo[w], (uint32_t)v);
                            const uint32_t carry = ((uint32_t)(old + (uint32_t)v) < old) ? 1u : 0u;
                            const uint32_t h = (uint32_t)(v >> 32) + carry;
                            if (h) atomicAdd(&hi[w], h);
                        }
                        break;
                    }
                    const uint32_t leader = __ffs(exec) - 1;
                    const uint64_t a0 = __shfl_sync(GX_FULL, addr, leader);
                    if (__all_sync(GX_FULL, !me || addr == a0)) {
                        /* every executing lane targets one address: one atomic for the warp */
                        const uint64_t ident = (op & 0xF0) == 0x50 ? ~0ull : 0;
                        const uint64_t mine = me ? sv : ident;
                        if (!fetch) {
                            const uint64_t agg = group_reduce(GX_FULL, op, mine, w32);
                            if (lane == leader) global_atomic(op, a0, agg, w32, false);
                        } else {
                            /* inclusive scan over the warp in lane order */
                            uint64_t inc = w32 ? (uint32_t)mine : mine;
                            for (int d = 1; d < 32; d <<= 1) {
                                uint64_t o = __shfl_up_sync(GX_FULL, inc, d);
                                if ((int)lane >= d) inc = apply_op(op, inc, o);
                            }
                            if (w32) inc = (uint32_t)inc;
                            const uint64_t agg = __shfl_sync(GX_FULL, inc, 31);
                            uint64_t old = 0;
                            if (lane == leader) old = global_atomic(op, a0, agg, w32, true);
                            old = __shfl_sync(GX_FULL, old, leader);
                            /* exclusive prefix = inclusive of the previous lane */
                            uint64_t exc = __shfl_up_sync(GX_FULL, inc, 1);
                            if (lane == 0) exc = ident;
                            uint64_t res = apply_op(op, old, exc);
                            if (w32) res = (uint32_t)res;
                            if (me) R[in.src * 32 + lane] = res;
                        }
                        break;
                    }
                    /* mixed addresses: per-lane atomics for plain ops; address groups for FETCH */
                    if (!fetch) {
                        if (me) global_atomic(op, addr, sv, w32, false);
                        break;
                    }
                    const unsigned peers = __match_any_sync(GX_FULL, me ? addr : 0ull);
                    if (me) {
                        const uint32_t gl = __ffs(peers) - 1;
                        uint64_t pre = (op & 0xF0) == 0x50 ? ~0ull : 0, tot = pre;
                        for (unsigned m = peers; m; m &= m - 1) {
                            const int j = __ffs(m) - 1;
                            const uint64_t vj = __shfl_sync(peers, sv, j);
                            if (j < (int)lane) pre = apply_op(op, pre, vj);
                            tot = apply_op(op, tot, vj);
                        }
                        uint64_t old = 0;
                        if (lane == gl) old = global_atomic(op, addr, tot, w32, true);
                        old = __shfl_sync(peers, old, gl);
                        uint64_t res = apply_op(op, old, pre);
                        R[in.src * 32 + lane] = w32 ? (uint32_t)res : res;
                    }
                    break;
                }

                /* ---------------- helpers (a4-a6, a8) */
                case GX_CALL_LOOKUP_ARRAY:
                case GX_CALL_LOOKUP_PT:
                    if (me) {
                        const GxMapDesc &md = M[in.aux];
                        const uint32_t k = (in.flags & GXF_KEY_MAPV) ? *reinterpret_cast<const uint32_t *>(R[2 * 32 + lane])
                                                                      : (uint32_t)(K[(in.off >> 3) * 32 + lane] >> (8 * (in.off & 7)));
                        R[lane] = k < md.max_entries ? md.data + (uint64_t)k * md.value_size : 0;
                    }
                    if (in.flags & (GXF_FETCH | GXF_W32)) goto lookup_branch;
                    break;
                case GX_CALL_LOOKUP_HASH: {
                    const GxMapDesc &md = M[in.aux];
                    uint64_t k = 0;
                    if (me) {
                        k = (in.flags & GXF_KEY_MAPV)
                                ? (md.key_size == 4 ? *reinterpret_cast<const uint32_t *>(R[2 * 32 + lane])
                                                    : *reinterpret_cast<const uint64_t *>(R[2 * 32 + lane]))
                                : K[(in.off >> 3) * 32 + lane] >> (8 * (in.off & 7));
                        if (md.key_size == 4) k &= 0xFFFFFFFFull;
                    }
                    uint64_t *v = gxd::hash_lookup_coop(md, k, me, GX_FULL);
                    if (me) R[lane] = (uint64_t)v;
                    if (in.flags & (GXF_FETCH | GXF_W32)) goto lookup_branch;
                    break;
                }
                case GX_CALL_UPDATE_ARRAY:
                case GX_CALL_UPDATE_PT:
                    if (me) {
                        const GxMapDesc &md = M[in.aux];
                        const uint32_t k = (in.flags & GXF_KEY_MAPV) ? *reinterpret_cast<const uint32_t *>(R[2 * 32 + lane])
                                                                      : (uint32_t)(K[(in.off >> 3) * 32 + lane] >> (8 * (in.off & 7)));
                        const uint64_t flags = R[4 * 32 + lane];
                        /* ARRAY: lanes copying into one key (flags ANY / EXIST) keep the sequential
                         * result, the last such lane's value */
                        const bool copies = flags == 0 || flags == 2;
                        const unsigned kg = in.op == GX_CALL_UPDATE_ARRAY
                                                ? __match_any_sync(exec, k) & __ballot_sync(exec, copies) : (1u << lane);
                        int64_t rc = 0;
                        if (flags > 2) rc = -E_INVAL;
                        else if (k >= md.max_entries) rc = -E_2BIG;
                        else if (flags == 1) rc = -E_EXIST;
                        else if ((int)lane == 31 - __clz(kg)) {
                            const uint32_t nw = md.value_size / 8;
                            for (uint32_t w = 0; w < nw; w++) {
                                const uint64_t v = (in.flags & GXF_VAL_MAPV)
                                                       ? reinterpret_cast<const uint64_t *>(R[3 * 32 + lane])[w]
                                                       : K[((uint32_t)in.imm / 8 + w) * 32 + lane];
                                const uint64_t logical = md.data + (uint64_t)k * md.value_size + 8 * w;
                                if (in.op == GX_CALL_UPDATE_ARRAY) *reinterpret_cast<uint64_t *>(logical) = v;
                                else *reinterpret_cast<uint64_t *>(gxd::pt_phys(md, logical, shard)) = v;
                            }
                        }
                        if (rc) c_herr++;
                        R[lane] = (uint64_t)rc;
                    }
                    break;
                case GX_CALL_UPDATE_HASH: {
                    const GxMapDesc &md = M[in.aux];
                    uint64_t k = 0, v = 0, fl = 0;
                    if (me) {
                        k = (in.flags & GXF_KEY_MAPV)
                                ? (md.key_size == 4 ? *reinterpret_cast<const uint32_t *>(R[2 * 32 + lane])
                                                    : *reinterpret_cast<const uint64_t *>(R[2 * 32 + lane]))
                                : K[(in.off >> 3) * 32 + lane] >> (8 * (in.off & 7));
                        if (md.key_size == 4) k &= 0xFFFFFFFFull;
                        v = (in.flags & GXF_VAL_MAPV) ? *reinterpret_cast<const uint64_t *>(R[3 * 32 + lane])
                                                      : K[((uint32_t)in.imm / 8) * 32 + lane];
                        fl = R[4 * 32 + lane];
                    }
                    bool full;
                    const int64_t rc = gxd::hash_update_coop(md, k, v, fl, me, GX_FULL);
                    full = rc == -E_2BIG;
                    if (me) {
                        if (rc) c_herr++;
                        if (full) c_hfull++;
                        R[lane] = (uint64_t)rc;
                    }
                    break;
                }
                case GX_CALL_RINGBUF_OUTPUT: {
                    const GxMapDesc &md = M[in.aux];
                    const uint32_t size = (uint32_t)in.imm, flags = (uint32_t)(in.imm >> 32);
                    if (flags > 2) {
                        if (me) {
                            R[lane] = (uint64_t)(int64_t)-E_INVAL;
                            c_herr++;
                        }
                        break;
                    }
                    const uint64_t recb = (8 + size + 7) & ~7u;
                    const uint32_t cnt = __popc(exec), rank = __popc(exec & ((1u << lane) - 1));
                    const uint32_t leader = __ffs(exec) - 1;
                    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(md.aux);
                    uint64_t base = 0;
                    if (lane == leader) base = atomicAdd(&ctr[0], (unsigned long long)(cnt * recb));
                    base = __shfl_sync(GX_FULL, base, leader);
                    const uint64_t o = base + rank * recb;
                    const uint64_t cap = (uint64_t)md.cap_mask + 1;
                    const bool ok = me && (o + recb <= cap);
                    if (ok) {
                        uint64_t *dst = reinterpret_cast<uint64_t *>(md.data + o);
                        dst[0] = (uint64_t)size | ((o >> 12) << 32);
                        const uint32_t nw = (size + 7) / 8;
                        for (uint32_t w = 0; w < nw; w++) {
                            uint64_t v = (in.flags & GXF_VAL_MAPV) ? reinterpret_cast<const uint64_t *>(R[2 * 32 + lane])[w]
                                                                   : K[((uint32_t)(uint16_t)in.off / 8 + w) * 32 + lane];
                            if (w == nw - 1 && (size & 7)) v &= (1ull << (8 * (size & 7))) - 1;
                            dst[1 + w] = v;
                        }
                        R[lane] = 0;
                    } else if (me) {
                        R[lane] = (uint64_t)(int64_t)-E_AGAIN;
                        c_drop++;
                        c_herr++;
                    }
                    const uint32_t nok = __popc(__ballot_sync(GX_FULL, ok));
                    if (nok && lane == leader) {
                        atomicAdd(&ctr[1], (unsigned long long)(nok * recb));
                        c_rbb += nok * recb;
                    }
                    break;
                }

                case GX_CALL_PREFETCH_L2: {
                    if (me) {
                        const int64_t rc = gxd::l2_prefetch(M[in.aux], R[2 * 32 + lane], R[3 * 32 + lane]);
                        if (rc) c_herr++;
                        R[lane] = (uint64_t)rc;
                    }
                    break;
                }

                case GX_CALL_MEM_PREFETCH: {
                    const int64_t rc = gxd::pfq_request_coop(M[in.aux], R[2 * 32 + lane], R[3 * 32 + lane], me, GX_FULL, c_drop);
                    if (me) {
                        if (rc) c_herr++;
                        R[lane] = (uint64_t)rc;
                    }
                    break;
                }

                /* ---------------- jumps */
                case GX_JA:
                    npc = in.aux;
                    break;
                case GX_EXIT:
                    if (me && ret) ret[idx] = (in.flags & GXF_SX) ? in.imm : R[lane];
                    active &= ~exec;
                    npc = 0xFFFFFFFFu;
                    break;
                default:
                    if (in.op >= GX_JEQ && in.op <= GX_JSET32) {
                        const bool is32 = in.op >= GX_JEQ32;
                        const uint32_t cop = is32 ? in.op - (GX_JEQ32 - GX_JEQ) : in.op;
                        uint64_t d = R[in.dst * 32 + lane], s = S;
                        int64_t sd = (int64_t)d, ss = (int64_t)s;
                        if (is32) {
                            d = (uint32_t)d;
                            s = (uint32_t)s;
                            sd = (int32_t)d;
                            ss = (int32_t)s;
                        }
                        switch (cop) {
                        case GX_JEQ: taken = d == s; break;
                        case GX_JNE: taken = d != s; break;
                        case GX_JGT: taken = d > s; break;
                        case GX_JGE: taken = d >= s; break;
                        case GX_JLT: taken = d < s; break;
                        case GX_JLE: taken = d <= s; break;
                        case GX_JSGT: taken = sd > ss; break;
                        case GX_JSGE: taken = sd >= ss; break;
                        case GX_JSLT: taken = sd < ss; break;
                        case GX_JSLE: taken = sd <= ss; break;
                        default: taken = (d & s) != 0; break;
                        }
                        tgt = in.aux;
                        goto do_branch;
                    } else {
                        /* GX_OP_NOP: an instruction the verifier proved unreachable -- trap */
                        active &= ~exec;
                        if (me) c_herr++;
                        npc = 0xFFFFFFFFu;
                    }
                    break;
                }
                if (false) {
                lookup_branch:
                    taken = (in.flags & GXF_FETCH) ? R[lane] == 0 : R[lane] != 0;
                    tgt = (uint32_t)in.imm;
                do_branch:
                    taken = taken && me;
                    const unsigned tb = __ballot_sync(GX_FULL, taken);
                    if (uni) {
                        if (tb == exec) npc = tgt;
                        else if (tb != 0) {
                            uni = false;
                            mypc = taken ? tgt : pc + 1;
                            goto next_step;
                        }
                    } else {
                        npc = taken ? tgt : pc + 1;
                    }
                }
                if (uni) pc = npc;
                else if (me) mypc = npc;
            next_step:
                if (!active) break;
            }
        }
        __syncwarp();
    }

    /* ---------------- a9: epilogue -- stats and privatised shards */
    if (lane == 0) {
        atomicAdd(&sstats[GXS_RUN], c_run);
        atomicAdd(&sstats[GXS_SKIP], c_skip);
        atomicAdd(&sstats[GXS_DIVERGENT], c_div);
        atomicAdd(&sstats[GXS_STEPS], c_steps);
    }
    {
        /* per-lane counters */
        unsigned long long h = c_herr, rb = c_rbb, dr = c_drop, hf = c_hfull;
        for (int o = 16; o; o >>= 1) {
            h += __shfl_xor_sync(GX_FULL, h, o);
            rb += __shfl_xor_sync(GX_FULL, rb, o);
            dr += __shfl_xor_sync(GX_FULL, dr, o);
            hf += __shfl_xor_sync(GX_FULL, hf, o);
        }
        if (lane == 0) {
            if (h) atomicAdd(&sstats[GXS_HERR], h);
            if (rb) atomicAdd(&sstats[GXS_RB_BYTES], rb);
            if (dr) atomicAdd(&sstats[GXS_RB_DROPS], dr);
            if (hf) atomicAdd(&sstats[GXS_HFULL], hf);
        }
    }
    __syncthreads();
    for (uint32_t q = 0; q < L->n_priv; q++) {
        const GxMapDesc &md = M[L->priv_maps[q]];
        const uint32_t nw = md.max_entries * md.value_size / 8;
        const uint32_t *lo = spriv + md.priv_off / 4, *hi = lo + nw;
        unsigned long long *g = reinterpret_cast<unsigned long long *>(md.data);
        for (uint32_t w = tid; w < nw; w += GX_BLOCK) {
            const uint64_t v = (uint64_t)lo[w] | ((uint64_t)hi[w] << 32);
            if (v) atomicAdd(&g[w], v);
        }
    }
    if (tid < 8) {
        unsigned long long *gs = reinterpret_cast<unsigned long long *>(L->stats);
        if (sstats[tid]) atomicAdd(&gs[tid], sstats[tid]);
    }
}

/* host-side launcher (called from gx_runtime.cpp) */
extern "C" int gx_launch_exec(const GxLaunch *d_launch, const void *d_events, uint64_t n, uint64_t *d_ret,
                              uint32_t grid, uint32_t smem, cudaStream_t stream) {
    gx_exec_kernel<<<grid, GX_BLOCK, smem, stream>>>(d_launch, reinterpret_cast<const uint4 *>(d_events), n, d_ret);
    return (int)cudaGetLastError();
}

extern "C" int gx_exec_occupancy(uint32_t smem, int *blocks_per_sm) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(gx_exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return (int)e;
        attr_set = true;
    }
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, gx_exec_kernel, GX_BLOCK, smem);
}

extern "C" uint32_t gx_exec_block_threads() { return GX_BLOCK; }
