/*
 * gx_device.cuh -- device-side map primitives shared by the executor (gx_exec.cu) and the map
 * maintenance kernels (gx_maps.cu).  sm_100a only.
 */
#pragma once
#include <stdint.h>

#include "gx_internal.h"

#define GX_FULL 0xFFFFFFFFu

namespace gxd {

enum { E_NOENT = 2, E_2BIG = 7, E_AGAIN = 11, E_FAULT = 14, E_EXIST = 17, E_INVAL = 22 };

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t *p) {
    uint64_t r;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t *p) {
    uint64_t r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
}
/* HASH probes through L1 (keys are immutable once published): 0 never, 1 the home slot, 2 the whole
 * chain (default) */
#ifndef GX_HASH_L1PROBE
#define GX_HASH_L1PROBE 2
#endif
/* keys per probe step with the L1 chain (1, 2 or 4) */
#ifndef GX_HASH_PROBE_W
#define GX_HASH_PROBE_W 4
#endif
__device__ __forceinline__ uint64_t ld_nc(const uint64_t *p) {
    uint64_t r;
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint64_t ld_ca(const uint64_t *p) {
    uint64_t r;
    asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void st_relaxed(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

/* ---- HASH: open addressing, linear probing, keys and values in SEPARATE arrays of cap + 2 words
 * (cap = cap_mask + 1, a power of two >= 2 x max_entries):
 *     data[0 .. cap+1]            key words K: EMPTY (all-ones), BUSY (all-ones - 1: an insert in
 *                                 flight) or a published key; K[cap] / K[cap+1] are the presence
 *                                 states (0 absent, 2 inserting, 1 present) of the two keys that
 *                                 equal the sentinels, whose entries live in these side slots;
 *     data[cap+2 .. 2 cap+3]      value words V, V[i] belonging to K[i].
 * Values sit on lines of their own: the map's atomics (a hot LFU page takes millions of FETCH-ADDs
 * per batch) never contend with the probes that read keys (C3: 17 -> ~8 ms at 2^28 events,
 * profiles/r2_c3.md).  An insert claims a slot EMPTY -> BUSY (CAS), writes the value, and publishes
 * the key with a release store; a published key never changes (no deletes). */
constexpr uint64_t GX_HASH_BUSY = 0xFFFFFFFFFFFFFFFEull;
__device__ __forceinline__ uint64_t *hash_keys(const GxMapDesc &m) { return reinterpret_cast<uint64_t *>(m.data); }
__device__ __forceinline__ uint64_t *hash_vals(const GxMapDesc &m) {
    return reinterpret_cast<uint64_t *>(m.data) + (uint64_t)m.cap_mask + 3;
}
__device__ __forceinline__ void st_release(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

/* lookup: the value word of `key`, or nullptr.  An insert still in flight (BUSY) is not yet in the
 * map: a slot that was EMPTY when a probe for `key` passed it cannot be followed by `key`, so BUSY
 * ends the chain like EMPTY. */
__device__ __forceinline__ uint64_t *hash_find(const GxMapDesc &m, uint64_t key) {
    uint64_t *K = hash_keys(m), *V = hash_vals(m);
    const uint64_t cap = (uint64_t)m.cap_mask + 1;
    if (key == GX_HASH_EMPTY || key == GX_HASH_BUSY) {
        const uint64_t side = cap + (key == GX_HASH_BUSY ? 1 : 0);
        return ld_acquire(K + side) == 1 ? V + side : nullptr;
    }
    /* one slot per probe step: a 4-wide step measured 1.7x slower on C3 (round 1) */
    uint64_t h = mix64(key) & m.cap_mask;
#if GX_HASH_L1PROBE == 1
    /* home slot only through L1 (a key match there is final), then the coherent chain */
    if (ld_ca(K + h) == key) return V + h;
    for (uint64_t i = 0; i < cap; i++) {
        const uint64_t s = (h + i) & m.cap_mask;
        const uint64_t k = ld_acquire(K + s);
        if (k == key) return V + s;
        if (k >= GX_HASH_BUSY) return nullptr;
    }
#elif GX_HASH_L1PROBE
    /* a published key never changes, so any key read through L1 is final -- a match is the entry,
     * another key means probe on; only EMPTY / BUSY may be stale and are re-read at L2 (acquire:
     * the value written before the key's release is then visible).  The chain is read one 32-B
     * sector (4 key words, two 16-B loads, one L2 request) at a time in slot order: C3's chains of
     * ~1.5 slots per lane took 3.4 serial round trips per warp record one slot at a time. */
#if GX_HASH_PROBE_W == 1
    for (uint64_t i = 0; i < cap; i++) {
        const uint64_t s = (h + i) & m.cap_mask;
#if GX_HASH_L1PROBE == 3
        uint64_t k = ld_nc(K + s);
#else
        uint64_t k = ld_ca(K + s);
#endif
        if (k >= GX_HASH_BUSY) k = ld_acquire(K + s);
        if (k == key) return V + s;
        if (k >= GX_HASH_BUSY) return nullptr;
    }
#else
    constexpr uint32_t PW = GX_HASH_PROBE_W; /* 2 or 4 keys per step (16 or 32 B; a 32-B sector is one L2 request) */
    unsigned valid = ((1u << PW) - 1) << ((uint32_t)h & (PW - 1)); /* the first step starts at the home slot */
    for (uint64_t i = 0; i < cap; i += PW) {
        const uint64_t b = ((h & ~(uint64_t)(PW - 1)) + i) & m.cap_mask;
        uint64_t kk[PW];
#pragma unroll
        for (uint32_t q = 0; q < PW; q += 2) {
#if GX_HASH_L1PROBE == 3
            asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(kk[q]), "=l"(kk[q + 1]) : "l"(K + b + q));
#else
            asm volatile("ld.global.ca.v2.u64 {%0, %1}, [%2];" : "=l"(kk[q]), "=l"(kk[q + 1]) : "l"(K + b + q));
#endif
        }
        /* branch-free scan of the step: the first slot (in probe order) holding the key or a
         * sentinel decides */
        unsigned hit = 0, stop = 0;
#pragma unroll
        for (uint32_t j = 0; j < PW; j++) {
            hit |= (kk[j] == key ? 1u : 0u) << j;
            stop |= (kk[j] >= GX_HASH_BUSY ? 1u : 0u) << j;
        }
        hit &= valid;
        stop &= valid;
        valid = (1u << PW) - 1;
        if (hit | stop) {
            const uint32_t j = __ffs(hit | stop) - 1;
            if ((hit >> j) & 1) return V + b + j;
            /* EMPTY / BUSY read through L1 may be stale: re-read coherently; a key that arrived
             * meanwhile continues the chain slot by slot (rare) */
            for (uint64_t s = b + j, n = 0; n < cap; n++, s = (s + 1) & m.cap_mask) {
                const uint64_t k = ld_acquire(K + s);
                if (k == key) return V + s;
                if (k >= GX_HASH_BUSY) return nullptr;
            }
            return nullptr;
        }
    }
#endif
#else
    for (uint64_t i = 0; i < cap; i++) {
        const uint64_t s = (h + i) & m.cap_mask;
        const uint64_t k = ld_acquire(K + s);
        if (k == key) return V + s;
        if (k >= GX_HASH_BUSY) return nullptr;
    }
#endif
    return nullptr;
}

/* 1: the doing lanes of a warp run their insert attempts in lock-step rounds (required: with each
 * lane on its own, a lane waiting for reservations can starve a reservation holder of its own warp --
 * independent thread scheduling gives a spinning branch no fairness -- until the safety valve
 * refuses the insert; the fuzz caught it at a 1024-entry map filled to capacity) */
#ifndef GX_HASH_LOCKSTEP
#define GX_HASH_LOCKSTEP 1
#endif
#ifndef GX_HASH_VALVE
#define GX_HASH_VALVE (1u << 20)
#endif
/* bpf_map_update_elem on a HASH with 8-byte values (bpf.h:1762-1776): 0 or -errno; `full` set when
 * refused for capacity (hash_full).
 * Capacity (max_entries, exact): aux[1] counts committed entries, aux[2] reservations (committed +
 * in-flight inserts).  An insert of an absent key first reserves (aux[2]++); a reservation below
 * max_entries may claim its slot (EMPTY -> BUSY), write the value, publish the key and then commit
 * (aux[1]++); a lost claim returns the
 * reservation and probes again (the winner may hold our key).  With no reservation to be had: if the
 * committed count has reached max_entries the map is full for good, and one more probe that still
 * finds the key absent refuses the insert (-E2BIG, linearised at that probe); otherwise other inserts
 * hold the excess reservations only transiently -- each publishes or returns its reservation without
 * waiting on anything -- so the insert waits and probes again.  The map never holds more than
 * max_entries entries and never refuses an insert while it has room (reading I-22).
 *
 * hash_step is ONE attempt; `st` carries state between attempts (0 initially, kHashFullSeen after
 * the count reached max_entries).  Returns kHashDone (rc / full set), kHashAgain (probe again now)
 * or kHashWait (reservations in flight: back off, then probe again). */
enum { kHashDone = 0, kHashAgain = 1, kHashWait = 2, kHashFullSeen = 1 };
__device__ __forceinline__ int hash_step(const GxMapDesc &m, uint64_t key, uint64_t val, uint64_t flags, uint32_t &st,
                                         int64_t &rc, bool &full) {
    full = false;
    rc = 0;
    if (flags > 2) {
        rc = -E_INVAL;
        return kHashDone;
    }
    uint64_t *K = hash_keys(m), *V = hash_vals(m);
    unsigned long long *ctr = reinterpret_cast<unsigned long long *>(m.aux);
    const uint64_t cap = (uint64_t)m.cap_mask + 1;
    const bool side = key == GX_HASH_EMPTY || key == GX_HASH_BUSY;
    uint64_t s = 0;
    bool present = false;
    if (side) {
        s = cap + (key == GX_HASH_BUSY ? 1 : 0);
        const uint64_t st8 = ld_acquire(K + s);
        if (st8 == 2) return kHashWait; /* its insert is in flight */
        present = st8 == 1;
    } else {
        const uint64_t h = mix64(key) & m.cap_mask;
        uint64_t i = 0;
        for (; i < cap; i++) {
            s = (h + i) & m.cap_mask;
            const uint64_t k = ld_acquire(K + s);
            if (k == key) {
                present = true;
                break;
            }
            if (k == GX_HASH_BUSY) return kHashWait; /* an insert in flight: it may be this key */
            if (k == GX_HASH_EMPTY) break;
        }
        if (i == cap) {
            full = true;
            rc = -E_2BIG;
            return kHashDone;
        }
    }
    if (present) {
        if (flags == 1) rc = -E_EXIST;
        else st_relaxed(V + s, val);
        return kHashDone;
    }
    if (flags == 2) {
        rc = -E_NOENT;
        return kHashDone;
    }
    if (st == kHashFullSeen) { /* absent at a probe after the committed count reached max_entries */
        full = true;
        rc = -E_2BIG;
        return kHashDone;
    }
    /* a reservation: the counter is watched with a plain load first (no RMW storm on its line while
     * the map sits at its capacity) */
    bool got = false;
    if (ld_relaxed(reinterpret_cast<const uint64_t *>(&ctr[2])) < m.max_entries) {
        got = atomicAdd(&ctr[2], 1ull) < m.max_entries;
        if (!got) atomicAdd(&ctr[2], ~0ull); /* return it */
    }
    if (!got) {
        if (ld_relaxed(reinterpret_cast<const uint64_t *>(&ctr[1])) >= m.max_entries) {
            st = kHashFullSeen; /* full for good; our key may have arrived since the probe */
            return kHashAgain;
        }
        return kHashWait;
    }
    const unsigned long long from = side ? 0ull : GX_HASH_EMPTY, busy = side ? 2ull : GX_HASH_BUSY;
    if (atomicCAS(reinterpret_cast<unsigned long long *>(K + s), from, busy) == from) {
        st_relaxed(V + s, val);
        st_release(K + s, side ? 1ull : key);
        atomicAdd(&ctr[1], 1ull);
        return kHashDone;
    }
    atomicAdd(&ctr[2], ~0ull); /* lost the slot: return the reservation, probe again */
    return kHashAgain;
}
/* one thread on its own (host control-plane kernels, gx_maps.cu) */
__device__ __forceinline__ int64_t hash_update(const GxMapDesc &m, uint64_t key, uint64_t val, uint64_t flags,
                                               bool &full) {
    uint32_t st = 0, waits = 0;
    int64_t rc;
    for (;;) {
        const int r = hash_step(m, key, val, flags, st, rc, full);
        if (r == kHashDone) return rc;
        if (r == kHashWait) {
            if (++waits > GX_HASH_VALVE) { /* safety valve, far beyond any in-flight insert */
                full = true;
                return -E_2BIG;
            }
            __nanosleep(waits < 7 ? 32u << waits : 2048u);
        }
    }
}

/* JIT builds move the cold, code-heavy group paths out of line (one copy per module instead of one
 * per call site and per uniform / min-PC block copy); the interpreter keeps them inline. */
#if defined(GX_JIT) && !defined(GX_COLD_INLINE)
#define GXD_COLD __noinline__
#else
#define GXD_COLD __forceinline__
#endif

/* Warp-cooperative HASH helpers: the lanes of `mask` call together; `me` marks the lanes whose
 * event is executing the helper.  When every executing lane asks for the same key (a warp-uniform
 * key -- a page swept by a whole warp record in C3's prefill), one lane probes and the others reuse
 * its result instead of 31 probes on one chain.  Sequential equivalent: the leader's event goes first. */
__device__ __forceinline__ uint64_t *hash_lookup_coop(const GxMapDesc &m, uint64_t key, bool me, unsigned mask) {
    const unsigned part = __ballot_sync(mask, me);
    if (!part) return nullptr;
    const unsigned lane = threadIdx.x & 31;
    const int leader = __ffs(part) - 1;
    const uint64_t k0 = __shfl_sync(mask, key, leader);
    if (__all_sync(mask, !me || key == k0)) {
        uint64_t *v = nullptr;
        if ((int)lane == leader) v = hash_find(m, key);
        return reinterpret_cast<uint64_t *>(__shfl_sync(mask, reinterpret_cast<unsigned long long>(v), leader));
    }
    return me ? hash_find(m, key) : nullptr;
}
/* update(map, key, val, flags): lanes asking for the same key with the same flags form a group
 * (__match_any_sync) and take the group's SEQUENTIAL result in lane order with one map update (S1;
 * the lanes of a record are consecutive events):
 *   NOEXIST -- the group's first lane inserts (0 / -EEXIST / -E2BIG); the later lanes then find the
 *              key present (-EEXIST), or the map still full (-E2BIG);
 *   ANY / EXIST -- every lane meets the same state (present: all overwrite, the last value stays;
 *              absent: all insert-or-overwrite, resp. all -ENOENT; full: all -E2BIG), so the group's
 *              LAST lane performs the update with its value and every lane takes its result.
 * The doing lanes of the warp run their attempts in lock-step rounds (hash_step), so a lane waiting
 * for reservations never spins past a lane of its own warp that holds one. */
__device__ GXD_COLD int64_t hash_update_coop(const GxMapDesc m, uint64_t key, uint64_t val, uint64_t flags, bool me,
                                             unsigned mask) {
    const unsigned part = __ballot_sync(mask, me);
    if (!me) return 0;
    const unsigned lane = threadIdx.x & 31;
    const unsigned grp = __match_any_sync(part, key) & __match_any_sync(part, flags);
    const int doer = flags == 1 ? __ffs(grp) - 1 : 31 - __clz(grp);
    const bool is_doer = (int)lane == doer;
#if GX_HASH_LOCKSTEP
    /* the doing lanes of the warp run their attempts in lock-step rounds */
    const unsigned doers = __ballot_sync(part, is_doer);
    int64_t rc = 0;
    if (is_doer) {
        bool f = false;
        uint32_t st = 0, waits = 0;
        unsigned pend = doers;
        for (;;) {
            const int r = hash_step(m, key, val, flags, st, rc, f);
            const unsigned still = __ballot_sync(pend, r != kHashDone);
            if (r == kHashDone) break;
            if (__any_sync(still, r == kHashWait)) {
                if (++waits > GX_HASH_VALVE) { /* safety valve, far beyond any in-flight insert */
                    rc = -E_2BIG;
                    break;
                }
                __nanosleep(waits < 7 ? 32u << waits : 2048u);
            }
            pend = still;
        }
    }
#else
    /* each doing lane on its own (measurement knob only; see GX_HASH_LOCKSTEP) */
    int64_t rc = 0;
    if (is_doer) {
        bool f;
        rc = hash_update(m, key, val, flags, f);
    }
#endif
    rc = (int64_t)__shfl_sync(grp, (unsigned long long)rc, doer);
    if (!is_doer && flags == 1 && rc == 0) rc = -E_EXIST;
    return rc; /* refused for capacity (hash_full) exactly when -E2BIG */
}

/* ---- PREFETCH QUEUE: gdev_mem_prefetch(queue, addr, len) (F-1..F-3).
 * Called by every lane of `mask`; `me` marks lanes whose event executes the helper.  A request is
 * the page run {addr >> 12, npages}; identical requests of the group are merged (prefetching is
 * idempotent, F-2) -- one queue slot per distinct request, one atomicAdd per group.  Slots at or
 * beyond the capacity are dropped (-EAGAIN, counted per requesting lane). */
template <typename Counter>
__device__ __forceinline__ int64_t pfq_request_coop(const GxMapDesc &md, uint64_t addr, uint64_t len, bool me,
                                                    unsigned mask, Counter &drops) {
    const bool valid = me && len != 0 && len <= (2ull << 20) && addr + len >= addr;
    uint64_t first = 0, np = 0;
    if (valid) {
        first = addr >> 12;
        np = ((addr + len - 1) >> 12) - first + 1;
    }
    const unsigned vm = __ballot_sync(mask, valid);
    if (!vm) return me ? -(int64_t)E_INVAL : 0;
    const uint64_t key = valid ? (first << 10) | (np - 1) : ~0ull; /* first < 2^52, np <= 513 */
    const unsigned peers = __match_any_sync(mask, key);
    const unsigned lane = threadIdx.x & 31;
    const unsigned myhead = __ffs(peers) - 1;
    bool head = valid && myhead == lane;
    /* request filter (md.nshards words after the records, emptied at every drain): a request
     * whose filter word already holds it was queued earlier in this drain epoch -- set semantics
     * let it go; a plain load first keeps hot requests off the atomic unit */
    bool dup = false;
    unsigned long long *fw = nullptr;
    const unsigned long long tag = key + 1;
    if (head) {
        unsigned long long *filt =
            reinterpret_cast<unsigned long long *>(md.data + 16ull * ((uint64_t)md.cap_mask + 1));
        fw = filt + (mix64(key) & (md.nshards - 1));
        dup = ld_relaxed(reinterpret_cast<const uint64_t *>(fw)) == tag || atomicExch(fw, tag) == tag;
        head = !dup;
    }
    const bool dup_g = __shfl_sync(mask, dup, myhead);
    const unsigned heads = __ballot_sync(mask, head);
    unsigned long long base = 0;
    if (heads) { /* uniform over the group */
        const unsigned leader = __ffs(heads) - 1;
        if (lane == leader) base = atomicAdd(reinterpret_cast<unsigned long long *>(md.aux), (unsigned long long)__popc(heads));
        base = __shfl_sync(mask, base, leader);
    }
    const uint64_t slot = base + __popc(heads & ((1u << myhead) - 1));
    const bool ok = slot <= (uint64_t)md.cap_mask;
    if (head && ok) {
        uint64_t *d = reinterpret_cast<uint64_t *>(md.data + 16 * slot);
        d[0] = first;
        d[1] = np;
    }
    /* a dropped request was not queued: take it back out of the filter so a repeat is refused
     * (-EAGAIN, counted) like the oracle's, not passed as a duplicate */
    if (head && !ok) atomicCAS(fw, tag, 0ull);
    if (!me) return 0;
    if (!valid) return -(int64_t)E_INVAL;
    if (dup_g) return 0;
    if (!ok) {
        drops++;
        return -(int64_t)E_AGAIN;
    }
    return 0;
}

/* gdev_prefetch_l2(region, addr, len) (F-7; "Device-side L2 prefetch
 * instructions (prefetch.global.L2)", Table 1 "GPU L2 Stride Prefetch"): per lane, one
 * prefetch.global.L2 per 128-B line of [addr, addr + len) when the range lies inside the REGION map
 * [md.data, md.data + md.aux) (caller-owned device memory registered with gx_region_map).  R0: 0,
 * -EINVAL (len 0 or > 64 KiB), -EFAULT (not inside the region).  A hint: no state changes. */
__device__ __forceinline__ int64_t l2_prefetch(const GxMapDesc &md, uint64_t addr, uint64_t len) {
    if (len == 0 || len > 65536) return -(int64_t)E_INVAL;
    const uint64_t off = addr - md.data;
    if (addr < md.data || off > md.aux || len > md.aux - off) return -(int64_t)E_FAULT;
    const uint64_t end = addr + len;
    for (uint64_t a = addr & ~127ull; a < end; a += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    return 0;
}

/* ---- per-thread ARRAY (S4): one private copy per executor thread ("shard").  Value pointers a
 * program holds are LOGICAL addresses data + key*vs + off; the physical word is
 *     pt_word_index(K, W, k, w, shard) = ((q*K*W) + ((k - r) mod K)*W + w) * 32 + l
 * with shard = 32q + l, r = l mod K, K = max_entries, W = value_size/8 (a power of two).
 * Lanes are innermost and the key index is rotated by the lane, so a warp whose lane l touches
 * key l (C2's per-lane statistics) -- and any warp when K == 1 -- touches 256 contiguous bytes. */
__device__ __forceinline__ uint64_t pt_word_index(uint32_t K, uint32_t W, uint32_t k, uint32_t w, uint32_t shard) {
    const uint32_t q = shard >> 5, l = shard & 31;
    const uint32_t r = l < K ? l : l % K;
    const uint32_t kk = k >= r ? k - r : k + K - r;
    return ((uint64_t)q * K * W + (uint64_t)kk * W + w) * 32 + l;
}
__device__ __forceinline__ uint8_t *pt_phys(const GxMapDesc &m, uint64_t logical, uint32_t shard) {
    const uint64_t lo = logical - m.data;
    const uint32_t W = m.value_size >> 3, sh = __popc(W - 1);
    const uint32_t wi = (uint32_t)(lo >> 3);
    const uint64_t idx = pt_word_index(m.max_entries, W, wi >> sh, wi & (W - 1), shard);
    return reinterpret_cast<uint8_t *>(m.data) + idx * 8 + (lo & 7);
}

}  // namespace gxd
