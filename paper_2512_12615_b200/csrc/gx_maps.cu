/*
 * gx_maps.cu -- map maintenance kernels: per-thread fold, host control-plane writes, hash
 * initialisation, and the snapshot-and-merge delta/apply kernels.
 * Not on the per-event hot path; each is a simple grid-stride kernel.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "gx_device.cuh"
#include "gx_internal.h"

namespace {

/* canonical per-thread value = SUM over shards of each u64 word (S4); one warp per canonical word,
 * coalesced over the lane-innermost layout (gxd::pt_word_index) */
__global__ void pt_fold_kernel(const uint64_t *__restrict__ data, uint32_t nshards, uint32_t K, uint32_t W,
                               uint64_t *__restrict__ out) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    for (uint64_t j = warp; j < (uint64_t)K * W; j += nw) {
        const uint32_t k = (uint32_t)(j / W), w = (uint32_t)(j % W);
        uint64_t s = 0;
        for (uint32_t sh = lane; sh < nshards; sh += 32) s += data[gxd::pt_word_index(K, W, k, w, sh)];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(GX_FULL, s, o);
        if (lane == 0) out[j] = s;
    }
}

/* host write of key k: shard 0 = value, every other shard's copy of key k = 0 */
__global__ void pt_set_kernel(uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, uint32_t k, const uint64_t *vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)W * nshards;
         i += gridDim.x * (uint64_t)blockDim.x) {
        const uint32_t w = (uint32_t)(i / nshards), s = (uint32_t)(i % nshards);
        data[gxd::pt_word_index(K, W, k, w, s)] = s == 0 ? vals[w] : 0;
    }
}

/* canonical content -> shard 0, zero the rest (after a merge) */
__global__ void pt_store_canonical_kernel(uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, const uint64_t *vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)K * W * nshards;
         i += gridDim.x * (uint64_t)blockDim.x) {
        const uint64_t j = i / nshards;
        const uint32_t s = (uint32_t)(i % nshards);
        data[gxd::pt_word_index(K, W, (uint32_t)(j / W), (uint32_t)(j % W), s)] = s == 0 ? vals[j] : 0;
    }
}

/* Runtime-daemon publish point (include/gx.h): runs on the batch's stream
 * right after its kernel and writes into a pinned, device-mapped host slot -- block b handles
 * item b: a prefetch queue (u64 count, then count x 16-B requests; the queue is emptied) or a
 * watched map's canonical snapshot (ARRAY copy, PERTHREAD SUM fold). */
__global__ void publish_kernel(const GxPublishItem *__restrict__ items, uint8_t *__restrict__ host) {
    const GxPublishItem it = items[blockIdx.x];
    uint64_t *out = reinterpret_cast<uint64_t *>(host + it.host_off);
    if (it.kind == 0) { /* prefetch queue */
        unsigned long long *ctr = reinterpret_cast<unsigned long long *>(it.aux);
        const uint64_t n = min((uint64_t)*ctr, it.cap);
        const uint64_t *src = reinterpret_cast<const uint64_t *>(it.data);
        for (uint64_t i = threadIdx.x; i < 2 * n; i += blockDim.x) out[1 + i] = src[i];
        __syncthreads();
        if (threadIdx.x == 0) {
            out[0] = n;
            *ctr = 0;
        }
    } else if (it.kind == 1) { /* ARRAY */
        const uint64_t *src = reinterpret_cast<const uint64_t *>(it.data);
        for (uint64_t i = threadIdx.x; i < (uint64_t)it.K * it.W; i += blockDim.x) out[i] = src[i];
    } else { /* PERTHREAD: canonical value = SUM over shards (S4) */
        const uint64_t *src = reinterpret_cast<const uint64_t *>(it.data);
        const uint32_t lane = threadIdx.x & 31;
        for (uint64_t j = threadIdx.x >> 5; j < (uint64_t)it.K * it.W; j += blockDim.x >> 5) {
            const uint32_t k = (uint32_t)(j / it.W), w = (uint32_t)(j % it.W);
            uint64_t acc = 0;
            for (uint32_t sh = lane; sh < it.nshards; sh += 32) acc += src[gxd::pt_word_index(it.K, it.W, k, w, sh)];
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(GX_FULL, acc, o);
            if (lane == 0) out[j] = acc;
        }
    }
}

__global__ void hash_init_kernel(uint64_t *slots, uint64_t cap) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 1;
         i += gridDim.x * (uint64_t)blockDim.x) {
        slots[2 * i] = i < cap ? GX_HASH_EMPTY : 0; /* side slot: present flag 0 */
        slots[2 * i + 1] = 0;
    }
}

/* host control-plane updates, applied in order by one thread (bpf semantics per call) */
__global__ void hash_host_update_kernel(GxMapDesc m, const uint64_t *keys, const uint64_t *vals, uint64_t n,
                                        uint64_t flags, int64_t *rc, unsigned long long *full) {
    if (blockIdx.x || threadIdx.x) return;
    for (uint64_t i = 0; i < n; i++) {
        bool f;
        rc[i] = gxd::hash_update(m, keys[i], vals[i], flags, f);
        if (f) atomicAdd(full, 1ull);
    }
}

__global__ void sub_kernel(const uint64_t *a, const uint64_t *b, uint64_t *out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x)
        out[i] = a[i] - b[i];
}
__global__ void add_kernel(const uint64_t *a, const uint64_t *b, uint64_t *out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x)
        out[i] = a[i] + b[i];
}

/* hash delta export: entries whose value differs from the base copy (or are new), bucketed by
 * owner = mix64(key) mod nranks.  Pass 0 counts per owner, pass 1 scatters at per-owner offsets. */
__device__ __forceinline__ bool export_entry(const GxMapDesc &m, const GxMapDesc &base, uint64_t i, uint64_t &k,
                                             uint64_t &d) {
    const uint64_t *slots = reinterpret_cast<const uint64_t *>(m.data);
    const uint64_t cap = (uint64_t)m.cap_mask + 1;
    k = slots[2 * i];
    const uint64_t v = slots[2 * i + 1];
    if (i < cap) {
        if (k == GX_HASH_EMPTY) return false;
    } else {
        if (k != 1) return false;
        k = GX_HASH_EMPTY;
    }
    const uint64_t *bv = gxd::hash_find(base, k);
    d = v - (bv ? *bv : 0);
    return !(bv && d == 0);
}
__global__ void hash_export_kernel(GxMapDesc m, GxMapDesc base, uint32_t nranks, int32_t owner, int pass,
                                   unsigned long long *counts, unsigned long long *offsets, uint64_t *keys,
                                   uint64_t *deltas, uint64_t cap_out) {
    const uint64_t cap = (uint64_t)m.cap_mask + 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 1;
         i += gridDim.x * (uint64_t)blockDim.x) {
        uint64_t k, d;
        if (!export_entry(m, base, i, k, d)) continue;
        const uint32_t g = (uint32_t)(gxd::mix64(k) % nranks);
        if (owner >= 0 && g != (uint32_t)owner) continue;
        if (pass == 0) {
            atomicAdd(&counts[g], 1ull);
        } else {
            const unsigned long long o = atomicAdd(&offsets[g], 1ull);
            if (o < cap_out) {
                keys[o] = k;
                deltas[o] = d;
            }
        }
    }
}

/* hash merge accumulate: value += delta, inserting absent keys at 0 */
__global__ void hash_accumulate_kernel(GxMapDesc m, const uint64_t *keys, const uint64_t *deltas, uint64_t n,
                                       unsigned long long *full) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x) {
        uint64_t *v = gxd::hash_find(m, keys[i]);
        if (!v) {
            bool f;
            gxd::hash_update(m, keys[i], 0, 1 /* NOEXIST */, f);
            if (f) {
                atomicAdd(full, 1ull);
                continue;
            }
            v = gxd::hash_find(m, keys[i]);
        }
        if (v) atomicAdd(reinterpret_cast<unsigned long long *>(v), (unsigned long long)deltas[i]);
    }
}

inline uint32_t grid_for(uint64_t n, uint32_t block) {
    uint64_t g = (n + block - 1) / block;
    if (g > 148 * 8) g = 148 * 8;
    return g ? (uint32_t)g : 1;
}

}  // namespace

extern "C" {

int gx_k_pt_fold(const uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, uint64_t *out, cudaStream_t s) {
    pt_fold_kernel<<<grid_for((uint64_t)K * W * 32, 256), 256, 0, s>>>(data, nshards, K, W, out);
    return (int)cudaGetLastError();
}
int gx_k_pt_set(uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, uint32_t k, const uint64_t *vals,
                cudaStream_t s) {
    pt_set_kernel<<<grid_for((uint64_t)W * nshards, 256), 256, 0, s>>>(data, nshards, K, W, k, vals);
    return (int)cudaGetLastError();
}
int gx_k_pt_store_canonical(uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, const uint64_t *vals,
                            cudaStream_t s) {
    pt_store_canonical_kernel<<<grid_for((uint64_t)K * W * nshards, 256), 256, 0, s>>>(data, nshards, K, W, vals);
    return (int)cudaGetLastError();
}
int gx_k_publish(const GxPublishItem *items, uint32_t n_items, uint8_t *host_slot, cudaStream_t s) {
    if (!n_items) return 0;
    publish_kernel<<<n_items, 256, 0, s>>>(items, host_slot);
    return (int)cudaGetLastError();
}

int gx_k_hash_init(uint64_t *slots, uint64_t cap, cudaStream_t s) {
    hash_init_kernel<<<grid_for(cap + 1, 256), 256, 0, s>>>(slots, cap);
    return (int)cudaGetLastError();
}
int gx_k_hash_host_update(const GxMapDesc *m, const uint64_t *keys, const uint64_t *vals, uint64_t n, uint64_t flags,
                          int64_t *rc, unsigned long long *full, cudaStream_t s) {
    hash_host_update_kernel<<<1, 1, 0, s>>>(*m, keys, vals, n, flags, rc, full);
    return (int)cudaGetLastError();
}
int gx_k_sub(const uint64_t *a, const uint64_t *b, uint64_t *out, uint64_t n, cudaStream_t s) {
    sub_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, b, out, n);
    return (int)cudaGetLastError();
}
int gx_k_add(const uint64_t *a, const uint64_t *b, uint64_t *out, uint64_t n, cudaStream_t s) {
    add_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, b, out, n);
    return (int)cudaGetLastError();
}
int gx_k_hash_export(const GxMapDesc *m, const GxMapDesc *base, uint32_t nranks, int32_t owner, int pass,
                     unsigned long long *counts, unsigned long long *offsets, uint64_t *keys, uint64_t *deltas,
                     uint64_t cap_out, cudaStream_t s) {
    hash_export_kernel<<<grid_for((uint64_t)m->cap_mask + 2, 256), 256, 0, s>>>(*m, *base, nranks, owner, pass, counts,
                                                                               offsets, keys, deltas, cap_out);
    return (int)cudaGetLastError();
}
int gx_k_hash_accumulate(const GxMapDesc *m, const uint64_t *keys, const uint64_t *deltas, uint64_t n,
                         unsigned long long *full, cudaStream_t s) {
    hash_accumulate_kernel<<<grid_for(n, 256), 256, 0, s>>>(*m, keys, deltas, n, full);
    return (int)cudaGetLastError();
}

}  // extern "C"
