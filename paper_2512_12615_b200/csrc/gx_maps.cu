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

/* the same fold as a streaming pass: the shard blocks (K*W*32 contiguous words per 32 shards) are
 * read coalesced by the whole grid, each block accumulates the K*W canonical words in shared
 * memory (un-rotating the lane-rotated key index) and adds them to `out` (zeroed first) once */
__global__ void pt_fold_stream_kernel(const uint64_t *__restrict__ data, uint32_t nshards, uint32_t K, uint32_t W,
                                      unsigned long long *__restrict__ out) {
    extern __shared__ unsigned long long acc[];
    const uint32_t KW = K * W;
    for (uint32_t j = threadIdx.x; j < KW; j += blockDim.x) acc[j] = 0;
    __syncthreads();
    const uint64_t total = (uint64_t)nshards * KW;   /* = (nshards / 32) * KW * 32 */
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += gridDim.x * (uint64_t)blockDim.x) {
        const uint32_t l = (uint32_t)(i & 31);
        const uint32_t wq = (uint32_t)((i >> 5) % KW);   /* kk * W + w within the 32-shard block */
        const uint32_t kk = wq / W, w = wq % W;
        const uint32_t r = l % K;
        const uint32_t k = kk + r >= K ? kk + r - K : kk + r;
        const uint64_t v = data[i];
        if (v) atomicAdd(&acc[k * W + w], (unsigned long long)v);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < KW; j += blockDim.x)
        if (acc[j]) atomicAdd(&out[j], acc[j]);
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
 * right after its kernel and writes into a pinned, device-mapped host slot.  blockIdx.y = item: a
 * prefetch queue (u64 count, then count x 16-B requests) or an ARRAY-shaped snapshot (an ARRAY,
 * or a per-thread map already SUM-folded into a device staging copy by gx_k_pt_fold); the blocks
 * of x stride over the item.  publish_reset_kernel (stream-ordered after it) empties the queues
 * and their request filters. */
__global__ void publish_kernel(const GxPublishItem *__restrict__ items, uint8_t *__restrict__ host) {
    const GxPublishItem it = items[blockIdx.y];
    uint64_t *out = reinterpret_cast<uint64_t *>(host + it.host_off);
    const uint64_t *src = reinterpret_cast<const uint64_t *>(it.data);
    const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, step = gridDim.x * (uint64_t)blockDim.x;
    if (it.kind == 0) {
        const uint64_t n = min((uint64_t)*reinterpret_cast<const unsigned long long *>(it.aux), it.cap);
        for (uint64_t i = t0; i < 2 * n; i += step) out[1 + i] = src[i];
        if (t0 == 0) out[0] = n;
    } else {
        for (uint64_t i = t0; i < (uint64_t)it.K * it.W; i += step) out[i] = src[i];
    }
}
__global__ void publish_reset_kernel(const GxPublishItem *__restrict__ items) {
    const GxPublishItem it = items[blockIdx.y];
    if (it.kind != 0) return;
    uint64_t *filt = reinterpret_cast<uint64_t *>(it.data) + 2 * it.cap;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < it.nshards; i += gridDim.x * (uint64_t)blockDim.x)
        filt[i] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<unsigned long long *>(it.aux) = 0;
}

__global__ void hash_init_kernel(uint64_t *data, uint64_t cap) {
    /* key words EMPTY, the two side-slot presence states 0, value words 0 (gx_device.cuh layout) */
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 2;
         i += gridDim.x * (uint64_t)blockDim.x) {
        data[i] = i < cap ? GX_HASH_EMPTY : 0;
        data[cap + 2 + i] = 0;
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
    const uint64_t cap = (uint64_t)m.cap_mask + 1;
    k = gxd::hash_keys(m)[i];
    const uint64_t v = gxd::hash_vals(m)[i];
    if (i < cap) {
        if (k >= gxd::GX_HASH_BUSY) return false;
    } else {
        if (k != 1) return false;
        k = i == cap ? GX_HASH_EMPTY : gxd::GX_HASH_BUSY; /* side slots */
    }
    const uint64_t *bv = gxd::hash_find(base, k);
    d = v - (bv ? *bv : 0);
    return !(bv && d == 0);
}
__global__ void hash_export_kernel(GxMapDesc m, GxMapDesc base, uint32_t nranks, int32_t owner, int pass,
                                   unsigned long long *counts, unsigned long long *offsets, uint64_t *keys,
                                   uint64_t *deltas, uint64_t cap_out) {
    const uint64_t cap = (uint64_t)m.cap_mask + 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap + 2;
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

/* %nsmid: one more than the largest %smid the device can report (PTX: SM ids need not be
 * contiguous) -- sizes the per-thread shards the f4 hooks key by (SM, warp slot, lane) */
__global__ void nsmid_kernel(uint32_t *out) {
    uint32_t v;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(v));
    *out = v;
}

extern "C" {

int gx_k_pt_fold(const uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, uint64_t *out, cudaStream_t s) {
    if (nshards % 32 == 0 && (uint64_t)K * W * 8 <= 48 * 1024) {
        cudaError_t e = cudaMemsetAsync(out, 0, 8ull * K * W, s);
        if (e) return (int)e;
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        pt_fold_stream_kernel<<<nsm * 4, 512, 8ull * K * W, s>>>(data, nshards, K, W, (unsigned long long *)out);
    } else {
        pt_fold_kernel<<<grid_for((uint64_t)K * W * 32, 256), 256, 0, s>>>(data, nshards, K, W, out);
    }
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
    publish_kernel<<<dim3(148, n_items), 256, 0, s>>>(items, host_slot);
    publish_reset_kernel<<<dim3(64, n_items), 256, 0, s>>>(items);
    return (int)cudaGetLastError();
}

int gx_k_hash_init(uint64_t *slots, uint64_t cap, cudaStream_t s) {
    hash_init_kernel<<<grid_for(cap + 2, 256), 256, 0, s>>>(slots, cap);
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
    hash_export_kernel<<<grid_for((uint64_t)m->cap_mask + 3, 256), 256, 0, s>>>(*m, *base, nranks, owner, pass, counts,
                                                                               offsets, keys, deltas, cap_out);
    return (int)cudaGetLastError();
}
int gx_k_hash_accumulate(const GxMapDesc *m, const uint64_t *keys, const uint64_t *deltas, uint64_t n,
                         unsigned long long *full, cudaStream_t s) {
    hash_accumulate_kernel<<<grid_for(n, 256), 256, 0, s>>>(*m, keys, deltas, n, full);
    return (int)cudaGetLastError();
}

int gx_k_nsmid(uint32_t *out_host) {
    uint32_t *d = nullptr;
    cudaError_t e = cudaMalloc(&d, 4);
    if (e) return (int)e;
    nsmid_kernel<<<1, 1>>>(d);
    e = cudaMemcpy(out_host, d, 4, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (int)e;
}

}  // extern "C"
