/*
 * gen_cuda.cu -- device implementation of the gxin event generator (gxin/gen.py).
 *
 * INPUT GENERATION ONLY (task rule ③: the seeded input generators are the one module both the
 * CUDA path and the oracle may use; this file holds none of the method's arithmetic).  Every
 * field is the same pure function of (seed, config, i, n_total) as gen.py; the threshold tables
 * (quantised CDFs) and the C4 bounds are data computed by gen.py and passed in.
 * A GPU test checks this generator byte for byte against gen.py.
 */
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint64_t C_STREAM = 0xD1B54A32D192ED03ull;
constexpr uint64_t C_GOLD = 0x9E3779B97F4A7C15ull;
constexpr uint64_t NPAGES = 1ull << 20;
constexpr uint64_t NWEIGHT = 24ull * 32768;
constexpr uint64_t PERM_A = 500009, PERM_B = 12345;
constexpr uint64_t NLISTS = 4096;
constexpr uint64_t QUERY_RECS = 64 + 16 * 32;

struct Tables {
    const uint64_t *sm;        /* 148 */
    const uint64_t *zipf_w;    /* NWEIGHT, theta 0.99 */
    const uint64_t *zipf_l;    /* NLISTS, theta 0.8 */
    const uint64_t *tenant;    /* 4 */
    const uint64_t *bounds;    /* NLISTS + 1 */
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}
__device__ __forceinline__ uint64_t rnd(uint64_t seed, uint64_t stream, uint64_t j) {
    return mix64((seed ^ (stream * C_STREAM)) + j * C_GOLD);
}
/* #{k : t_k <= u}, clamped to K-1 (numpy searchsorted side='right') */
__device__ __forceinline__ uint64_t draw(const uint64_t *t, uint64_t K, uint64_t u) {
    uint64_t lo = 0, hi = K;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (t[mid] <= u) lo = mid + 1;
        else hi = mid;
    }
    return lo < K ? lo : K - 1;
}

struct F {
    uint64_t addr, size, kind, block_id, sm_id, warp_id;
};

__device__ __forceinline__ void common(uint64_t seed, uint64_t rec, F &f) {
    f.block_id = rnd(seed, 2, rec) % 65536;
    f.sm_id = rnd(seed, 3, rec) % 148;
    f.warp_id = rnd(seed, 4, rec) % 64;
}

__device__ F c1(uint64_t seed, uint64_t i, uint64_t rec, uint64_t lane, uint64_t, const Tables &) {
    F f;
    common(seed, rec, f);
    f.addr = (rnd(seed, 1, i) & 0xFFFFFFFFull) & ~7ull;
    f.size = 8;
    f.kind = 0;
    return f;
}
__device__ F c2(uint64_t seed, uint64_t i, uint64_t rec, uint64_t lane, uint64_t, const Tables &T) {
    F f;
    f.sm_id = draw(T.sm, 148, rnd(seed, 3, rec));
    uint64_t w = rnd(seed, 4, rec);
    f.warp_id = f.sm_id == 0 ? 32 + w % 32 : w % 64;
    f.block_id = rnd(seed, 2, rec) % 65536;
    uint64_t base = (rnd(seed, 5, rec) & 0xFFFFFFFFFFull) & ~0x1FFull;
    f.addr = base + 16 * lane;
    f.size = 1ull << (rnd(seed, 7, rec) % 5);
    f.kind = 0;
    return f;
}
__device__ F c3(uint64_t seed, uint64_t i, uint64_t rec, uint64_t lane, uint64_t n_total, const Tables &T) {
    F f;
    common(seed, rec, f);
    const uint64_t prefill = (n_total >> 5) / 4;
    f.kind = 0;
    if (rec < prefill) {
        f.addr = (rec % NWEIGHT) * 4096 + lane * 128;
        f.size = 128;
        return f;
    }
    const uint64_t r2 = rec - prefill;
    uint64_t page;
    if (rnd(seed, 6, i) % 5 < 4) {
        uint64_t z = draw(T.zipf_w, NWEIGHT, rnd(seed, 8, i));
        page = (z * PERM_A + PERM_B) % NWEIGHT;
    } else {
        const uint64_t nkv = NPAGES - NWEIGHT;
        uint64_t a = (r2 >> 3) % nkv, back = rnd(seed, 9, i) % 16;
        page = NWEIGHT + (a + nkv - back) % nkv;
    }
    f.addr = page * 4096 + (rnd(seed, 1, i) & 0xFF8ull);
    f.size = 8;
    return f;
}
__device__ F c4(uint64_t seed, uint64_t i, uint64_t rec, uint64_t lane, uint64_t n_total, const Tables &T) {
    F f;
    common(seed, rec, f);
    f.kind = 0;
    f.size = 16;
    const uint64_t b0 = T.bounds[0], bend = T.bounds[NLISTS];
    const uint64_t build = (n_total >> 5) * 3 / 10;
    if (rec < build) {
        f.addr = b0 + (rec * 512) % (bend - b0) + lane * 16;
        return f;
    }
    const uint64_t q = rec - build, query = q / QUERY_RECS, k = q % QUERY_RECS;
    if (k < 64) {
        f.addr = (rnd(seed, 13, rec) % NLISTS) * 512 + lane * 16;
        return f;
    }
    const uint64_t kk = k - 64, j = kk / 32, s = kk % 32;
    const uint64_t lst = draw(T.zipf_l, NLISTS, rnd(seed, 12, query * 16 + j));
    uint64_t a = T.bounds[lst] + s * 512 + lane * 16;
    f.addr = a < bend - 16 ? a : bend - 16;
    return f;
}

__global__ void gen_kernel(int config, uint64_t seed, uint64_t i0, uint64_t n, uint64_t n_total, Tables T,
                           uint4 *__restrict__ out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += gridDim.x * (uint64_t)blockDim.x) {
        const uint64_t i = i0 + t, rec = i >> 5, lane = i & 31;
        F f;
        uint64_t hook;
        if (config == 5) {
            const uint64_t tenant = draw(T.tenant, 4, rnd(seed, 10, rec));
            switch (tenant) {
            case 0: f = c1(seed, i, rec, lane, n_total, T); break;
            case 1: f = c2(seed, i, rec, lane, n_total, T); break;
            case 2: f = c3(seed, i, rec, lane, n_total, T); break;
            default: f = c4(seed, i, rec, lane, n_total, T); break;
            }
            const bool fault = tenant == 2 && rnd(seed, 11, rec) % 10 == 0;
            f.kind = fault ? 2 : 0;
            if (fault) f.size = 4096;
            hook = f.kind | (tenant << 8);
        } else {
            switch (config) {
            case 1: f = c1(seed, i, rec, lane, n_total, T); break;
            case 2: f = c2(seed, i, rec, lane, n_total, T); break;
            case 3: f = c3(seed, i, rec, lane, n_total, T); break;
            default: f = c4(seed, i, rec, lane, n_total, T); break;
            }
            hook = f.kind;
        }
        const uint64_t ts = rec * 1000;
        uint4 a, b;
        a.x = (uint32_t)f.addr;
        a.y = (uint32_t)(f.addr >> 32);
        a.z = (uint32_t)ts;
        a.w = (uint32_t)(ts >> 32);
        b.x = (uint32_t)hook;
        b.y = (uint32_t)f.block_id;
        b.z = (uint32_t)(f.sm_id & 0xFFFF) | ((uint32_t)(f.warp_id & 0xFF) << 16) | ((uint32_t)lane << 24);
        b.w = (uint32_t)f.size;
        out[2 * t] = a;
        out[2 * t + 1] = b;
    }
}

}  // namespace

extern "C" int gxgen_generate(int config, uint64_t seed, uint64_t i0, uint64_t n, uint64_t n_total,
                              const uint64_t *sm, const uint64_t *zipf_w, const uint64_t *zipf_l,
                              const uint64_t *tenant, const uint64_t *bounds, void *out, void *stream) {
    Tables T{sm, zipf_w, zipf_l, tenant, bounds};
    if (n == 0) return 0;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    gen_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(config, seed, i0, n, n_total, T,
                                                                    reinterpret_cast<uint4 *>(out));
    return (int)cudaGetLastError();
}
