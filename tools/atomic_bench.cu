// atomic_bench.cu -- L2 atomic throughput on B200 (the R_atom denominator of SURVEY.md §8d).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomic_bench tools/atomic_bench.cu
//   ./atomic_bench > profiles/atomics_b200.json
// Every thread issues ITERS atomics; addresses are SplitMix64-random 8-B slots of a buffer sized
// like C3's hash table (32 MiB), or one address (contention), or per-warp-uniform.  Reports
// atomics/s for: returning atom.add.u64 (random), red.add.u64 (random), atom.cas.b64 (random),
// atom.cas.b128 (random 16-B slots), red.add.u64 warp-uniform address, atom.add.u64 same address.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    return x;
}

template <int MODE>
__global__ void kern(unsigned long long *buf, uint64_t mask, int iters, unsigned long long *sink) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    unsigned long long acc = 0;
    for (int i = 0; i < iters; i++) {
        uint64_t r = mix64(t * 0x9E3779B97F4A7C15ull + i);
        if (MODE == 0) acc += atomicAdd(&buf[r & mask], 1ull);                 // returning, random
        if (MODE == 1) atomicAdd(&buf[r & mask], 1ull);                        // RED, random
        if (MODE == 2) acc += atomicCAS(&buf[r & mask], acc, acc + 1);         // CAS64, random
        if (MODE == 3) {                                                        // CAS128, random 16-B slots
            uint64_t *a = reinterpret_cast<uint64_t *>(&buf[(r & mask) & ~1ull]);
            uint64_t ol, oh;
            asm volatile("{\n\t.reg .b128 d, b, c;\n\tmov.b128 b, {%2, %3};\n\tmov.b128 c, {%4, %5};\n\t"
                         "atom.global.cas.b128 d, [%6], b, c;\n\tmov.b128 {%0, %1}, d;\n\t}"
                         : "=l"(ol), "=l"(oh) : "l"(acc), "l"(0ull), "l"(acc + 1), "l"(0ull), "l"(a) : "memory");
            acc += ol;
        }
        if (MODE == 4) {                                                        // warp-uniform address
            uint64_t w = mix64((t >> 5) * 0x9E3779B97F4A7C15ull + i);
            atomicAdd(&buf[w & mask], 1ull);
        }
        if (MODE == 5) acc += atomicAdd(&buf[0], 1ull);                         // one address
        if (MODE == 6 && (threadIdx.x & 31) == 0) acc += atomicAdd(&buf[0], 32ull); // one address, one returning op per warp
        if (MODE == 7 && (threadIdx.x & 31) == 0) atomicAdd(&buf[0], 32ull);        // one address, one RED per warp
        if (MODE == 8) {                                                        // dependent chain: one returning
            uint64_t d = mix64(t * 0x9E3779B97F4A7C15ull + i + (acc >> 62));    // atomic in flight per thread
            acc += atomicAdd(&buf[d & mask], 1ull);                             // (C3's per-record pattern)
        }
        if (MODE == 9) {                                                        // two dependent chains per thread
            uint64_t d = mix64(t * 0x9E3779B97F4A7C15ull + i + (acc >> 62));
            uint64_t e = mix64(d);
            acc += atomicAdd(&buf[d & mask], 1ull) + atomicAdd(&buf[e & mask], 1ull);
        }
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

template <int MODE>
double run(unsigned long long *buf, uint64_t mask, unsigned long long *sink, int blocks, int iters) {
    kern<MODE><<<blocks, 256>>>(buf, mask, iters, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(a);
        kern<MODE><<<blocks, 256>>>(buf, mask, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return (double)blocks * 256 * iters / (best / 1e3);
}

int main() {
    const uint64_t words = (32ull << 20) / 8;
    unsigned long long *buf, *sink;
    cudaMalloc(&buf, words * 8);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 0, words * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, iters = 256;
    double r0 = run<0>(buf, words - 1, sink, blocks, iters);
    double r1 = run<1>(buf, words - 1, sink, blocks, iters);
    double r2 = run<2>(buf, words - 1, sink, blocks, iters);
    double r3 = run<3>(buf, words - 1, sink, blocks, iters);
    double r4 = run<4>(buf, words - 1, sink, blocks, iters);
    double r5 = run<5>(buf, words - 1, sink, sms, 16);
    double r6 = run<6>(buf, words - 1, sink, sms * 8, 16) / 32;   /* warp-level ops */
    double r7 = run<7>(buf, words - 1, sink, sms * 8, 16) / 32;
    double r8a = run<8>(buf, words - 1, sink, sms * 4, 64), r8b = run<8>(buf, words - 1, sink, sms * 8, 64);
    double r9a = run<9>(buf, words - 1, sink, sms * 4, 32) * 2, r9b = run<9>(buf, words - 1, sink, sms * 8, 32) * 2;
    fprintf(stderr, "{\"dependent_chain_1024thr_per_s\": %.4g, \"dependent_chain_2048thr_per_s\": %.4g, "
            "\"two_chains_1024thr_per_s\": %.4g, \"two_chains_2048thr_per_s\": %.4g}\n", r8a, r8b, r9a, r9b);
    printf("{\"device\": \"B200\", \"buffer_bytes\": %llu, \"atom_add_u64_random_per_s\": %.4g, "
           "\"red_add_u64_random_per_s\": %.4g, \"atom_cas_b64_random_per_s\": %.4g, "
           "\"atom_cas_b128_random_per_s\": %.4g, \"red_add_u64_warp_uniform_per_s\": %.4g, "
           "\"atom_add_u64_same_address_per_s\": %.4g, \"atom_add_u64_same_address_warp_ops_per_s\": %.4g, "
           "\"red_add_u64_same_address_warp_ops_per_s\": %.4g}\n",
           (unsigned long long)(words * 8), r0, r1, r2, r3, r4, r5, r6, r7);
    return cudaGetLastError() != cudaSuccess;
}
