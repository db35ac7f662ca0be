"""f4 inputs: the vector-add kernel the paper instruments for its hook-overhead
microbenchmark as CUDA C++ source for gx_instrument, and the policy it
calls.  INPUT description only (no method arithmetic)."""

# hooks on both loads of c[i] = a[i] + b[i]; the group is the ballot of the bounds test, taken
# while the warp is converged.  GX_HOOKS 0 compiles the same kernel without hooks (the baseline).
VADD = r"""
#ifndef GX_HOOKS
#define GX_HOOKS 1
#endif
extern "C" __global__ void vadd(const float *a, const float *b, float *c, unsigned long long *r,
                                unsigned long long n) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    const bool in = i < n;
#if GX_HOOKS
    const unsigned g = __ballot_sync(0xFFFFFFFFu, in);
    if (in) {
        const unsigned long long ra = gx_hook_access(g, a + i, 4, false);
        const unsigned long long rb = gx_hook_access(g, b + i, 4, false);
        if (r) { r[2 * i] = ra; r[2 * i + 1] = rb; }
    }
#endif
    if (in) c[i] = a[i] + b[i];
}
"""

# the attached policy: per-page access counter (P1's map) and R0 = (addr >> 2) & 7
PI = """
    ldxdw r6, [r1+0]          ; addr
    mov64 r2, r6
    rsh64 r2, 12
    and64 r2, 255
    stxw [r10-4], r2
    lddw r1, map:counts
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, +2
    mov64 r1, 1
    atomic_add64 [r0+0], r1
    mov64 r0, r6
    rsh64 r0, 2
    and64 r0, 7
    exit
"""
