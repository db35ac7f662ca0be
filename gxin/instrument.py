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

# P7: GPU L2 stride prefetch (Table 1 "GPU L2 Stride Prefetch ... Device"): on an access
# at addr whose bits under cfg.mask are zero (the first access of each mask+1-byte chunk; mask 0 =
# every access), prefetch [addr + dist, addr + dist + len) into L2 (gdev_prefetch_l2, helper 1001);
# dist / len / mask from cfg (the host side of the policy sets the stride distance).  R0 = the
# helper's result (0 when not triggered); outcome[0 | 1 | 2 | 3] counts issued / -EINVAL / -EFAULT /
# not triggered
P7_L2_STRIDE = """
    ldxdw r6, [r1+0]          ; addr
    stw [r10-4], 0
    lddw r1, map:cfg
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, out
    ldxdw r7, [r0+0]          ; dist
    ldxdw r3, [r0+8]          ; len
    ldxdw r8, [r0+16]         ; trigger mask
    mov64 r9, 0
    mov64 r2, 3
    mov64 r4, r6
    and64 r4, r8
    jne r4, 0, count          ; not the first access of its chunk
    mov64 r2, r6
    add64 r2, r7
    lddw r1, map:region
    call 1001
    mov64 r9, r0
    mov64 r2, 0
    jeq r9, 0, count
    mov64 r2, 1
    jeq r9, -22, count
    mov64 r2, 2
count:
    stxw [r10-8], r2
    lddw r1, map:outcome
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, +2
    mov64 r1, 1
    atomic_add64 [r0+0], r1
    mov64 r0, r9
    exit
out:
    mov64 r0, 0
    exit
"""


def setup_l2(engine, region_fd, dist, length, mask=0):
    """Maps of P7 on `engine` (oracle or runtime) around an existing region map: cfg {dist, len,
    mask}, outcome[4].  Returns the asm symbol table."""
    ARRAY = 2
    cfg = engine.create_map(ARRAY, 4, 24, 1)
    engine.update_map(cfg, (0).to_bytes(4, "little"), b"".join(int(x).to_bytes(8, "little") for x in (dist, length, mask)))
    return {"region": region_fd, "cfg": cfg, "outcome": engine.create_map(ARRAY, 4, 8, 4)}
