"""GPU parity for the f4 row: a policy JIT-compiled as inline hooks into a user
vector-add kernel (gx_instrument) gives the oracle's map contents and per-event R0 over the same
access events (the hooks' addresses a + 4i, b + 4i)."""
import numpy as np
import pytest

from gxin import asm, gen, instrument
from oracle.oracle import ARRAY, Oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 31, 1000, (1 << 16) + 17])
def test_instrumented_vadd_parity(gpu, n):
    import torch
    import paper_2512_12615_b200 as gx
    rt = gx.Runtime(0)
    counts = rt.create_map(ARRAY, 4, 8, 256)
    prog = rt.load_prog(asm.assemble(instrument.PI, {"counts": counts}))
    k = gx.gx_instrument(rt.rt, prog, instrument.VADD)
    a = torch.randn(n, device="cuda")
    b = torch.randn(n, device="cuda")
    c = torch.empty(n, device="cuda")
    r = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
    gx.gx_kernel_launch(rt.rt, k, "vadd", ((n + 255) // 256,), (256,), [a, b, c, r, n])
    torch.cuda.synchronize()
    assert torch.equal(c, a + b)
    addr = np.empty(2 * n, dtype=np.uint64)
    addr[0::2] = a.data_ptr() + 4 * np.arange(n, dtype=np.uint64)
    addr[1::2] = b.data_ptr() + 4 * np.arange(n, dtype=np.uint64)
    env = Oracle()
    oc = env.create_map(ARRAY, 4, 8, 256)
    want = env.run(gen.records(2 * n, addr=addr), env.load_prog(asm.assemble(instrument.PI, {"counts": oc})))
    assert (r.cpu().numpy().view(np.uint64) == want).all()
    assert rt.dump(counts) == env.dump(oc)
    gx.gx_kernel_free(rt.rt, k)


def test_instrument_needs_verified_program(gpu):
    import paper_2512_12615_b200 as gx
    rt = gx.Runtime(0)
    fd = gx.gx_load_prog(rt.rt, 0, asm.assemble("mov64 r0, 0\nexit"))
    with pytest.raises(gx.GxError):
        gx.gx_instrument(rt.rt, fd, instrument.VADD)


PROBE_KERNEL = r"""
extern "C" __global__ void probe_k(unsigned long long *r, unsigned n) {
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = i < n;
    const unsigned g = __ballot_sync(0xFFFFFFFFu, in);
    if (in) {
        r[4 * i] = gx_hook_probe(g, 7);                        /* device function 7 starts */
        const unsigned v = i * 3;                              /* its body */
        r[4 * i + 1] = gx_hook_retprobe(g, 7, v);              /* ... and returns v */
        r[4 * i + 2] = gx_hook_fence(g, 2);                    /* a fence point, scope 2 */
        r[4 * i + 3] = gx_hook_access(g, (const void *)(unsigned long long)(8ull * i), 8, true);
    }
}
"""

# counts the hook kinds it sees; R0 = addr + size + is_write
KINDS = """
    ldxw r6, [r1+16]
    ldxdw r7, [r1+0]
    ldxw r8, [r1+28]
    mov64 r2, r6
    and64 r2, 255
    stxw [r10-4], r2
    lddw r1, map:kc
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, +2
    mov64 r1, 1
    atomic_add64 [r0+0], r1
    mov64 r0, r7
    add64 r0, r8
    rsh64 r6, 16
    add64 r0, r6
    exit
"""


@pytest.mark.parametrize("n", [32, 1000 + 7])
def test_probe_retprobe_fence_hooks(gpu, n):
    """gdev_sched_ops.probe / .retprobe and gdev_mem_ops.fence
    hooks inlined into a user kernel: per-call R0 and the per-kind counts against the oracle over
    the same hook records (kinds 6, 7, 3, 0 with their addr / size / is_write)."""
    import torch
    import paper_2512_12615_b200 as gx
    rt = gx.Runtime(0)
    kc = rt.create_map(ARRAY, 4, 8, 8)
    k = gx.gx_instrument(rt.rt, rt.load_prog(asm.assemble(KINDS, {"kc": kc})), PROBE_KERNEL)
    r = torch.zeros(4 * n, dtype=torch.int64, device="cuda")
    gx.gx_kernel_launch(rt.rt, k, "probe_k", ((n + 127) // 128,), (128,), [r, gx_u32(n)])
    torch.cuda.synchronize()
    i = np.arange(n, dtype=np.uint64)
    addr = np.stack([np.full(n, 7, np.uint64), np.full(n, 7, np.uint64), np.full(n, 2, np.uint64), 8 * i], 1).reshape(-1)
    hook = np.stack([np.full(n, 6), np.full(n, 7), np.full(n, 3), np.full(n, 0x10000)], 1).reshape(-1).astype(np.uint32)
    size = np.stack([np.zeros(n), 3 * i, np.zeros(n), np.full(n, 8)], 1).reshape(-1).astype(np.uint32)
    env = Oracle()
    ok = env.create_map(ARRAY, 4, 8, 8)
    want = env.run(gen.records(4 * n, addr=addr, hook=hook, size=size), env.load_prog(asm.assemble(KINDS, {"kc": ok})))
    assert (r.cpu().numpy().view(np.uint64) == want).all()
    assert rt.dump(kc) == env.dump(ok)
    assert rt.array_u64(kc).tolist() == [n, 0, 0, n, 0, 0, n, n]
    gx.gx_kernel_free(rt.rt, k)


def gx_u32(v):
    import ctypes
    return ctypes.c_uint32(v)
