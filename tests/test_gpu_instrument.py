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
