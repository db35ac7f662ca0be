"""GPU parity for the f2 row: gdev_mem_prefetch + prefetch queue on both engines
and both ingests, and the runtime daemon (prefetch handler + snapshot flush at kernel-completion
boundaries) against the oracle (tests/test_oracle_prefetch.py pins it)."""
import numpy as np
import pytest

from gxin import asm, configs, gen
from gpu_util import ENGINES, make_runtime, oracle_run, outputs

pytestmark = pytest.mark.gpu

CALL = """
    ldxdw r2, [r1+0]
    ldxdw r3, [r1+8]
    lddw r1, map:q
    call 1000
    exit
"""


def _dev(ev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("n", [1000, (1 << 18) + 5])
def test_c6_prefetch_policy_parity(gpu, engine, n):
    """P6 (stride prefetch policy) over the C3 page trace: request set, call counter and R0."""
    import torch
    ev = configs.events("C6", configs.SEEDS["C6"], n)
    env, so, r0o = oracle_run("C6", ev)
    rt = make_runtime(engine)
    s = configs.setup(rt, "C6")
    ret = torch.zeros(n, dtype=torch.int64, device="cuda")
    rt.run(_dev(ev), s.prog_arg, ret=ret)
    torch.cuda.synchronize()
    assert (ret.cpu().numpy().view(np.uint64) == r0o).all()
    assert outputs(rt, s) == outputs(env, so)
    assert rt.stats()["ringbuf_drops"] == 0


@pytest.mark.parametrize("engine", ENGINES)
def test_prefetch_edge_cases_parity(gpu, engine):
    """Page math and -EINVAL cases, one per lane, identical requests merged."""
    import torch
    from oracle.oracle import PREFETCH_QUEUE, Oracle
    cases = [(0x1000, 1), (0x1fff, 2), (0x200000, 2 << 20), (0x200001, 2 << 20), (0, 4096), (0x1000, 0),
             (0x1000, (2 << 20) + 1), (2**64 - 4096, 8192), (0x5000, 100), (0x5000, 100), (0x5fff, 1)] * 3
    ev = gen.records(len(cases), addr=np.array([a for a, _ in cases], dtype=np.uint64),
                     ts=np.array([l for _, l in cases], dtype=np.uint64))
    env = Oracle()
    qo = env.create_map(PREFETCH_QUEUE, 0, 0, 64)
    want = env.run(ev, env.load_prog(asm.assemble(CALL, {"q": qo})))
    rt = make_runtime(engine)
    qg = rt.create_map(PREFETCH_QUEUE, 0, 0, 64)
    ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda")
    rt.run(_dev(ev), rt.load_prog(asm.assemble(CALL, {"q": qg})), ret=ret)
    assert (ret.cpu().numpy().view(np.uint64) == want).all()
    assert rt.prefetch_requests(qg) == env.prefetch_requests(qo)


def test_prefetch_queue_capacity(gpu):
    """65 distinct requests into a 64-request queue: 64 queued, one -EAGAIN (which one is
    order-dependent), one drop counted."""
    import torch
    from oracle.oracle import PREFETCH_QUEUE
    ev = gen.records(65, addr=np.arange(65, dtype=np.uint64) * 4096, ts=np.uint64(1))
    rt = make_runtime("jit")
    q = rt.create_map(PREFETCH_QUEUE, 0, 0, 64)
    ret = torch.zeros(65, dtype=torch.int64, device="cuda")
    rt.run(_dev(ev), rt.load_prog(asm.assemble(CALL, {"q": q})), ret=ret)
    r = ret.cpu().numpy()
    assert (r == -11).sum() == 1 and (r == 0).sum() == 64
    assert rt.stats()["ringbuf_drops"] == 1
    got = rt.prefetch_requests(q)
    assert len(got) == 64 and set(got) <= {(p, 1) for p in range(65)}


@pytest.mark.parametrize("engine", ["jit", "jit_ring", "interp"])
def test_daemon_prefetch_and_snapshot(gpu, engine):
    """Runtime daemon over 4 back-to-back C6 batches: the handler receives (as a union) exactly the
    oracle's request set; the watched ARRAY's last snapshot equals the map; one publish point per
    batch; the caller's stream never waits for the host."""
    import torch
    import paper_2512_12615_b200 as gx
    n = (1 << 17) + 32
    ev = configs.events("C6", configs.SEEDS["C6"], 4 * n)
    env, so, _ = oracle_run("C6", ev)
    rt = make_runtime(engine)
    s = configs.setup(rt, "C6")
    got = []
    gx.gx_daemon_watch(rt.rt, s.fds[(0, "pstat")])
    rt.daemon_start(lambda fd, reqs: got.extend(reqs))
    d = _dev(ev)
    for k in range(4):
        rt.run(d[k * n:(k + 1) * n], s.prog_arg, overlap=(k > 0))
    torch.cuda.synchronize()
    rt.daemon_stop()
    assert sorted(set(got)) == env.prefetch_requests(so.fds[(0, "pfq")])
    snap, ver = gx.gx_snapshot_read(rt.rt, s.fds[(0, "pstat")], 8)
    assert ver == 4 and snap == rt.dump(s.fds[(0, "pstat")]) == env.dump(so.fds[(0, "pstat")])
    st = gx.gx_daemon_get_stats(rt.rt)
    assert st["batches"] == 4 and st["requests"] == len(got)


def test_daemon_perthread_snapshot(gpu):
    """C2 with the daemon watching the histogram and the per-thread map: published snapshots are
    the canonical (SUM-folded) contents at the last kernel-completion boundary."""
    import torch
    import paper_2512_12615_b200 as gx
    n = (1 << 18) + 64
    ev = configs.events("C2", configs.SEEDS["C2"], 2 * n)
    env, so, _ = oracle_run("C2", ev)
    rt = make_runtime("jit")
    s = configs.setup(rt, "C2")
    for name in ("hist", "lane_pt"):
        gx.gx_daemon_watch(rt.rt, s.fds[(0, name)])
    rt.daemon_start(None)
    d = _dev(ev)
    rt.run(d[:n], s.prog_arg)
    rt.run(d[n:], s.prog_arg)
    torch.cuda.synchronize()
    rt.daemon_stop()
    for name, nbytes in (("hist", 148 * 64 * 8), ("lane_pt", 32 * 16)):
        snap, ver = gx.gx_snapshot_read(rt.rt, s.fds[(0, name)], nbytes)
        assert ver == 2 and snap == env.dump(so.fds[(0, name)]), name


# ---- gdev_prefetch_l2 (F-7): R0 against the oracle on both engines; the
# prefetches themselves land in a real device buffer (registered as the region)
L2CALL = """
    ldxdw r2, [r1+0]
    ldxdw r3, [r1+8]
    lddw r1, map:region
    call 1001
    exit
"""


@pytest.mark.parametrize("engine", ENGINES)
def test_prefetch_l2_parity(gpu, engine):
    import torch
    from oracle.oracle import Oracle
    span = 4 << 20
    buf = torch.empty(span, dtype=torch.uint8, device="cuda")
    base = buf.data_ptr()
    n = 20000 + 13
    rng = np.random.default_rng(7)
    off = rng.integers(-(16 << 10), span + (16 << 10), n)
    lens = rng.choice(np.array([0, 1, 8, 128, 4096, 65535, 65536, 65537, 1 << 20], dtype=np.int64), n)
    ev = gen.records(n, addr=(base + off).astype(np.uint64), ts=lens.astype(np.uint64))
    env = Oracle()
    want = env.run(ev, env.load_prog(asm.assemble(L2CALL, {"region": env.region_map(base, span)})))
    rt = make_runtime(engine)
    prog = rt.load_prog(asm.assemble(L2CALL, {"region": rt.region_map(base, span)}))
    ret = torch.zeros(n, dtype=torch.int64, device="cuda")
    rt.run(_dev(ev), prog, ret=ret)
    torch.cuda.synchronize()
    got = ret.cpu().numpy().view(np.uint64)
    assert (got == want).all()
    assert {0, 2**64 - 14, 2**64 - 22} <= set(want.tolist())      # every outcome occurs
    assert rt.stats()["helper_errors"] == env.stats()["helper_errors"]


def test_region_map_has_no_content(gpu):
    import torch
    import paper_2512_12615_b200 as gx
    buf = torch.empty(4096, dtype=torch.uint8, device="cuda")
    rt = make_runtime("jit")
    reg = rt.region_map(buf.data_ptr(), 4096)
    assert rt.update_map(reg, b"\0" * 4, b"\0" * 8) == -22
    with pytest.raises(gx.GxError):
        rt.region_map(0, 16)


@pytest.mark.parametrize("n", [1000, (1 << 16) + 17])
def test_l2_stride_policy_instrumented(gpu, n):
    """P7 inlined into the vector-add (gx_instrument): both loads of c[i] = a[i] + b[i] run the L2
    stride prefetch policy; a and b share one registered buffer, so the prefetches ahead of a land
    in b and those ahead of b's end fall outside (-EFAULT).  R0 per hook and outcome[] vs the oracle."""
    import torch
    import paper_2512_12615_b200 as gx
    from gxin import instrument
    from oracle.oracle import Oracle
    buf = torch.randn(2 * n, device="cuda")
    a, b = buf[:n], buf[n:]
    c = torch.empty(n, device="cuda")
    r = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
    dist, ln = 1024, 128
    rt = gx.Runtime(0)
    fds = instrument.setup_l2(rt, rt.region_map(buf.data_ptr(), 8 * n), dist, ln)
    k = gx.gx_instrument(rt.rt, rt.load_prog(asm.assemble(instrument.P7_L2_STRIDE, fds)), instrument.VADD)
    gx.gx_kernel_launch(rt.rt, k, "vadd", ((n + 255) // 256,), (256,), [a, b, c, r, n])
    torch.cuda.synchronize()
    assert torch.equal(c, a + b)
    addr = np.empty(2 * n, dtype=np.uint64)
    addr[0::2] = a.data_ptr() + 4 * np.arange(n, dtype=np.uint64)
    addr[1::2] = b.data_ptr() + 4 * np.arange(n, dtype=np.uint64)
    env = Oracle()
    ofds = instrument.setup_l2(env, env.region_map(buf.data_ptr(), 8 * n), dist, ln)
    want = env.run(gen.records(2 * n, addr=addr), env.load_prog(asm.assemble(instrument.P7_L2_STRIDE, ofds)))
    assert (r.cpu().numpy().view(np.uint64) == want).all()
    assert rt.dump(fds["outcome"]) == env.dump(ofds["outcome"])
    gx.gx_kernel_free(rt.rt, k)
