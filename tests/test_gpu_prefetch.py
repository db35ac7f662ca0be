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
