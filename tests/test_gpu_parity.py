"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
on the same seeded events (task rule ③; SURVEY.md §8c parity matrix).  Integer work: bit-exact.
ORDER_INSENSITIVE configs only (c.3 S1): map dumps, ringbuf multisets, R0, stats."""
import numpy as np
import pytest

from gxin import asm, configs, gen
import closed_forms as cf
from gpu_util import ENGINES, first_diff, gpu_run, make_runtime, oracle_run, outputs

pytestmark = pytest.mark.gpu


def _compare(config, ev, threshold=None, check_r0=True, engine="jit"):
    env, so, r0o = oracle_run(config, ev, threshold)
    rt, sg, r0g = gpu_run(config, ev, threshold, engine=engine)
    oo, og = outputs(env, so), outputs(rt, sg)
    for key in oo:
        a, b = oo[key], og[key]
        if isinstance(a, tuple):
            assert a == b, (config, key, "ringbuf multiset differs", len(a), len(b))
        else:
            assert a == b, (config, key, "first differing byte", first_diff(a, b))
    if check_r0:
        bad = np.nonzero(r0o != r0g)[0]
        assert bad.size == 0, (config, "R0 differs at", bad[:8], r0o[bad[:8]], r0g[bad[:8]])
    so_stats, sg_stats = env.stats(), rt.stats()
    for k in ("events_run", "events_skipped", "ringbuf_drops", "hash_full"):
        assert so_stats[k] == sg_stats[k], (config, k, so_stats[k], sg_stats[k])
    return rt, sg, sg_stats


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("config,n", [("C1", 10 ** 6), ("C1", 1 << 20), ("C1d", 10 ** 6), ("C2", (1 << 18) + 13),
                                      ("C3", (1 << 18) + 5), ("C4", (1 << 18) + 31), ("C5", (1 << 18) + 1)])
def test_config_parity(gpu, config, n, engine):
    ev = configs.events(config, configs.SEEDS[config], n)
    rt, s, st = _compare(config, ev, engine=engine)
    if config == "C4" and engine == "interp":
        assert st["divergent_steps"] > 0   # straddling records exercise the min-PC path


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 65, 1000])
@pytest.mark.parametrize("config", ["C1", "C3", "C5"])
def test_ragged_tails(gpu, config, n, engine):
    ev = configs.events(config, configs.SEEDS[config], n)
    _compare(config, ev, threshold=2 if config == "C3" else None, engine=engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_c3_threshold_small(gpu, engine):
    """Threshold T=2 makes many FETCH-ADD crossings: ringbuf multiset must equal the oracle's."""
    ev = configs.events("C3", 99, 1 << 16)
    rt, s, st = _compare("C3", ev, threshold=2, engine=engine)
    assert st["ringbuf_drops"] == 0


def test_empty_batch(gpu):
    import torch
    import paper_2512_12615_b200 as gx
    rt = gx.Runtime(0)
    s = configs.setup(rt, "C1")
    rt.run(torch.empty((0, 32), dtype=torch.uint8, device="cuda"), s.prog_arg)
    assert int(rt.array_u64(s.fds[(0, "counts")]).sum()) == 0


def test_fig2_pin_gpu(gpu):
    sm = np.concatenate([np.full(382, 15), np.full(3, 6)]).astype(np.uint16)
    ev = gen.records(len(sm), sm_id=sm, warp_id=(np.arange(len(sm)) % 64).astype(np.uint8), size=4)
    rt, s, _ = gpu_run("C2", ev)
    hist = rt.array_u64(s.fds[(0, "hist")]).reshape(148, 64).sum(axis=1)
    assert int(hist[15]) == 382 and int(hist[6]) == 3


def test_device_generator(gpu):
    """The CUDA generator reproduces gxin.gen byte for byte (any shard offset)."""
    from gxin import gen_gpu
    for config in gen.CONFIGS:
        n_total = 1 << 20
        for i0, n in ((0, 4096), (1 << 19, 4099), (n_total - 777, 777)):
            want = gen.generate(config, 1234, n, i0, n_total)
            got = gen_gpu.generate_device(config, 1234, n, i0, n_total).cpu().numpy()
            assert got.tobytes() == want.tobytes(), (config, i0)


PRE = "ldxdw r0, [r1+0]\nldxdw r2, [r1+8]\n"


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("W", [64, 32])
def test_isa_parity_alu_jmp(gpu, W, engine):
    """Every ALU / JMP op over the edge grid: GPU R0 == oracle R0 (and == closed form)."""
    import itertools
    import torch
    import paper_2512_12615_b200 as gx
    from oracle.oracle import Oracle
    grid = cf.edge_grid(20)
    pairs = list(itertools.product(grid, grid))
    ev = gen.records(len(pairs), addr=np.array([p[0] for p in pairs], dtype=np.uint64),
                     ts=np.array([p[1] for p in pairs], dtype=np.uint64))
    d_ev = torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda()
    rt = make_runtime(engine)
    texts = []
    for name in cf.ALU_NAMES:
        if name == "movsx32" and W == 32:
            continue
        texts.append(f"{name}{W} r0" if name == "neg" else f"{name}{W} r0, r2")
    sfx = "32" if W == 32 else ""
    for name in cf.JMP_NAMES:
        texts.append(f"mov64 r3, r0\nmov64 r0, 0\n{name}{sfx} r3, r2, +1\nja +1\nmov64 r0, 1")
    for w in (16, 32, 64):
        texts += [f"le{w} r0", f"be{w} r0", f"bswap{w} r0"]
    for body in texts:
        prog = asm.assemble(PRE + body + "\nexit")
        env = Oracle()
        want = env.run(ev, env.load_prog(prog))
        fd = rt.load_prog(prog)
        ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda")
        rt.run(d_ev, fd, ret=ret)
        got = ret.cpu().numpy().view(np.uint64)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (body, [(hex(pairs[i][0]), hex(pairs[i][1]), hex(int(got[i])), hex(int(want[i]))) for i in bad[:4]])


@pytest.mark.parametrize("engine", ENGINES)
def test_micro_pins_gpu(gpu, engine):
    """The hand-computed micro-pins (tests/golden/micro_pins.txt) on the GPU."""
    import os
    import torch
    rt = None
    path = os.path.join(os.path.dirname(__file__), "golden", "micro_pins.txt")
    for k, line in enumerate(l for l in open(path) if l.strip() and not l.startswith("#")):
        if k % 32 == 0:   # a runtime holds at most 64 programs
            if rt is not None:
                rt.close()
            rt = make_runtime(engine)
        name, ops, d, s, want = [x.strip() for x in line.split("|")]
        ev = gen.records(32, addr=int(d, 0), ts=int(s, 0))
        fd = rt.load_prog(asm.assemble(PRE + ops.replace(" / ", "\n") + "\nexit"))
        ret = torch.zeros(32, dtype=torch.int64, device="cuda")
        rt.run(torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda(), fd, ret=ret)
        got = ret.cpu().numpy().view(np.uint64)
        assert (got == np.uint64(int(want, 0))).all(), (name, hex(int(got[0])))


def test_unverified_program_refused(gpu):
    import torch
    import paper_2512_12615_b200 as gx
    rt = gx.Runtime(0)
    fd = gx.gx_load_prog(rt.rt, 0, asm.assemble("mov64 r0, 0\nexit"))
    with pytest.raises(gx.GxError):
        rt.run(torch.zeros((32, 32), dtype=torch.uint8, device="cuda"), fd)


@pytest.mark.parametrize("engine", ENGINES)
def test_run_batch_host_parity(gpu, engine):
    """gx_run_batch_host (chunked H2D pipeline) gives the oracle's result too."""
    import paper_2512_12615_b200 as gx
    ev = configs.events("C2", 7, (1 << 18) + 3)
    env, so, r0o = oracle_run("C2", ev)
    rt = make_runtime(engine)
    s = configs.setup(rt, "C2")
    r0 = np.zeros(len(ev), dtype=np.uint64)
    gx.gx_run_batch_host(rt.rt, ev, prog_fd=s.prog_arg, ret=r0)
    assert outputs(rt, s) == outputs(env, so)
    assert (r0 == r0o).all()


# Per-thread ARRAY stress (a5): many lane-varying keys per thread (register write-back cache
# evictions in the JIT), three maps with value sizes 8 / 16 / 32, sub-word loads and stores,
# 32- and 64-bit atomics and update_elem -- all ADD-type, so the SUM fold over shards is
# shard-invariant and must equal the oracle's sequential result exactly.
PT_STRESS = """
    mov64 r6, r1
    ldxdw r7, [r6+0]          ; addr (lane-varying)
    mov64 r2, r7
    rsh64 r2, 3
    and64 r2, 7
    stxw [r10-4], r2          ; key A = (addr >> 3) & 7
    lddw r1, map:pa
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, b
    ldxdw r1, [r0+0]
    add64 r1, 1
    stxdw [r0+0], r1
    ldxw r1, [r6+28]
    atomic_add64 [r0+8], r1
    ldxb r1, [r0+8]            ; sub-word read of the word just updated (not stored back)
b:
    mov64 r2, r7
    rsh64 r2, 7
    and64 r2, 3
    stxw [r10-8], r2          ; key B = (addr >> 7) & 3
    lddw r1, map:pb
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, c
    mov64 r8, r0
    mov64 r1, 2
    atomic_fetch_add32 [r8+4], r1
    mov64 r3, r7
    rsh64 r3, 10
    and64 r3, 127
    jne r3, 0, c              ; sub-word counters on 1/128 of the events, independent of key B:
                              ; < 256 per key in total, so no byte wrap on any shard or in the fold
    ldxb r3, [r8+0]
    add64 r3, 1
    stxb [r8+0], r3           ; byte counter (small counts: no carry)
    ldxh r3, [r8+2]
    add64 r3, 3
    stxh [r8+2], r3
c:
    mov64 r2, r7
    rsh64 r2, 5
    and64 r2, 15
    stxw [r10-12], r2         ; key C = (addr >> 5) & 15
    lddw r1, map:pc
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, out
    ldxdw r3, [r0+24]
    add64 r3, r7
    stxdw [r10-24], r3        ; value for update_elem: old + addr in word 3
    ldxdw r3, [r0+0]
    add64 r3, 1
    stxdw [r10-48], r3
    ldxdw r3, [r0+8]
    stxdw [r10-40], r3
    ldxdw r3, [r0+16]
    add64 r3, 5
    stxdw [r10-32], r3
    lddw r1, map:pc
    mov64 r2, r10
    add64 r2, -12
    mov64 r3, r10
    add64 r3, -48
    mov64 r4, 0
    call 2
out:
    mov64 r0, 0
    exit
"""


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("n", [1000, (1 << 16) + 7])
def test_perthread_stress_parity(gpu, engine, n):
    import torch
    from oracle.oracle import Oracle
    rng = np.random.default_rng(11 + n)
    ev = gen.records(n, addr=rng.integers(0, 1 << 20, n, dtype=np.uint64) * 8,
                     ts=np.zeros(n, dtype=np.uint64))
    ev["size"] = rng.integers(1, 17, n).astype(np.uint32)
    specs = {"pa": (6, 4, 16, 8), "pb": (6, 4, 8, 4), "pc": (6, 4, 32, 16)}
    env, rt = Oracle(), make_runtime(engine)
    fo = {k: env.create_map(*v) for k, v in specs.items()}
    fg = {k: rt.create_map(*v) for k, v in specs.items()}
    want = env.run(ev, env.load_prog(asm.assemble(PT_STRESS, fo)))
    ret = torch.zeros(n, dtype=torch.int64, device="cuda")
    rt.run(torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda(), rt.load_prog(asm.assemble(PT_STRESS, fg)), ret=ret)
    assert (ret.cpu().numpy().view(np.uint64) == want).all()
    for k in specs:
        assert rt.dump(fg[k]) == env.dump(fo[k]), k


@pytest.mark.parametrize("engine", ["jit", "jit_ring"])
@pytest.mark.parametrize("config", ["C2", "C3", "C5"])
def test_overlapped_batches_parity(gpu, config, engine):
    """gx_run_batch_ex(GX_RUN_OVERLAP): back-to-back batches launched with programmatic dependent
    launch keep the sequential semantics of one stream (S1): after 4 overlapped batches the maps and
    ringbuf equal the oracle's over the concatenated events."""
    import torch
    n = (1 << 16) + 96
    ev = configs.events(config, configs.SEEDS[config], 4 * n)
    env, so, _ = oracle_run(config, ev, threshold=2 if config == "C3" else None)
    rt = make_runtime(engine)
    s = configs.setup(rt, config, threshold=2 if config == "C3" else None)
    d_ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda()
    for k in range(4):
        rt.run(d_ev[k * n:(k + 1) * n], s.prog_arg, overlap=True)
    torch.cuda.synchronize()
    assert outputs(rt, s) == outputs(env, so)
    st, ost = rt.stats(), env.stats()
    assert st["events_run"] + st["events_skipped"] == 4 * n
    assert (st["events_run"], st["events_skipped"]) == (ost["events_run"], ost["events_skipped"])


@pytest.mark.parametrize("engine", ["jit", "jit_ring", "interp"])
@pytest.mark.parametrize("config", ["C2", "C3"])
def test_batches_on_different_streams_stay_ordered(gpu, config, engine):
    """Batches of one runtime given to different streams run in submission order (include/gx.h):
    4 batches alternating between two fresh streams, no host synchronisation in between, give the
    oracle's maps over the concatenated events -- per-thread shards (C2) and hash + FETCH-ADD +
    ringbuf (C3) would race if two batches overlapped."""
    import torch
    n = (1 << 18) + 32
    ev = configs.events(config, configs.SEEDS[config], 4 * n)
    env, so, _ = oracle_run(config, ev, threshold=2 if config == "C3" else None)
    rt = make_runtime(engine)
    s = configs.setup(rt, config, threshold=2 if config == "C3" else None)
    d_ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda()
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for k in range(4):
        rt.run(d_ev[k * n:(k + 1) * n], s.prog_arg, stream=streams[k % 2])
    torch.cuda.synchronize()
    assert outputs(rt, s) == outputs(env, so)


@pytest.mark.parametrize("mode,stages,release,claim,rpw", [
    (0, 3, "atom", "dynamic", 1), (1, 2, "atom", "dynamic", 1), (2, 4, "atom", "dynamic", 1),
    (3, 4, "atom", "dynamic", 1), (3, 3, "mbar", "dynamic", 1), (3, 3, "atom", "static", 1),
    (3, 3, "mbar", "static", 1), (3, 3, "atom", "static", 2), (3, 2, "atom", "static", 3),
    (3, 2, "atom", "static", 1)])
@pytest.mark.parametrize("config", ["C2", "C3", "C5"])
def test_ingest_variants_parity(gpu, config, mode, stages, release, claim, rpw, monkeypatch):
    """The alternative event-ingest variants kept for measurement (profiles/r1_jit_variants.md:
    per-lane / coalesced cp.async rings, per-warp TMA ring, deeper block ring) give the oracle's
    results too (ragged tail included)."""
    monkeypatch.setenv("GX_JIT_STAGE_MODE", str(mode))
    monkeypatch.setenv("GX_JIT_STAGES", str(stages))
    monkeypatch.setenv("GX_JIT_RING_RELEASE", release)
    monkeypatch.setenv("GX_JIT_RING_CLAIM", claim)
    monkeypatch.setenv("GX_JIT_RING_RPW", str(rpw))
    n = (1 << 17) + 21
    ev = configs.events(config, configs.SEEDS[config], n)
    rt, s, st = _compare(config, ev, threshold=2 if config == "C3" else None, engine="jit_ring")


@pytest.mark.parametrize("probe,cache", [("0", "0"), ("1", "0"), ("2", "0"), ("2", "2048"), ("2", "16"), ("1", "2048")])
@pytest.mark.parametrize("config,engine", [("C3", "jit_ring"), ("C3", "jit"), ("C5", "jit_ring")])
def test_hash_probe_variants_parity(gpu, config, engine, probe, cache, monkeypatch):
    """HASH probes through L1 (GX_JIT_HASH_L1PROBE: none / home slot / whole chain; keys never change
    once published, so a non-EMPTY key read through L1 is final) and the per-block shared-memory
    key -> slot cache (GX_JIT_HASH_CACHE entries; 16 forces constant entry collisions) give the
    oracle's results."""
    monkeypatch.setenv("GX_JIT_HASH_L1PROBE", probe)
    monkeypatch.setenv("GX_JIT_HASH_CACHE", cache)
    n = (1 << 17) + 5
    ev = configs.events(config, configs.SEEDS[config], n)
    _compare(config, ev, threshold=2 if config == "C3" else None, engine=engine)


@pytest.mark.parametrize("hint", ["0", "1", "2"])
@pytest.mark.parametrize("config", ["C2", "C5"])
def test_pt_hint_variants_parity(gpu, config, hint, monkeypatch):
    """Per-thread word accesses with L1 eviction-priority hints (GX_JIT_PT_HINT) give the oracle's
    results."""
    monkeypatch.setenv("GX_JIT_PT_HINT", hint)
    n = (1 << 17) + 9
    _compare(config, configs.events(config, configs.SEEDS[config], n), engine="jit_ring")
