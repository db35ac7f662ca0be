"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times (JIT engine,
runtime-chosen ingest, no per-event R0), on device-generated events (task rule ③).

The oracle cannot interpret 2^28-2^31 events in test time, so every map is compared with the
closed form of its config -- the same definitions the oracle is pinned against in
tests/test_oracle_configs.py (tests/closed_forms.py) -- evaluated with plain torch reductions
(bincount / unique / searchsorted) over the very event tensor the kernel read.  Integer results:
exact equality."""
import numpy as np
import pytest

from gxin import configs, gen, gen_gpu
from gpu_util import make_runtime

pytestmark = pytest.mark.gpu


def _fields(ev):
    """u64 columns of the (N, 32) event tensor (SURVEY.md §8b layout), as int64 views."""
    w = ev.view(-1, 32).view(dtype=__import__("torch").int64)
    return w[:, 0], w[:, 3]


def _run(config, n):
    import torch
    rt = make_runtime("jit")
    s = configs.setup(rt, config)
    ev = gen_gpu.generate_device(config, configs.SEEDS[config], n)
    rt.run(ev, s.prog_arg)
    torch.cuda.synchronize()
    st = rt.stats()
    assert st["events_run"] + st["events_skipped"] == n
    # helper_errors is parity-unpinned: a NOEXIST insert that loses a race to another
    # warp returns -EEXIST and the program re-looks the key up, as it does sequentially
    assert st["hash_full"] == 0 and st["ringbuf_drops"] == 0
    return rt, s, ev


def test_c2_full_size(gpu):
    """C2 (the bench's headline workload): 2^30 events; hist = bincount(sm*64 + warp), the
    per-thread fold = per-lane event counts and byte sums (closed_forms.c2_expected)."""
    import torch
    n = 1 << 30
    rt, s, ev = _run("C2", n)
    _, w3 = _fields(ev)
    hist = torch.zeros(148 * 64, dtype=torch.int64, device=ev.device)
    cnt = torch.zeros(32, dtype=torch.int64, device=ev.device)
    byt = torch.zeros(32, dtype=torch.int64, device=ev.device)
    for c in range(0, n, 1 << 27):
        x = w3[c:c + (1 << 27)]
        key = (x & 0xFFFF) * 64 + ((x >> 16) & 0xFF)
        lane = (x >> 24) & 0xFF
        hist += torch.bincount(key, minlength=148 * 64)
        cnt += torch.bincount(lane, minlength=32)
        byt.index_add_(0, lane, (x >> 32) & 0xFFFFFFFF)
    got_hist = rt.array_u64(s.fds[(0, "hist")])
    assert (got_hist == hist.cpu().numpy().astype(np.uint64)).all()
    assert int(got_hist.sum()) == n                      # north star: counter total = event count
    pt = rt.array_u64(s.fds[(0, "lane_pt")]).reshape(32, 2)
    assert (pt[:, 0] == cnt.cpu().numpy().astype(np.uint64)).all()
    assert (pt[:, 1] == byt.cpu().numpy().astype(np.uint64)).all()


def test_c3_full_size(gpu):
    """C3: 2^28 LLM page-trace events; the LFU hash = exact page counts, the ringbuf = one
    {page, 64} record per page whose count reaches 64 (closed_forms.c3_expected)."""
    import torch
    n = 1 << 28
    rt, s, ev = _run("C3", n)
    addr, _ = _fields(ev)
    pages, counts = torch.unique(addr >> 12, return_counts=True)
    want = dict(zip(pages.cpu().tolist(), counts.cpu().tolist()))
    got = {k: int(v[0]) for k, v in rt.hash_items(s.fds[(0, "lfu")]).items()}
    assert got == want
    hot = pages[counts >= 64].cpu().numpy().astype(np.uint64)
    want_rb = sorted(int(p).to_bytes(8, "little") + (64).to_bytes(8, "little") for p in hot)
    assert rt.ringbuf_records(s.fds[(0, "rb")]) == want_rb


def test_c4_full_size(gpu):
    """C4: 2^31 vector-search events (64 GiB); list id = searchsorted(bounds, addr) - 1 for scans,
    centroid scans counted (closed_forms.c4_expected)."""
    import torch
    n = 1 << 31
    rt, s, ev = _run("C4", n)
    addr, w3 = _fields(ev)
    bounds = torch.from_numpy(gen.c4_tables()["bounds"].astype(np.int64)).to(ev.device)
    cent = torch.zeros((), dtype=torch.int64, device=ev.device)
    hits = torch.zeros(4096, dtype=torch.int64, device=ev.device)
    lbytes = torch.zeros(4096, dtype=torch.int64, device=ev.device)
    scan_bytes = torch.zeros((), dtype=torch.int64, device=ev.device)
    for c in range(0, n, 1 << 27):
        a = addr[c:c + (1 << 27)].contiguous()
        size = (w3[c:c + (1 << 27)] >> 32) & 0xFFFFFFFF
        is_c = a < bounds[0]
        cent += is_c.sum()
        lst = (torch.searchsorted(bounds, a, right=True) - 1).clamp(0, 4095)[~is_c]
        sz = size[~is_c]
        hits += torch.bincount(lst, minlength=4096)
        lbytes.index_add_(0, lst, sz)
        scan_bytes += sz.sum()
    assert int(rt.array_u64(s.fds[(0, "cstat")])[0]) == int(cent)
    h = hits.cpu().numpy()
    want_hits = {int(k): int(h[k]) for k in np.nonzero(h)[0]}
    got_hits = {k: int(v[0]) for k, v in rt.hash_items(s.fds[(0, "list_hits")]).items()}
    assert got_hits == want_hits
    assert (rt.array_u64(s.fds[(0, "list_bytes")]) == lbytes.cpu().numpy().astype(np.uint64)).all()
    assert int(rt.array_u64(s.fds[(0, "scan_pt")])[0]) == int(scan_bytes)


def test_c5_full_size(gpu):
    """C5: 2^28 multi-tenant events (the bench's single-GPU C5 batch), four programs through the
    attach table; every tenant's maps against its closed form (closed_forms: c1_counts / c2_expected /
    c3_expected / c4_expected restricted to the tenant's events, SURVEY.md §8c c.5 "C5 mix"), the
    ringbuf = one {page, sm_id} record per FAULT event of tenant 2 (as a multiset)."""
    import torch
    import paper_2512_12615_b200 as gx
    n = 1 << 28
    rt, s, ev = _run("C5", n)
    w = ev.view(-1, 32).view(dtype=torch.int64)
    addr, hookw, w3 = w[:, 0], w[:, 2], w[:, 3]
    tenant = (hookw >> 8) & 0xFF
    kind = hookw & 0xFF
    sm, warp, lane, size = w3 & 0xFFFF, (w3 >> 16) & 0xFF, (w3 >> 24) & 0xFF, (w3 >> 32) & 0xFFFFFFFF
    assert rt.stats()["events_skipped"] == 0
    # tenant 0: P1
    t0 = tenant == 0
    want = torch.bincount(((addr[t0] >> 12) & 255), minlength=256)
    assert (rt.array_u64(s.fds[(0, "counts")]) == want.cpu().numpy().astype(np.uint64)).all()
    # tenant 1: P2
    t1 = tenant == 1
    hist = torch.bincount(sm[t1] * 64 + warp[t1], minlength=148 * 64)
    assert (rt.array_u64(s.fds[(1, "hist")]) == hist.cpu().numpy().astype(np.uint64)).all()
    cnt = torch.bincount(lane[t1], minlength=32)
    byt = torch.zeros(32, dtype=torch.int64, device=ev.device).index_add_(0, lane[t1], size[t1])
    pt = rt.array_u64(s.fds[(1, "lane_pt")]).reshape(32, 2)
    assert (pt[:, 0] == cnt.cpu().numpy().astype(np.uint64)).all()
    assert (pt[:, 1] == byt.cpu().numpy().astype(np.uint64)).all()
    # tenant 2: P3' (page counts + unconditional FAULT records)
    t2 = tenant == 2
    pages, counts = torch.unique(addr[t2] >> 12, return_counts=True)
    got = {k: int(v[0]) for k, v in rt.hash_items(s.fds[(2, "lfu")]).items()}
    assert got == dict(zip(pages.cpu().tolist(), counts.cpu().tolist()))
    f = t2 & (kind == 2)
    want_rb = torch.stack([addr[f] >> 12, sm[f]], 1).cpu().numpy().astype(np.uint64)
    recs = gx.gx_ringbuf_drain(rt.rt, s.fds[(2, "rb")])
    assert len(recs) == len(want_rb) > 0 and all(len(r) == 16 for r in recs[:1000])
    got_rb = np.frombuffer(b"".join(recs), dtype=np.uint64).reshape(-1, 2)
    o1, o2 = np.lexsort(got_rb.T[::-1]), np.lexsort(want_rb.T[::-1])
    assert (got_rb[o1] == want_rb[o2]).all()
    # tenant 3: P4
    t3 = tenant == 3
    a3, s3 = addr[t3].contiguous(), size[t3]
    bounds = torch.from_numpy(gen.c4_tables()["bounds"].astype(np.int64)).to(ev.device)
    is_c = a3 < bounds[0]
    lst = (torch.searchsorted(bounds, a3, right=True) - 1).clamp(0, 4095)[~is_c]
    assert int(rt.array_u64(s.fds[(3, "cstat")])[0]) == int(is_c.sum())
    h = torch.bincount(lst, minlength=4096).cpu().numpy()
    got_hits = {k: int(v[0]) for k, v in rt.hash_items(s.fds[(3, "list_hits")]).items()}
    assert got_hits == {int(k): int(h[k]) for k in np.nonzero(h)[0]}
    lb = torch.zeros(4096, dtype=torch.int64, device=ev.device).index_add_(0, lst, s3[~is_c])
    assert (rt.array_u64(s.fds[(3, "list_bytes")]) == lb.cpu().numpy().astype(np.uint64)).all()
    assert int(rt.array_u64(s.fds[(3, "scan_pt")])[0]) == int(s3[~is_c].sum())
