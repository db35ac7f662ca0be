"""Differential-fuzz plumbing shared by tests/test_fuzz_oracle.py (CPU: the generator's
determinism claims, checked on the oracle) and tests/test_gpu_fuzz.py (the CUDA path vs the
oracle).  An `engine` is the oracle's `Oracle` or the binding's `Runtime`: both expose
create_map / update_map / load_prog / attach / run / dump / ringbuf_records / stats."""
from __future__ import annotations

import numpy as np

from gxin import asm, fuzzprog as fp

RINGBUF = 27
COMPARED_STATS = ("events_run", "events_skipped", "ringbuf_drops", "hash_full")


def setup(engine, texts, seed, verify=None):
    """Creates the fuzz maps, writes their initial contents, loads + attaches the programs.
    Returns (fds, prog_arg): prog_arg = the single program's fd, or -1 (attach table)."""
    fds = {name: engine.create_map(*spec) for name, spec in fp.MAPS.items()}
    for name, keys, vals, n in fp.map_init(seed):
        _, ks, vs, _ = fp.MAPS[name]
        if hasattr(engine, "update_many"):
            assert engine.update_many(fds[name], keys, vals, n) == 0
        else:
            for i in range(n):
                assert engine.update_map(fds[name], keys[i * ks:(i + 1) * ks], vals[i * vs:(i + 1) * vs]) == 0
    progs = [engine.load_prog(asm.assemble(t, fds)) for t in texts]
    if len(progs) == 1:
        return fds, progs[0]
    for t, p in enumerate(progs):
        engine.attach(p, 0, t)
        engine.attach(p, 2, t)
    return fds, -1


def outputs(engine, fds, keep_stats=False):
    out = {}
    for name, fd in fds.items():
        if fp.MAPS[name][0] == RINGBUF:
            out[name] = tuple(engine.ringbuf_records(fd))
        else:
            out[name] = engine.dump(fd)
    st = engine.stats()
    out["stats"] = tuple(st[k] for k in COMPARED_STATS)
    if keep_stats:
        out["_stats"] = st
    return out


def verified(text) -> bool:
    import paper_2512_12615_b200 as gx
    fds = {name: i + 3 for i, name in enumerate(fp.MAPS)}
    v, _, _ = gx.gx_verify_offline(asm.assemble(text, fds), {fds[n]: s for n, s in fp.MAPS.items()})
    return v == 0


def case(seed):
    """One fuzz case: 1-3 verifier-accepted programs and an event batch (ragged sizes)."""
    rng = np.random.default_rng(seed)
    n_prog = 1 if rng.random() < 0.6 else int(rng.integers(2, 4))
    n = int(rng.choice([1, 31, 33, 64, 100, 257, 1000, 2048 + 13, 4096 + 31, 8192]))
    texts, k = [], 0
    while len(texts) < n_prog:
        t = fp.program(seed * 1000 + k)
        k += 1
        if verified(t):
            texts.append(t)
    ev = fp.events(seed, n, n_tenants=n_prog, skip_tenant=n_prog > 1 and rng.random() < 0.7)
    return texts, ev


def first_diff(a, b):
    if isinstance(a, tuple):
        return f"multiset sizes {len(a)} vs {len(b)}"
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return f"byte {i}"
    return f"lengths {len(a)} vs {len(b)}"
