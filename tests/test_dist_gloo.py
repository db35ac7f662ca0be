"""Multi-rank S3 merge protocol (tests/merge_protocol.py, the reference implementation the C-ABI
gx_merge is checked against on the GPU) on CPU: world_size 2 and 3 over gloo,
each rank running its contiguous event shard on an ORACLE-backed engine.  The merged maps on every
rank must equal (a) the oracle's own S3 snapshot-and-merge (ora_merge) and (b) for partition-
insensitive configs, the single-environment unsharded run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gxin import configs, gen

HASH, ARRAY, PT, RINGBUF = 1, 2, 6, 27
M64 = (1 << 64) - 1


class OracleEngine:
    """Merge-interface adapter over one oracle environment (test infrastructure).  Base snapshots
    are plain numpy copies of the canonical dumps taken at the previous merge point."""

    device = torch.device("cpu")

    def __init__(self, env, fds):
        self.env = env
        self.base = {}
        for fd in fds:
            self.base[fd] = self._read(fd)

    def spec(self, fd):
        return self.env.specs[fd]

    def _read(self, fd):
        t = self.spec(fd)[0]
        if t == HASH:
            return {k: int(v[0]) for k, v in self.env.hash_items(fd).items()}
        if t == RINGBUF:
            return None
        return self.env.array_u64(fd).copy()

    def merge_snapshot(self, fd):
        self.base[fd] = self._read(fd)

    def merge_words(self, fd):
        return self.spec(fd)[2] * self.spec(fd)[3] // 8

    def merge_export(self, fd, out):
        d = self.env.array_u64(fd) - self.base[fd]
        out.copy_(torch.from_numpy(d.view(np.int64)))

    def merge_apply(self, fd, total):
        new = self.base[fd] + total.numpy().view(np.uint64)
        vs = self.spec(fd)[2]
        for k in range(self.spec(fd)[3]):
            self.env.update_map(fd, k.to_bytes(4, "little"), new[k * vs // 8:(k + 1) * vs // 8].tobytes(), 0)
        self.base[fd] = new

    def hash_export(self, fd, nranks, owner):
        cur = self._read(fd)
        base = self.base[fd]
        rows = [(k, (v - base.get(k, 0)) & M64) for k, v in cur.items() if k not in base or v != base[k]]
        own = [int(gen.mix64(np.uint64(k))) % nranks for k, _ in rows]
        grouped = [[r for r, o in zip(rows, own) if o == g and (owner < 0 or g == owner)] for g in range(nranks)]
        flat = [r for g in grouped for r in g]
        keys = torch.tensor([np.int64(np.uint64(k)) for k, _ in flat] or [], dtype=torch.int64)
        vals = torch.tensor([np.int64(np.uint64(d)) for _, d in flat] or [], dtype=torch.int64)
        return keys, vals, [len(g) for g in grouped]

    def hash_apply(self, fd, keys, vals, restore, commit):
        ks = self.spec(fd)[1]
        acc = {}
        for k, d in zip(keys.numpy().view(np.uint64).tolist(), vals.numpy().view(np.uint64).tolist()):
            acc[k] = (acc.get(k, 0) + d) & M64
        cur = self._read(fd)
        for k, d in acc.items():
            start = self.base[fd].get(k, 0) if restore else cur.get(k, 0)
            self.env.update_map(fd, k.to_bytes(ks, "little"), ((start + d) & M64).to_bytes(8, "little"), 0)
        if commit:
            self.base[fd] = self._read(fd)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, config, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_2512_12615_b200.dist import shard_range
    from merge_protocol import ProtocolMerger as Merger
    env = Oracle()
    s = configs.setup(env, config)
    fds = [fd for fd in s.fds.values() if env.specs[fd][0] != RINGBUF]
    eng = OracleEngine(env, fds)
    m = Merger(eng, fds)
    i0, i1 = shard_range(n, rank, world)
    ev = configs.events(config, configs.SEEDS[config], i1 - i0, i0, n)
    half = (i1 - i0) // 2 // 32 * 32
    env.run(ev[:half], s.prog_arg, index_base=i0)       # two merge points per rank
    m.merge()
    env.run(ev[half:], s.prog_arg, index_base=i0 + half)
    m.merge()
    q.put((rank, {key: env.dump(fd) for key, fd in s.fds.items() if env.specs[fd][0] != RINGBUF}))
    dist.destroy_process_group()


@pytest.mark.parametrize("config,world", [("C1", 2), ("C2", 2), ("C4", 2), ("C5", 3), ("C3", 2)])
def test_merge_protocol_gloo(config, world):
    from oracle.oracle import Oracle
    n = 1 << 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, config, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # (a) the oracle's own S3 merge of the same shards (two merge points)
    from paper_2512_12615_b200.dist import shard_range
    init = Oracle()
    si = configs.setup(init, config)
    ev = configs.events(config, configs.SEEDS[config], n)
    cuts = [shard_range(n, r, world) for r in range(world)]
    for part in (0, 1):
        locals_ = [init.clone() for _ in range(world)]
        for r, env in enumerate(locals_):
            i0, i1 = cuts[r]
            half = (i1 - i0) // 2 // 32 * 32
            a, b = (i0, i0 + half) if part == 0 else (i0 + half, i1)
            env.run(ev[a:b], si.prog_arg, index_base=a)
        init.merge(locals_)
    want = {key: init.dump(fd) for key, fd in si.fds.items() if init.specs[fd][0] != RINGBUF}
    for r in range(world):
        assert res[r] == want, (config, r)
    # (b) partition-insensitive configs: equal to the unsharded sequential run
    if config != "C3":
        one = Oracle()
        so = configs.setup(one, config)
        one.run(ev, so.prog_arg)
        assert {key: one.dump(fd) for key, fd in so.fds.items() if one.specs[fd][0] != RINGBUF} == want


def test_shard_range_partition():
    from paper_2512_12615_b200.dist import shard_range
    for n in (0, 1, 31, 32, 1000, 1 << 20, 10 ** 10):
        for world in (1, 2, 3, 8):
            cuts = [shard_range(n, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            for (a, b), (c, d) in zip(cuts, cuts[1:]):
                assert b == c and a <= b
            assert all(a % 32 == 0 or a == n for a, _ in cuts)
