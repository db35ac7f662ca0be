"""The C-ABI multi-GPU merge (gx_comm_init / gx_merge, include/gx.h) against the oracle's S3
snapshot-and-merge (SURVEY.md §8c c.3 S3, §8e loopback).  G processes share cuda:0: NCCL refuses two
ranks on one device, so the ranks join through gx_comm_init_host with gloo collectives on host
buffers (paper_2512_12615_b200.dist.comm_init); every other step -- delta export, packing, the
owner-sharded HASH exchange, apply -- is the same gx_merge code the NCCL path runs.  The NCCL path
itself runs at G = 1 here (and at G = 2..8 in `bench.py --gpus N`).  Every rank must end with the
oracle's merged maps, at G = 2, 3 and 8 (C5 at 2^24 events: SURVEY.md §8d parity matrix)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gxin import configs

pytestmark = pytest.mark.gpu
RINGBUF = 27


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, config, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2512_12615_b200 as gx
    from paper_2512_12615_b200.dist import Merger, shard_range

    rt = gx.Runtime(0)
    s = configs.setup(rt, config)
    m = Merger(rt)
    i0, i1 = shard_range(n, rank, world)
    ev = configs.events(config, configs.SEEDS[config], i1 - i0, i0, n)
    d_ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda()
    half = (i1 - i0) // 2 // 32 * 32
    rt.run(d_ev[:half], s.prog_arg)
    m.merge()
    rt.run(d_ev[half:], s.prog_arg)
    m.merge()
    q.put((rank, {key: rt.dump(fd) for key, fd in s.fds.items() if rt.specs[fd][0] != RINGBUF}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("config,world,lg", [("C2", 2, 16), ("C3", 2, 16), ("C4", 3, 16), ("C5", 2, 16),
                                             ("C5", 8, 24)])
def test_gpu_merge_matches_oracle_s3(gpu, config, world, lg):
    from oracle.oracle import Oracle
    from paper_2512_12615_b200.dist import shard_range
    n = (1 << lg) + 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, config, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
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


def test_merge_nccl_single_rank(gpu):
    """The NCCL transport itself (gx_comm_init at G = 1): a merge leaves every map as it is."""
    import torch
    import paper_2512_12615_b200 as gx
    rt = gx.Runtime(0)
    s = configs.setup(rt, "C5")
    gx.gx_comm_init(rt.rt, gx.gx_comm_unique_id(), 1, 0)
    ev = configs.events("C5", configs.SEEDS["C5"], 1 << 16)
    rt.run(torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda(), s.prog_arg)
    before = {key: rt.dump(fd) for key, fd in s.fds.items() if rt.specs[fd][0] != RINGBUF}
    gx.gx_merge(rt.rt)
    after = {key: rt.dump(fd) for key, fd in s.fds.items() if rt.specs[fd][0] != RINGBUF}
    assert before == after
    rt.run(torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda(), s.prog_arg)
    gx.gx_merge(rt.rt)   # the base advanced: a second batch merges onto the first
    rt.close()


def test_merge_refuses_non_additive_maps(gpu):
    """S3 legality: an ARRAY written by a plain store (or a HASH updated with BPF_ANY) has no
    snapshot-and-merge -- gx_merge returns -EINVAL and leaves every map untouched."""
    import torch
    import paper_2512_12615_b200 as gx
    from gxin import asm
    for text, spec in (("ldxdw r2, [r1+0]\nstdw [r10-8], 0\nmov64 r3, 0\nstxw [r10-4], r3\nlddw r1, map:m\n"
                        "mov64 r2, r10\nadd64 r2, -4\ncall 1\njeq r0, 0, +1\nstdw [r0+0], 7\nmov64 r0, 0\nexit",
                        (2, 4, 8, 4)),
                       ("ldxdw r2, [r1+0]\nstxdw [r10-8], r2\nstdw [r10-16], 1\nlddw r1, map:m\nmov64 r2, r10\n"
                        "add64 r2, -8\nmov64 r3, r10\nadd64 r3, -16\nmov64 r4, 0\ncall 2\nmov64 r0, 0\nexit",
                        (1, 8, 8, 64))):
        rt = gx.Runtime(0)
        fd = rt.create_map(*spec)
        rt.load_prog(asm.assemble(text, {"m": fd}))
        gx.gx_comm_init(rt.rt, gx.gx_comm_unique_id(), 1, 0)
        with pytest.raises(gx.GxError) as e:
            gx.gx_merge(rt.rt)
        assert e.value.errno == 22
        rt.close()
