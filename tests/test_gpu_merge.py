"""GPU merge kernels through the C ABI (gx_merge_export / gx_merge_apply / gx_hash_export /
gx_hash_apply) driven by the real protocol (paper_2512_12615_b200.dist.Merger): two processes
share cuda:0 (NCCL refuses two ranks on one device, so the collectives run over gloo with host
staging -- the 8-GPU NCCL path is the same Merger on CUDA tensors).  Every rank must end with the
oracle's own S3 snapshot-and-merge of the same shards (loopback merge)."""
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
    from paper_2512_12615_b200.dist import GxEngine, Merger, shard_range

    class Staged(GxEngine):
        def __init__(self, rt):
            super().__init__(rt)
            self.gpu = self.device
            self.device = torch.device("cpu")

        def merge_export(self, fd, out):
            tmp = torch.empty(out.shape, dtype=out.dtype, device=self.gpu)
            super().merge_export(fd, tmp)
            out.copy_(tmp.cpu())

        def merge_apply(self, fd, total):
            super().merge_apply(fd, total.to(self.gpu))
            torch.cuda.synchronize()

        def hash_export(self, fd, nranks, owner):
            self.device = self.gpu
            k, v, c = super().hash_export(fd, nranks, owner)
            self.device = torch.device("cpu")
            return k.cpu(), v.cpu(), c

        def hash_apply(self, fd, keys, vals, restore, commit):
            super().hash_apply(fd, keys.to(self.gpu), vals.to(self.gpu), restore, commit)

    rt = gx.Runtime(0)
    s = configs.setup(rt, config)
    fds = [fd for fd in s.fds.values() if rt.specs[fd][0] != RINGBUF]
    m = Merger(Staged(rt), fds)
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


@pytest.mark.parametrize("config", ["C2", "C3", "C5"])
def test_gpu_merge_matches_oracle_s3(gpu, config):
    from oracle.oracle import Oracle
    from paper_2512_12615_b200.dist import shard_range
    world, n = 2, (1 << 16) + 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, config, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
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
