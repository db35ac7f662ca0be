"""Multi-GPU process bootstrap for gx_merge (§8c S3).

"Consistency across shards is maintained via snapshot-based aggregation at GPU kernel completion
boundaries" (§5.3); maps are merged "into canonical snapshots at synchronization
points" (§4.4.3).  One process per GPU runs its contiguous event shard against
replicated maps; the merge itself -- delta export, the NCCL collectives over NVLink / NVSwitch, the
owner-sharded HASH exchange, apply -- is ONE C-ABI call, gx_merge (include/gx.h), on the library's
own communicator.  This module only bootstraps it:

  * comm_init(runtime, group): NCCL process groups -> rank 0 makes an NCCL unique id
    (gx_comm_unique_id), torch.distributed ships it, every rank calls gx_comm_init;
    gloo groups (several ranks sharing one device, CPU-side tests) -> gx_comm_init_host with
    callbacks that run the three collectives on host buffers over the group;
  * Merger(runtime, group).merge() -> gx_merge on the current stream;
  * shard_range (the partition), ringbuf_union (ring buffers stay rank-local: their union is the
    multiset union of the drained records).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def _host_ops(group):
    """The three host collectives of gx_comm_host_ops over a torch.distributed group."""
    world = dist.get_world_size(group)

    def allreduce(buf_u64):
        t = torch.from_numpy(buf_u64.view(np.int64))        # shares memory; int64 SUM wraps like u64
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    def alltoallv(send, sb, so, recv, rb, ro):
        parts = [torch.from_numpy(send[int(so[g]):int(so[g] + sb[g])].copy()) for g in range(world)]
        inp = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.uint8)
        out = torch.empty(int(rb.sum()), dtype=torch.uint8)
        dist.all_to_all_single(out, inp, [int(x) for x in rb], [int(x) for x in sb], group=group)
        o = out.numpy()
        pos = 0
        for g in range(world):
            n = int(rb[g])
            recv[int(ro[g]):int(ro[g]) + n] = o[pos:pos + n]
            pos += n

    def allgather(send, recv):
        n = send.shape[0]
        outs = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(outs, torch.from_numpy(send.copy()), group=group)
        for g, t in enumerate(outs):
            recv[g * n:(g + 1) * n] = t.numpy()

    return allreduce, alltoallv, allgather


def comm_init(runtime, group=None):
    """Joins this rank's gx_rt to the merge communicator of `group` (collective).  Call it after
    every rank created the same maps and wrote the same initial contents: the base snapshot taken
    here is the state all ranks agree on."""
    import paper_2512_12615_b200 as gx
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        obj = [gx.gx_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        gx.gx_comm_init(runtime.rt, obj[0], world, rank)
        runtime._comm_ops = None
    else:
        ar, a2a, ag = _host_ops(group)
        runtime._comm_ops = gx.gx_comm_init_host(runtime.rt, ar, a2a, ag, world, rank)


class Merger:
    """merge() = one synchronisation point: gx_merge on every rank of the group."""

    def __init__(self, runtime, group=None):
        self.rt = runtime
        self.group = group
        comm_init(runtime, group)
        self.merges = 0

    def merge(self, stream=None):
        import paper_2512_12615_b200 as gx
        gx.gx_merge(self.rt.rt, stream)
        self.merges += 1


def shard_range(n_total: int, rank: int, world: int, align: int = 32):
    """Contiguous, 32-event-aligned shard [i0, i1) of a global batch (SURVEY.md §8e partition)."""
    cut = lambda g: min(n_total, ((g * n_total // world) + align - 1) // align * align) if g < world else n_total
    return cut(rank), cut(rank + 1)


def ringbuf_union(records: list[bytes], group=None) -> list[bytes]:
    """Multiset union of every rank's drained ring-buffer records (sorted), on every rank."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, records, group=group)
    return sorted(r for rs in out for r in rs)
