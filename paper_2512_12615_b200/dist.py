"""Multi-GPU snapshot-and-merge of gx maps (§8c S3).

"Consistency across shards is maintained via snapshot-based aggregation at GPU kernel completion
boundaries" (§5.3); maps are merged "into canonical snapshots at synchronization
points" (§4.4.3).  Each rank runs its contiguous event shard against replicated maps;
at a merge point every rank reaches

    canonical = init + sum over ranks of (local_rank - init)

(per u64 word, mod 2^64) for ARRAY and per-thread ARRAY maps, and the key union with summed value
deltas for HASH maps.  Ring buffers stay rank-local (their union is the multiset union, see
`ringbuf_union`).

Transport is torch.distributed (NCCL over NVLink on GPUs; gloo in the CPU tests) -- plumbing only;
every delta / apply step is a libgx kernel behind the C ABI (gx_merge_export / gx_merge_apply /
gx_hash_export / gx_hash_apply).  The protocol:
  1. additive maps: export deltas into ONE packed u64 buffer -> all_reduce(SUM) -> apply
     (u64 wraparound addition is what an int64 SUM does, so the allreduce is exact);
  2. hash maps (key-sharded): export (key, delta) grouped by owner = mix64(key) mod G -> exchange
     counts (all_to_all) -> exchange pairs (all_to_all) -> the owner accumulates its keys onto the
     base snapshot -> the owner exports its merged deltas -> all_gather -> every rank rebuilds
     local := base + merged deltas and commits it as the new base.

The engine is duck-typed: `Runtime` (the C-ABI library) on GPUs, or any object with the same
merge_* / hash_* methods (the CPU tests use an oracle-backed adapter).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

HASH, ARRAY, PERTHREAD_ARRAY, RINGBUF = 1, 2, 6, 27


class GxEngine:
    """Adapter giving `Runtime` the merge interface used by `Merger`."""

    def __init__(self, runtime):
        import paper_2512_12615_b200 as gx
        self.gx = gx
        self.rt = runtime
        self.device = torch.device("cuda", runtime.device)

    def spec(self, fd):
        return self.rt.specs[fd]

    def merge_snapshot(self, fd):
        self.gx.gx_merge_snapshot(self.rt.rt, fd)

    def merge_words(self, fd) -> int:
        return self.gx.gx_merge_words(self.rt.rt, fd)

    def merge_export(self, fd, out):
        self.gx.gx_merge_export(self.rt.rt, fd, out)

    def merge_apply(self, fd, total):
        self.gx.gx_merge_apply(self.rt.rt, fd, total)

    def hash_export(self, fd, nranks, owner):
        cap = self.spec(fd)[3] * 2 + 16
        keys = torch.empty(cap, dtype=torch.int64, device=self.device)
        vals = torch.empty(cap, dtype=torch.int64, device=self.device)
        counts = self.gx.gx_hash_export(self.rt.rt, fd, keys, vals, nranks, owner)
        n = sum(counts)
        return keys[:n], vals[:n], counts

    def hash_apply(self, fd, keys, vals, restore, commit):
        flags = (self.gx.GX_MERGE_RESTORE if restore else 0) | (self.gx.GX_MERGE_COMMIT if commit else 0)
        self.gx.gx_hash_apply(self.rt.rt, fd, keys.contiguous(), vals.contiguous(), keys.numel(), flags)


class Merger:
    def __init__(self, runtime_or_engine, fds, group=None):
        self.eng = runtime_or_engine if hasattr(runtime_or_engine, "merge_export") else GxEngine(runtime_or_engine)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.additive = [fd for fd in fds if self.eng.spec(fd)[0] in (ARRAY, PERTHREAD_ARRAY)]
        self.hashes = [fd for fd in fds if self.eng.spec(fd)[0] == HASH]
        for fd in self.additive + self.hashes:   # the agreed initial state
            self.eng.merge_snapshot(fd)
        self.words = [self.eng.merge_words(fd) for fd in self.additive]
        self.packed = torch.zeros(sum(self.words), dtype=torch.int64, device=self.eng.device)
        self.merges = 0

    def merge(self):
        """One synchronisation point (collective over all ranks of the group)."""
        # 1. additive maps: one packed allreduce
        if self.additive:
            off = 0
            for fd, w in zip(self.additive, self.words):
                self.eng.merge_export(fd, self.packed[off:off + w])
                off += w
            dist.all_reduce(self.packed, op=dist.ReduceOp.SUM, group=self.group)
            off = 0
            for fd, w in zip(self.additive, self.words):
                self.eng.merge_apply(fd, self.packed[off:off + w])
                off += w
        # 2. hash maps: key-sharded exchange
        for fd in self.hashes:
            self._merge_hash(fd)
        self.merges += 1

    def _merge_hash(self, fd):
        G, dev = self.world, self.eng.device
        keys, vals, counts = self.eng.hash_export(fd, G, -1)
        send_counts = torch.tensor(counts, dtype=torch.int64, device=dev)
        recv_counts = torch.empty(G, dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        rc = [int(x) for x in recv_counts.tolist()]
        rk = torch.empty(sum(rc), dtype=torch.int64, device=dev)
        rv = torch.empty(sum(rc), dtype=torch.int64, device=dev)
        dist.all_to_all_single(rk, keys, rc, counts, group=self.group)
        dist.all_to_all_single(rv, vals, rc, counts, group=self.group)
        # owner: base + all deltas of its keys (duplicates across ranks accumulate)
        self.eng.hash_apply(fd, rk, rv, restore=True, commit=False)
        ok, ov, _ = self.eng.hash_export(fd, G, self.rank)
        # replicate the owners' merged deltas
        n_mine = torch.tensor([ok.numel()], dtype=torch.int64, device=dev)
        sizes = [torch.empty(1, dtype=torch.int64, device=dev) for _ in range(G)]
        dist.all_gather(sizes, n_mine, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        mx = max(sizes) if sizes else 0
        pad_k = torch.zeros(mx, dtype=torch.int64, device=dev)
        pad_v = torch.zeros(mx, dtype=torch.int64, device=dev)
        pad_k[:ok.numel()] = ok
        pad_v[:ov.numel()] = ov
        gk = [torch.empty(mx, dtype=torch.int64, device=dev) for _ in range(G)]
        gv = [torch.empty(mx, dtype=torch.int64, device=dev) for _ in range(G)]
        dist.all_gather(gk, pad_k, group=self.group)
        dist.all_gather(gv, pad_v, group=self.group)
        allk = torch.cat([k[:s] for k, s in zip(gk, sizes)]) if mx else torch.empty(0, dtype=torch.int64, device=dev)
        allv = torch.cat([v[:s] for v, s in zip(gv, sizes)]) if mx else torch.empty(0, dtype=torch.int64, device=dev)
        self.eng.hash_apply(fd, allk, allv, restore=True, commit=True)


def shard_range(n_total: int, rank: int, world: int, align: int = 32):
    """Contiguous, 32-event-aligned shard [i0, i1) of a global batch (SURVEY.md §8e partition)."""
    cut = lambda g: min(n_total, ((g * n_total // world) + align - 1) // align * align) if g < world else n_total
    return cut(rank), cut(rank + 1)


def ringbuf_union(records: list[bytes], group=None) -> list[bytes]:
    """Multiset union of every rank's drained ring-buffer records (sorted), on every rank."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, records, group=group)
    return sorted(r for rs in out for r in rs)
