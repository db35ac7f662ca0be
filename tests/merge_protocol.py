"""A second, independent implementation of the S3 snapshot-and-merge protocol (SURVEY.md §8c c.3,
§8e) in plain torch.distributed over an engine object -- TEST INFRASTRUCTURE.  tests/test_dist_gloo.py
drives it over an oracle-backed engine (OracleEngine) at world sizes 2 and 3 and compares it with the
oracle's own merge (ora_merge) and the unsharded run; the product path is the C-ABI gx_merge
(include/gx.h), checked in tests/test_gpu_merge.py.

    additive maps: export (local - base) into one packed u64 buffer -> all_reduce(SUM) -> apply;
    hash maps: (key, delta) grouped by owner = mix64(key) mod G -> all_to_all of counts and pairs ->
    the owner accumulates onto the base -> the owner's merged deltas -> all_gather -> every rank
    rebuilds base + merged deltas and commits it.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

HASH, ARRAY, PERTHREAD_ARRAY = 1, 2, 6


class ProtocolMerger:
    def __init__(self, eng, fds, group=None):
        self.eng = eng
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.additive = [fd for fd in fds if eng.spec(fd)[0] in (ARRAY, PERTHREAD_ARRAY)]
        self.hashes = [fd for fd in fds if eng.spec(fd)[0] == HASH]
        for fd in self.additive + self.hashes:
            eng.merge_snapshot(fd)
        self.words = [eng.merge_words(fd) for fd in self.additive]
        self.packed = torch.zeros(sum(self.words), dtype=torch.int64, device=eng.device)

    def merge(self):
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
        for fd in self.hashes:
            self._merge_hash(fd)

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
        self.eng.hash_apply(fd, rk, rv, restore=True, commit=False)
        ok, ov, _ = self.eng.hash_export(fd, G, self.rank)
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
