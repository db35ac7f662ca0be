"""ctypes wrapper of liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this module.  The product path (paper_2512_12615_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "gx_oracle.c")

HASH, ARRAY, PERTHREAD_ARRAY, RINGBUF, PREFETCH_QUEUE, REGION = 1, 2, 6, 27, 64, 65
FN_MEM_PREFETCH = 1000   # gdev_mem_prefetch (F-1)
STATS = ("events_run", "events_skipped", "ringbuf_drops", "hash_full", "helper_errors", "insns")


def build(force: bool = False) -> str:
    """Compile the oracle (plain C11, -O2, no -march tuning)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", LIB_PATH, SRC_PATH])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp, i32, u32, u64, p64 = C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint64)
        L.ora_new.restype = vp
        L.ora_free.argtypes = [vp]
        L.ora_fault.restype = C.c_char_p
        L.ora_fault.argtypes = [vp]
        L.ora_clear_fault.argtypes = [vp]
        L.ora_stats.argtypes = [vp, p64]
        L.ora_reset_stats.argtypes = [vp]
        L.ora_map_create.argtypes = [vp, u32, u32, u32, u32]
        L.ora_region_map.argtypes = [vp, u64, u64]
        L.ora_map_update.argtypes = [vp, i32, vp, vp, u64]
        L.ora_map_update_n.argtypes = [vp, i32, vp, vp, u64, u64]
        L.ora_prog_load.argtypes = [vp, vp, u32]
        L.ora_attach.argtypes = [vp, i32, u32, u32]
        L.ora_set_pt_shards.argtypes = [vp, u32]
        L.ora_run.argtypes = [vp, vp, u64, i32, p64, p64, u64]
        L.ora_map_dump.argtypes = [vp, i32, vp, u64, p64]
        L.ora_ringbuf_dump.argtypes = [vp, i32, vp, u64, p64, p64]
        L.ora_ringbuf_used.argtypes = [vp, i32]
        L.ora_ringbuf_used.restype = u64
        L.ora_pfq_dump.argtypes = [vp, i32, p64, u64, p64, p64]
        L.ora_pfq_reset.argtypes = [vp, i32]
        u32p = C.POINTER(C.c_uint32)
        L.ora_sched_run.argtypes = [vp, i32, C.c_uint32, u32p, u32p, C.c_uint32, C.c_uint32, u32p,
                                    C.POINTER(C.c_uint8), p64, p64, u32p, p64]
        L.ora_clone.argtypes = [vp]
        L.ora_clone.restype = vp
        L.ora_merge.argtypes = [vp, C.POINTER(vp), i32]
        _lib = L
    return _lib


class OracleFault(RuntimeError):
    pass


class Oracle:
    """One sequential eBPF environment (maps + programs + attach table)."""

    def __init__(self, _handle=None):
        self.L = lib()
        self.h = _handle if _handle is not None else self.L.ora_new()
        self.specs = {}

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ora_free(self.h)
            self.h = None

    def create_map(self, type, key_size, value_size, max_entries) -> int:
        fd = self.L.ora_map_create(self.h, type, key_size, value_size, max_entries)
        if fd < 0:
            raise OSError(-fd, "ora_map_create")
        self.specs[fd] = (type, key_size, value_size, max_entries)
        return fd

    def region_map(self, base: int, length: int) -> int:
        """A device byte range [base, base + length) for gdev_prefetch_l2 (F-7)."""
        fd = self.L.ora_region_map(self.h, base, length)
        if fd < 0:
            raise OSError(-fd, "ora_region_map")
        self.specs[fd] = (REGION, 0, 0, 1)
        return fd

    def update_map(self, fd, key: bytes, val: bytes, flags=0) -> int:
        return self.L.ora_map_update(self.h, fd, key, val, flags)

    def update_many(self, fd, keys: bytes, vals: bytes, n: int, flags=0) -> int:
        return self.L.ora_map_update_n(self.h, fd, keys, vals, n, flags)

    def load_prog(self, slots: bytes) -> int:
        p = self.L.ora_prog_load(self.h, slots, len(slots) // 8)
        if p < 0:
            raise OSError(-p, "ora_prog_load")
        return p

    def attach(self, prog, kind, tenant):
        assert self.L.ora_attach(self.h, prog, kind, tenant) == 0

    def set_pt_shards(self, S):
        assert self.L.ora_set_pt_shards(self.h, S) == 0

    def run(self, events: np.ndarray, prog: int = -1, order=None, index_base: int = 0, want_r0=True):
        ev = np.ascontiguousarray(events)
        n = len(ev)
        r0 = np.zeros(n, dtype=np.uint64) if want_r0 else None
        o = None
        if order is not None:
            order = np.ascontiguousarray(order, dtype=np.uint64)
            o = order.ctypes.data_as(C.POINTER(C.c_uint64))
        rc = self.L.ora_run(self.h, ev.ctypes.data, n, prog,
                            r0.ctypes.data_as(C.POINTER(C.c_uint64)) if want_r0 else None, o, index_base)
        if rc:
            raise OracleFault(self.L.ora_fault(self.h).decode())
        return r0

    def fault(self) -> str:
        return self.L.ora_fault(self.h).decode()

    def stats(self) -> dict:
        out = (C.c_uint64 * 8)()
        self.L.ora_stats(self.h, out)
        return dict(zip(STATS, list(out)[:len(STATS)]))

    def dump(self, fd) -> bytes:
        """Canonical map content as bytes; HASH: sorted (key||value) entries."""
        type_, ks, vs, me = self.specs[fd]
        cap = me * (vs + ks) + 8
        buf = C.create_string_buffer(cap)
        n = C.c_uint64()
        rc = self.L.ora_map_dump(self.h, fd, buf, cap, C.byref(n))
        if rc:
            raise OSError(-rc, "ora_map_dump")
        if type_ == HASH:
            return buf.raw[: n.value * (ks + vs)]
        return buf.raw[: n.value]

    def array_u64(self, fd) -> np.ndarray:
        return np.frombuffer(self.dump(fd), dtype=np.uint64)

    def hash_items(self, fd) -> dict:
        _, ks, vs, _ = self.specs[fd]
        raw = self.dump(fd)
        es = ks + vs
        out = {}
        for k in range(0, len(raw), es):
            key = int.from_bytes(raw[k:k + ks], "little")
            out[key] = np.frombuffer(raw[k + ks:k + es], dtype=np.uint64).copy()
        return out

    def ringbuf_records(self, fd) -> list[bytes]:
        """The ringbuf multiset as a sorted list of payloads."""
        used = self.L.ora_ringbuf_used(self.h, fd)
        cap = used * 2 + 16
        buf = C.create_string_buffer(int(cap))
        nr, nb = C.c_uint64(), C.c_uint64()
        rc = self.L.ora_ringbuf_dump(self.h, fd, buf, cap, C.byref(nr), C.byref(nb))
        if rc:
            raise OSError(-rc, "ora_ringbuf_dump")
        raw, out, o = buf.raw[: nb.value], [], 0
        while o < len(raw):
            ln = int.from_bytes(raw[o:o + 4], "little")
            out.append(raw[o + 4:o + 4 + ln])
            o += 4 + ln
        return out

    def prefetch_requests(self, fd) -> list[tuple[int, int]]:
        """The prefetch queue's canonical content (F-2): the sorted SET of
        (first_page, npages) requests; `self.last_pfq_calls` = requests appended."""
        cap = int(self.specs[fd][3])
        buf = (C.c_uint64 * (2 * cap + 2))()
        n, nc = C.c_uint64(), C.c_uint64()
        rc = self.L.ora_pfq_dump(self.h, fd, buf, cap, C.byref(n), C.byref(nc))
        if rc:
            raise OSError(-rc, "ora_pfq_dump")
        self.last_pfq_calls = nc.value
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)]

    def prefetch_reset(self, fd):
        self.L.ora_pfq_reset(self.h, fd)

    def sched_run(self, prog, cost_us, home, n_workers, steal_cost_us=0) -> dict:
        """f3 (F-5): the work-stealing scheduler as a discrete-event simulation, the hooks
        run by this oracle.  Returns executed_by, stolen, busy_us, end_us, steals, makespan_us."""
        import numpy as np
        cost = np.ascontiguousarray(cost_us, dtype=np.uint32)
        hm = np.ascontiguousarray(home, dtype=np.uint32)
        U = len(cost)
        ex = np.zeros(U, dtype=np.uint32)
        st = np.zeros(U, dtype=np.uint8)
        busy = np.zeros(n_workers, dtype=np.uint64)
        end = np.zeros(n_workers, dtype=np.uint64)
        steals = np.zeros(n_workers, dtype=np.uint32)
        ms = C.c_uint64()
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        rc = self.L.ora_sched_run(self.h, prog, U, P(cost, C.c_uint32), P(hm, C.c_uint32), n_workers, steal_cost_us,
                                  P(ex, C.c_uint32), P(st, C.c_uint8), P(busy, C.c_uint64), P(end, C.c_uint64),
                                  P(steals, C.c_uint32), C.byref(ms))
        if rc:
            raise OSError(-rc if rc < 0 else rc, "ora_sched_run: " + self.fault())
        return dict(executed_by=ex, stolen=st, busy_us=busy, end_us=end, steals=steals, makespan_us=ms.value)

    def clone(self) -> "Oracle":
        c = Oracle(self.L.ora_clone(self.h))
        c.specs = dict(self.specs)
        return c

    def merge(self, locals_: list["Oracle"]) -> int:
        """S3 snapshot-and-merge of `locals_` into self (self holds the common initial state)."""
        arr = (C.c_void_p * len(locals_))(*[x.h for x in locals_])
        return self.L.ora_merge(self.h, arr, len(locals_))
