"""Python binding of libgx.so (include/gx.h) -- argument marshalling only.

Every function named gx_* here calls the C-ABI entry point of the same name; every step
of the hot path runs in the library's sm_100a kernels.  There is no CPU fallback: if
libgx.so is missing or no sm_100 device is present, the calls raise.

PyTorch is used only for device memory and streams: event batches are torch.uint8 CUDA
tensors of shape (N, 32), streams are torch.cuda streams.

`Runtime` wraps one gx_rt with the engine methods gxin.configs.setup drives
(create_map / update_map / load_prog / attach) plus run / read helpers.
"""
from __future__ import annotations

import ctypes as C
import errno
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgx.so")

GX_MAP_HASH, GX_MAP_ARRAY, GX_MAP_PERTHREAD_ARRAY, GX_MAP_RINGBUF, GX_MAP_PREFETCH_QUEUE, GX_MAP_REGION = 1, 2, 6, 27, 64, 65
GX_FN_MEM_PREFETCH, GX_FN_PREFETCH_L2 = 1000, 1001
RULES = ("OK", "BAD_INSN", "BAD_REG", "BAD_JUMP", "FALLTHROUGH", "UNREACHABLE", "UNINIT_READ", "OOB_ACCESS",
         "NULL_DEREF", "MISALIGNED", "PTR_LEAK", "SHIFT_RANGE", "BAD_HELPER", "FORBIDDEN_SYNC", "UNBOUNDED_LOOP",
         "COMPLEXITY", "BUDGET", "UNIFORM_BRANCH", "UNIFORM_LOOP_BOUND", "UNIFORM_MAP_KEY", "NON_UNIFORM_ATOMIC",
         "MIXED_PTR")
EXPORTS = ("gx_open", "gx_close", "gx_last_error", "gx_create_map", "gx_update_map", "gx_read_map",
           "gx_ringbuf_drain", "gx_load_prog", "gx_verify", "gx_verify_offline", "gx_jit_offline", "gx_attach", "gx_run_batch", "gx_run_batch_ex", "gx_run_batch_host",
           "gx_get_stats", "gx_exec_info", "gx_set_engine", "gx_get_engine", "gx_merge_snapshot", "gx_merge_words", "gx_merge_export", "gx_merge_apply",
           "gx_hash_export", "gx_hash_apply", "gx_prefetch_drain", "gx_daemon_start", "gx_daemon_stop", "gx_daemon_watch",
           "gx_snapshot_read", "gx_daemon_get_stats", "gx_daemon_prefetch_range", "gx_instrument",
           "gx_kernel_launch", "gx_kernel_free", "gx_sched_run", "gx_sched_run_ex", "gx_comm_unique_id", "gx_comm_init",
           "gx_comm_init_host", "gx_merge", "gx_comm_free", "gx_region_map")


class gx_map_spec(C.Structure):
    _fields_ = [("type", C.c_uint32), ("key_size", C.c_uint32), ("value_size", C.c_uint32),
                ("max_entries", C.c_uint32), ("flags", C.c_uint32)]


class gx_verify_opts(C.Structure):
    _fields_ = [("simt_strict", C.c_uint32), ("max_insns", C.c_uint32), ("max_helpers", C.c_uint32),
                ("max_memops", C.c_uint32), ("complexity_limit", C.c_uint32)]


class gx_verify_report(C.Structure):
    _fields_ = [("verdict", C.c_int32), ("n_violations", C.c_uint32), ("first_insn", C.c_uint32),
                ("first_rule", C.c_uint32), ("worst_insns", C.c_uint64), ("worst_helpers", C.c_uint64),
                ("worst_memops", C.c_uint64), ("processed_insns", C.c_uint64), ("stack_depth", C.c_uint32),
                ("all_uniform", C.c_uint32), ("commutative", C.c_uint32), ("n_insns", C.c_uint32),
                ("image_insns", C.c_uint32), ("reserved", C.c_uint32)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["rule"] = RULES[self.first_rule] if self.first_rule < len(RULES) else "?"
        return d


class gx_batch_stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("events_run", "events_skipped", "divergent_steps", "helper_errors",
                                          "ringbuf_bytes", "ringbuf_drops", "hash_full", "warp_steps",
                                          "bounds_violations")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class gx_daemon_stats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("batches", "requests", "snapshots", "backpressure", "managed_prefetches")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# void handler(void *user, int map_fd, const uint64_t *reqs, uint64_t n_req)
PREFETCH_HANDLER = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.c_uint64)

_lib = None


def lib():
    """Loads libgx.so; raises (no fallback) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2512_12615_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, u32, u64, p64 = C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint64)
    sig = {
        "gx_open": (i32, [i32, C.POINTER(vp)]),
        "gx_close": (None, [vp]),
        "gx_last_error": (C.c_char_p, [vp]),
        "gx_create_map": (i32, [vp, C.POINTER(gx_map_spec), C.POINTER(i32)]),
        "gx_update_map": (i32, [vp, i32, vp, vp, u64, u64]),
        "gx_read_map": (i32, [vp, i32, vp, vp, u64, p64]),
        "gx_ringbuf_drain": (i32, [vp, i32, vp, u64, p64]),
        "gx_prefetch_drain": (i32, [vp, i32, p64, u64, p64]),
        "gx_daemon_start": (i32, [vp, PREFETCH_HANDLER, vp]),
        "gx_daemon_stop": (i32, [vp]),
        "gx_daemon_watch": (i32, [vp, i32]),
        "gx_snapshot_read": (i32, [vp, i32, vp, u64, p64]),
        "gx_daemon_get_stats": (i32, [vp, C.POINTER(gx_daemon_stats)]),
        "gx_daemon_prefetch_range": (i32, [vp, vp, u64]),
        "gx_instrument": (i32, [vp, i32, C.c_char_p, C.POINTER(vp), C.c_char_p, u64]),
        "gx_kernel_launch": (i32, [vp, vp, C.c_char_p, C.POINTER(u32), C.POINTER(u32), u32, C.POINTER(vp), vp]),
        "gx_kernel_free": (None, [vp, vp]),
        "gx_sched_run": (i32, [vp, i32, u32, C.POINTER(u32), C.POINTER(u32), u32, u32, C.POINTER(u32),
                               C.POINTER(C.c_uint8), p64, p64, C.POINTER(u32), p64]),
        "gx_sched_run_ex": (i32, [vp, i32, u32, u32, C.POINTER(u32), C.POINTER(u32), u32, u32, u32, C.POINTER(u32),
                                  C.POINTER(C.c_uint8), p64, p64, C.POINTER(u32), p64, vp, u64, p64]),
        "gx_load_prog": (i32, [vp, u32, vp, u32, C.POINTER(i32)]),
        "gx_region_map": (i32, [vp, vp, u64, C.POINTER(i32)]),
        "gx_verify": (i32, [vp, i32, C.POINTER(gx_verify_opts), C.POINTER(gx_verify_report), C.c_char_p, u64]),
        "gx_verify_offline": (i32, [vp, u32, vp, u32, C.POINTER(gx_verify_opts), C.POINTER(gx_verify_report),
                                    C.c_char_p, u64]),
        "gx_jit_offline": (i32, [vp, u32, vp, u32, C.c_char_p, u64, C.c_char_p, u64]),
        "gx_set_engine": (i32, [vp, i32]),
        "gx_get_engine": (i32, [vp]),
        "gx_attach": (i32, [vp, i32, u32, u32]),
        "gx_run_batch": (i32, [vp, vp, u64, i32, vp, vp]),
        "gx_run_batch_ex": (i32, [vp, vp, u64, i32, vp, vp, u32]),
        "gx_run_batch_host": (i32, [vp, vp, u64, i32, vp]),
        "gx_get_stats": (i32, [vp, C.POINTER(gx_batch_stats)]),
        "gx_exec_info": (i32, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32), p64]),
        "gx_merge_snapshot": (i32, [vp, i32]),
        "gx_merge_words": (i32, [vp, i32, p64]),
        "gx_merge_export": (i32, [vp, i32, vp, vp]),
        "gx_merge_apply": (i32, [vp, i32, vp, vp]),
        "gx_hash_export": (i32, [vp, i32, u32, C.c_int32, vp, vp, u64, p64]),
        "gx_hash_apply": (i32, [vp, i32, vp, vp, u64, u32, vp]),
        "gx_comm_unique_id": (i32, [vp]),
        "gx_comm_init": (i32, [vp, vp, i32, i32]),
        "gx_comm_init_host": (i32, [vp, C.POINTER(gx_comm_host_ops), i32, i32]),
        "gx_merge": (i32, [vp, vp]),
        "gx_comm_free": (i32, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class GxError(OSError):
    pass


# gx_comm_host_ops (include/gx.h): host-buffer transport callbacks of gx_merge
ALLREDUCE_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64)
ALLTOALLV_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p,
                           C.POINTER(C.c_uint64), C.POINTER(C.c_uint64))
ALLGATHER_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)


class gx_comm_host_ops(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_sum_u64", ALLREDUCE_CB), ("alltoallv", ALLTOALLV_CB),
                ("allgather", ALLGATHER_CB)]


def _check(rc, what, rt=None):
    if rc < 0:
        msg = lib().gx_last_error(rt).decode(errors="replace") if rt else ""
        raise GxError(-rc, f"{what}: {errno.errorcode.get(-rc, -rc)} {msg}")
    return rc


# ---------------------------------------------------------------- same-name thin wrappers

def gx_open(device: int = 0):
    h = C.c_void_p()
    _check(lib().gx_open(device, C.byref(h)), "gx_open (needs an sm_100 device)")
    return h


def gx_close(rt):
    lib().gx_close(rt)


def gx_create_map(rt, type, key_size, value_size, max_entries, flags=0) -> int:
    fd = C.c_int()
    spec = gx_map_spec(type, key_size, value_size, max_entries, flags)
    _check(lib().gx_create_map(rt, C.byref(spec), C.byref(fd)), "gx_create_map", rt)
    return fd.value


def gx_region_map(rt, base: int, length: int) -> int:
    fd = C.c_int()
    _check(lib().gx_region_map(rt, C.c_void_p(base), length, C.byref(fd)), "gx_region_map", rt)
    return fd.value


def gx_update_map(rt, fd, keys: bytes, vals: bytes, n: int, flags=0) -> int:
    return lib().gx_update_map(rt, fd, keys, vals, n, flags)


def gx_load_prog(rt, hook: int, slots: bytes) -> int:
    fd = C.c_int()
    _check(lib().gx_load_prog(rt, hook, slots, len(slots) // 8, C.byref(fd)), "gx_load_prog", rt)
    return fd.value


def gx_verify(rt, prog_fd, strict=False, max_insns=0, max_helpers=0, max_memops=0, complexity_limit=0):
    """Returns (verdict, report dict, log text).  Never raises on rejection."""
    opts = gx_verify_opts(1 if strict else 0, max_insns, max_helpers, max_memops, complexity_limit)
    rep = gx_verify_report()
    log = C.create_string_buffer(1 << 16)
    v = lib().gx_verify(rt, prog_fd, C.byref(opts), C.byref(rep), log, len(log))
    return v, rep.as_dict(), log.value.decode(errors="replace")


def gx_verify_offline(slots: bytes, maps: dict, strict=False, max_insns=0, max_helpers=0, max_memops=0,
                      complexity_limit=0):
    """Verifier without a device.  maps: {fd: (type, key_size, value_size, max_entries)}.
    Returns (verdict, report dict, log text)."""
    n = max(maps) + 1 if maps else 0
    arr = (gx_map_spec * max(n, 1))()
    for fd, (t, ks, vs, me) in maps.items():
        arr[fd] = gx_map_spec(t, ks, vs, me, 0)
    opts = gx_verify_opts(1 if strict else 0, max_insns, max_helpers, max_memops, complexity_limit)
    rep = gx_verify_report()
    log = C.create_string_buffer(1 << 16)
    v = lib().gx_verify_offline(slots, len(slots) // 8, arr, n, C.byref(opts), C.byref(rep), log, len(log))
    return v, rep.as_dict(), log.value.decode(errors="replace")


def gx_jit_offline(slots: bytes, maps: dict):
    """Generates + NVRTC-compiles the JIT kernel of one program without a device.
    Returns (rc, generated source, compiler log)."""
    n = max(maps) + 1 if maps else 0
    arr = (gx_map_spec * max(n, 1))()
    for fd, (t, ks, vs, me) in maps.items():
        arr[fd] = gx_map_spec(t, ks, vs, me, 0)
    src = C.create_string_buffer(1 << 20)
    log = C.create_string_buffer(1 << 16)
    rc = lib().gx_jit_offline(slots, len(slots) // 8, arr, n, src, len(src), log, len(log))
    return rc, src.value.decode(errors="replace"), log.value.decode(errors="replace")


GX_ENGINE_INTERP, GX_ENGINE_JIT = 0, 1


def gx_set_engine(rt, engine):
    _check(lib().gx_set_engine(rt, engine), "gx_set_engine", rt)


def gx_get_engine(rt) -> int:
    return lib().gx_get_engine(rt)


def gx_attach(rt, prog_fd, kind, tenant):
    _check(lib().gx_attach(rt, prog_fd, kind, tenant), "gx_attach", rt)


def _stream_handle(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


GX_RUN_OVERLAP = 1


def gx_run_batch(rt, events, n=None, prog_fd=-1, ret=None, stream=None, flags=0):
    """events: torch.uint8 CUDA tensor (N, 32) (or a raw device pointer with n); ret: u64 tensor or None.
    flags: 0, or GX_RUN_OVERLAP (gx_run_batch_ex: programmatic dependent launch; include/gx.h)."""
    if hasattr(events, "data_ptr"):
        n = events.shape[0] if n is None else n
        ptr = events.data_ptr()
    else:
        ptr = events
    rptr = ret.data_ptr() if ret is not None else None
    if flags:
        _check(lib().gx_run_batch_ex(rt, ptr, n, prog_fd, rptr, _stream_handle(stream), flags), "gx_run_batch_ex", rt)
    else:
        _check(lib().gx_run_batch(rt, ptr, n, prog_fd, rptr, _stream_handle(stream)), "gx_run_batch", rt)


def gx_run_batch_ex(rt, events, n=None, prog_fd=-1, ret=None, stream=None, flags=0):
    """gx_run_batch with launch flags (GX_RUN_OVERLAP)."""
    gx_run_batch(rt, events, n=n, prog_fd=prog_fd, ret=ret, stream=stream, flags=flags)


def gx_run_batch_host(rt, events: np.ndarray | int, n=None, prog_fd=-1, ret=None):
    """events: host array (numpy / pinned torch tensor) of N x 32 B; ret: host u64 array or None."""
    if hasattr(events, "data_ptr"):
        n = events.shape[0] if n is None else n
        ptr = events.data_ptr()
    elif isinstance(events, np.ndarray):
        n = len(events) if n is None else n
        ptr = events.ctypes.data
    else:
        ptr = events
    rptr = None
    if ret is not None:
        rptr = ret.data_ptr() if hasattr(ret, "data_ptr") else ret.ctypes.data
    _check(lib().gx_run_batch_host(rt, ptr, n, prog_fd, rptr), "gx_run_batch_host", rt)


def gx_get_stats(rt) -> dict:
    s = gx_batch_stats()
    _check(lib().gx_get_stats(rt, C.byref(s)), "gx_get_stats", rt)
    return s.as_dict()


def gx_exec_info(rt) -> dict:
    g, b, s, n = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
    _check(lib().gx_exec_info(rt, C.byref(g), C.byref(b), C.byref(s), C.byref(n)), "gx_exec_info", rt)
    return {"grid": g.value, "block": b.value, "smem": s.value, "launches": n.value}


def gx_read_map(rt, fd, spec):
    """Canonical content: ARRAY/PERTHREAD -> bytes (max_entries*value_size); HASH -> sorted (key, value) list."""
    type_, ks, vs, me = spec
    n = C.c_uint64()
    if type_ == GX_MAP_HASH:
        keys = C.create_string_buffer(ks * me + 8)
        vals = C.create_string_buffer(vs * me + 8)
        _check(lib().gx_read_map(rt, fd, keys, vals, me, C.byref(n)), "gx_read_map", rt)
        kr, vr = keys.raw, vals.raw   # .raw copies the whole buffer: take it once
        return [(int.from_bytes(kr[i * ks:(i + 1) * ks], "little"), vr[i * vs:(i + 1) * vs])
                for i in range(n.value)]
    vals = C.create_string_buffer(vs * me)
    _check(lib().gx_read_map(rt, fd, None, vals, me, C.byref(n)), "gx_read_map", rt)
    return vals.raw


def gx_prefetch_drain(rt, fd, cap) -> list[tuple[int, int]]:
    """Drains a prefetch queue: [(first_page, npages)] in queue order."""
    buf = (C.c_uint64 * (2 * cap + 2))()
    n = C.c_uint64()
    _check(lib().gx_prefetch_drain(rt, fd, buf, cap, C.byref(n)), "gx_prefetch_drain", rt)
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)]


def gx_daemon_start(rt, handler=None):
    """handler(map_fd, [(first_page, npages)]) in Python, or None for the default handler.
    Returns the ctypes callback object (keep it alive while the daemon runs)."""
    if handler is None:
        cb = C.cast(None, PREFETCH_HANDLER)
    else:
        def _tramp(user, fd, reqs, n):
            handler(int(fd), [(int(reqs[2 * i]), int(reqs[2 * i + 1]) & 0xFFFFFFFF) for i in range(n)])
        cb = PREFETCH_HANDLER(_tramp)
    _check(lib().gx_daemon_start(rt, cb, None), "gx_daemon_start", rt)
    return cb


def gx_daemon_stop(rt):
    _check(lib().gx_daemon_stop(rt), "gx_daemon_stop", rt)


def gx_daemon_watch(rt, fd):
    _check(lib().gx_daemon_watch(rt, fd), "gx_daemon_watch", rt)


def gx_snapshot_read(rt, fd, nbytes):
    """(bytes or None, version) of the latest published snapshot of a watched map."""
    buf = C.create_string_buffer(max(nbytes, 1))
    ver = C.c_uint64()
    _check(lib().gx_snapshot_read(rt, fd, buf, nbytes, C.byref(ver)), "gx_snapshot_read", rt)
    return (buf.raw[:nbytes] if ver.value else None), ver.value


def gx_daemon_get_stats(rt) -> dict:
    st = gx_daemon_stats()
    _check(lib().gx_daemon_get_stats(rt, C.byref(st)), "gx_daemon_get_stats", rt)
    return st.as_dict()


def gx_daemon_prefetch_range(rt, ptr, nbytes):
    _check(lib().gx_daemon_prefetch_range(rt, ptr, nbytes), "gx_daemon_prefetch_range", rt)


def gx_instrument(rt, prog_fd, user_src: str):
    """f4: the verified program as inline device hooks linked into user_src; returns a handle."""
    h = C.c_void_p()
    log = C.create_string_buffer(1 << 16)
    _check(lib().gx_instrument(rt, prog_fd, user_src.encode(), C.byref(h), log, len(log)), "gx_instrument", rt)
    return h


def gx_kernel_launch(rt, handle, name: str, grid, block, args, smem=0, stream=None):
    """args: torch tensors (passed as device pointers), Python ints (u64) or ctypes values."""
    keep = []
    for a in args:
        if hasattr(a, "data_ptr"):
            keep.append(C.c_void_p(a.data_ptr()))
        elif isinstance(a, int):
            keep.append(C.c_uint64(a))
        else:
            keep.append(a)
    argv = (C.c_void_p * max(len(keep), 1))(*[C.cast(C.pointer(k), C.c_void_p) for k in keep])
    g = (C.c_uint32 * 3)(*(list(grid) + [1, 1, 1])[:3])
    b = (C.c_uint32 * 3)(*(list(block) + [1, 1, 1])[:3])
    _check(lib().gx_kernel_launch(rt, handle, name.encode(), g, b, smem, argv, _stream_handle(stream)),
           "gx_kernel_launch", rt)


def gx_sched_run(rt, prog_fd, cost_us, home, n_workers, steal_cost_us=0) -> dict:
    """f3: the work-stealing block scheduler on the GPU with the policy prog_fd (include/gx.h)."""
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
    _check(lib().gx_sched_run(rt, prog_fd, U, P(cost, C.c_uint32), P(hm, C.c_uint32), n_workers, steal_cost_us,
                              P(ex, C.c_uint32), P(st, C.c_uint8), P(busy, C.c_uint64), P(end, C.c_uint64),
                              P(steals, C.c_uint32), C.byref(ms)), "gx_sched_run", rt)
    return dict(executed_by=ex, stolen=st, busy_ns=busy, end_ns=end, steals=steals, makespan_ns=ms.value)


GX_SCHED_CLC, GX_SCHED_PROBES = 1, 2
# gx_hook_log (include/gx.h): the 32-B record, R0, worker, the worker's hook sequence number
HOOK_LOG = np.dtype([("rec", np.uint8, 32), ("r0", np.uint64), ("worker", np.uint32), ("seq", np.uint32)])


def gx_sched_run_ex(rt, prog_fd, cost_us, home=None, n_workers=0, steal_cost_us=0, flags=0, smem_per_block=0,
                    log_cap=0) -> dict:
    """f3: gx_sched_run with modes (GX_SCHED_CLC: one block per unit, steals by cluster launch
    control; GX_SCHED_PROBES) and a hook log (include/gx.h).  Returns gx_sched_run's dict plus
    'log' (HOOK_LOG records, completion order) and 'log_n'."""
    cost = np.ascontiguousarray(cost_us, dtype=np.uint32)
    U = len(cost)
    hm = None if home is None else np.ascontiguousarray(home, dtype=np.uint32)
    W = U if flags & GX_SCHED_CLC else n_workers
    ex = np.zeros(U, dtype=np.uint32)
    st = np.zeros(U, dtype=np.uint8)
    busy = np.zeros(W, dtype=np.uint64)
    end = np.zeros(W, dtype=np.uint64)
    steals = np.zeros(W, dtype=np.uint32)
    log = np.zeros(log_cap, dtype=HOOK_LOG)
    ms, ln = C.c_uint64(), C.c_uint64()
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    _check(lib().gx_sched_run_ex(rt, prog_fd, flags, U, P(cost, C.c_uint32),
                                 None if hm is None else P(hm, C.c_uint32), n_workers, steal_cost_us, smem_per_block,
                                 P(ex, C.c_uint32), P(st, C.c_uint8), P(busy, C.c_uint64), P(end, C.c_uint64),
                                 P(steals, C.c_uint32), C.byref(ms), log.ctypes.data if log_cap else None, log_cap,
                                 C.byref(ln)), "gx_sched_run_ex", rt)
    return dict(executed_by=ex, stolen=st, busy_ns=busy, end_ns=end, steals=steals, makespan_ns=ms.value,
                log=log[:min(ln.value, log_cap)], log_n=ln.value)


def gx_kernel_free(rt, handle):
    lib().gx_kernel_free(rt, handle)


def gx_ringbuf_drain(rt, fd) -> list[bytes]:
    """Drains a ring buffer; returns the record payloads in buffer order."""
    n = C.c_uint64()
    rc = lib().gx_ringbuf_drain(rt, fd, None, 0, C.byref(n))
    if rc < 0 and -rc != errno.E2BIG:
        _check(rc, "gx_ringbuf_drain", rt)
    buf = C.create_string_buffer(max(n.value, 1))
    _check(lib().gx_ringbuf_drain(rt, fd, buf, n.value, C.byref(n)), "gx_ringbuf_drain", rt)
    raw, out, o = buf.raw[: n.value], [], 0
    while o + 8 <= len(raw):
        ln = int.from_bytes(raw[o:o + 4], "little")
        out.append(raw[o + 8:o + 8 + ln])
        o += (8 + ln + 7) & ~7
    return out


def gx_merge_snapshot(rt, fd):
    _check(lib().gx_merge_snapshot(rt, fd), "gx_merge_snapshot", rt)


def gx_merge_words(rt, fd) -> int:
    w = C.c_uint64()
    _check(lib().gx_merge_words(rt, fd, C.byref(w)), "gx_merge_words", rt)
    return w.value


def gx_merge_export(rt, fd, delta, stream=None):
    _check(lib().gx_merge_export(rt, fd, delta.data_ptr(), _stream_handle(stream)), "gx_merge_export", rt)


def gx_merge_apply(rt, fd, total, stream=None):
    _check(lib().gx_merge_apply(rt, fd, total.data_ptr(), _stream_handle(stream)), "gx_merge_apply", rt)


def gx_hash_export(rt, fd, keys, vals, nranks=1, owner=-1):
    """Fills keys/vals (u64 device tensors) grouped by owner; returns the per-owner counts."""
    counts = (C.c_uint64 * nranks)()
    _check(lib().gx_hash_export(rt, fd, nranks, owner, keys.data_ptr(), vals.data_ptr(), keys.numel(), counts),
           "gx_hash_export", rt)
    return list(counts)


GX_MERGE_RESTORE, GX_MERGE_COMMIT = 1, 2


def gx_hash_apply(rt, fd, keys, vals, n, flags=GX_MERGE_RESTORE | GX_MERGE_COMMIT, stream=None):
    _check(lib().gx_hash_apply(rt, fd, keys.data_ptr() if n else None, vals.data_ptr() if n else None, n, flags,
                               _stream_handle(stream)), "gx_hash_apply", rt)


def gx_comm_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for gx_comm_init (rank 0 makes it, the caller ships it)."""
    buf = C.create_string_buffer(128)
    _check(lib().gx_comm_unique_id(buf), "gx_comm_unique_id")
    return buf.raw


def gx_comm_init(rt, unique_id: bytes, nranks: int, rank: int):
    _check(lib().gx_comm_init(rt, unique_id, nranks, rank), "gx_comm_init", rt)


def gx_comm_init_host(rt, allreduce_sum_u64, alltoallv, allgather, nranks: int, rank: int):
    """Host-buffer transport: the three callables get numpy views of the library's host staging
    buffers (uint64 words for the all-reduce, uint8 bytes otherwise) and must fill them in place:
        allreduce_sum_u64(buf_u64)                          -- in-place SUM over ranks
        alltoallv(send_u8, send_bytes, send_off, recv_u8, recv_bytes, recv_off)
        allgather(send_u8, recv_u8)                          -- recv = concat over ranks
    Returns the ctypes object that must stay alive as long as the runtime merges."""
    def ar(user, buf, n):
        try:
            allreduce_sum_u64(np.ctypeslib.as_array(buf, shape=(n,)))
            return 0
        except Exception:
            return -errno.EIO

    def a2a(user, send, sb, so, recv, rb, ro):
        try:
            G = nranks
            sbv, sov = np.ctypeslib.as_array(sb, shape=(G,)).copy(), np.ctypeslib.as_array(so, shape=(G,)).copy()
            rbv, rov = np.ctypeslib.as_array(rb, shape=(G,)).copy(), np.ctypeslib.as_array(ro, shape=(G,)).copy()
            ns = int((sov + sbv).max()) if G else 0
            nr = int((rov + rbv).max()) if G else 0
            sa = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(max(ns, 1),)) if ns else np.zeros(0, np.uint8)
            ra = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), shape=(max(nr, 1),)) if nr else np.zeros(0, np.uint8)
            alltoallv(sa, sbv, sov, ra, rbv, rov)
            return 0
        except Exception:
            return -errno.EIO

    def ag(user, send, recv, nbytes):
        try:
            sa = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(nbytes,))
            ra = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), shape=(nbytes * nranks,))
            allgather(sa, ra)
            return 0
        except Exception:
            return -errno.EIO

    ops = gx_comm_host_ops(None, ALLREDUCE_CB(ar), ALLTOALLV_CB(a2a), ALLGATHER_CB(ag))
    _check(lib().gx_comm_init_host(rt, C.byref(ops), nranks, rank), "gx_comm_init_host", rt)
    return ops


def gx_merge(rt, stream=None):
    """Collective S3 merge of every map over the communicator's ranks (include/gx.h)."""
    _check(lib().gx_merge(rt, _stream_handle(stream)), "gx_merge", rt)


def gx_comm_free(rt):
    _check(lib().gx_comm_free(rt), "gx_comm_free", rt)


# ---------------------------------------------------------------- engine object

class Runtime:
    """One gx_rt.  Engine interface for gxin.configs.setup plus run / read helpers."""

    def __init__(self, device: int = 0, strict: bool = False, engine: int | None = None):
        self.rt = gx_open(device)
        if engine is not None:
            gx_set_engine(self.rt, engine)
        self.device = device
        self.strict = strict
        self.specs = {}
        self.reports = {}

    def close(self):
        if self.rt:
            gx_close(self.rt)
            self.rt = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # engine interface
    def create_map(self, type, key_size, value_size, max_entries) -> int:
        fd = gx_create_map(self.rt, type, key_size, value_size, max_entries)
        self.specs[fd] = (type, key_size, value_size, max_entries)
        return fd

    def region_map(self, base: int, length: int) -> int:
        """gx_region_map: caller-owned device memory [base, base + length) for gdev_prefetch_l2."""
        fd = gx_region_map(self.rt, base, length)
        self.specs[fd] = (GX_MAP_REGION, 0, 0, 1)
        return fd

    def update_map(self, fd, key: bytes, val: bytes, flags=0) -> int:
        return gx_update_map(self.rt, fd, key, val, 1, flags)

    def update_many(self, fd, keys: bytes, vals: bytes, n: int, flags=0) -> int:
        return gx_update_map(self.rt, fd, keys, vals, n, flags)

    def load_prog(self, slots: bytes, hook: int = 0) -> int:
        """load + verify; raises GxError on rejection (the report is kept in .reports)."""
        fd = gx_load_prog(self.rt, hook, slots)
        v, rep, log = gx_verify(self.rt, fd, strict=self.strict)
        self.reports[fd] = (v, rep, log)
        if v != 0:
            raise GxError(-v, f"verifier rejected program: {rep['rule']} at insn {rep['first_insn']}\n{log}")
        return fd

    def attach(self, prog, kind, tenant):
        gx_attach(self.rt, prog, kind, tenant)

    # execution
    def run(self, events, prog=-1, ret=None, stream=None, overlap=False):
        gx_run_batch(self.rt, events, prog_fd=prog, ret=ret, stream=stream, flags=GX_RUN_OVERLAP if overlap else 0)

    def stats(self) -> dict:
        return gx_get_stats(self.rt)

    # reads
    def dump(self, fd) -> bytes:
        spec = self.specs[fd]
        if spec[0] == GX_MAP_HASH:
            return b"".join(k.to_bytes(spec[1], "little") + v for k, v in gx_read_map(self.rt, fd, spec))
        return gx_read_map(self.rt, fd, spec)

    def array_u64(self, fd) -> np.ndarray:
        return np.frombuffer(self.dump(fd), dtype=np.uint64)

    def hash_items(self, fd) -> dict:
        return {k: np.frombuffer(v, dtype=np.uint64).copy() for k, v in gx_read_map(self.rt, fd, self.specs[fd])}

    def prefetch_requests(self, fd) -> list[tuple[int, int]]:
        """Drains a prefetch queue; returns its canonical content, the sorted SET of requests
        (F-2)."""
        return sorted(set(gx_prefetch_drain(self.rt, fd, self.specs[fd][3])))

    def daemon_start(self, handler=None):
        self._daemon_cb = gx_daemon_start(self.rt, handler)

    def daemon_stop(self):
        gx_daemon_stop(self.rt)
        self._daemon_cb = None

    def ringbuf_records(self, fd) -> list[bytes]:
        """Drains; returns the multiset as a sorted list of payloads."""
        return sorted(gx_ringbuf_drain(self.rt, fd))


def gx_last_error(rt) -> str:
    return lib().gx_last_error(rt).decode(errors="replace")
