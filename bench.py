#!/usr/bin/env python
"""bench.py -- device-side eBPF event throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Workload (BASELINE.json configs[1]): the per-SM / per-warp memory-access
histogram policy P2 (ARRAY 9472 x u64 with a record-uniform ATOMIC ADD + a per-thread ARRAY of
{cnt, bytes} updated by plain RMW) over 2^30 synthetic access events (32 GiB) per GPU.  A step is
one gx_run_batch over the whole batch (every §8a row the config exercises: ingest, staging,
interpretation, array / per-thread helpers, warp-aggregated atomics, epilogue); with N > 1 it
also includes the NCCL snapshot-and-merge of the maps (weak scaling: 2^30 events per GPU).
Inputs are generated on the device before timing and are larger than L2 (no flush needed).

One JSON line on rank 0 (keys per the driver contract + roofline / cpu_baseline / e2e / clocks).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "policy events/sec (device-timed)"
EVENT_BYTES = 32


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="C2")
    p.add_argument("--events", type=int, default=0, help="events per GPU (default: the config's size)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-c1", action="store_true", help="skip the C1 (1M-event counter) section")
    p.add_argument("--extra", action="store_true", help="also time C1/C3/C4 single-GPU lines (stderr)")
    p.add_argument("--no-configs", action="store_true",
                   help="skip the per-config records (C1-C5 at N=1; C4 strong / C5 weak scaling with gx_merge at N>1)")
    p.add_argument("--engine", default="jit", choices=["jit", "interp"],
                   help="headline engine (the other one is timed too and reported under 'engines')")
    return p.parse_args()


DEFAULT_EVENTS = {"C1": 1 << 20, "C1d": 1 << 20, "C2": 1 << 30, "C3": 1 << 28, "C4": 1 << 31, "C5": 1 << 28}
WORKLOAD = {
    "C1": "counter policy P1 (13-insn ARRAY lookup + atomic add, 256 keys)",
    "C1d": "counter policy P1d (8-insn direct-value ARRAY atomic add, 256 keys)",
    "C2": "per-SM/per-warp access histogram P2 (ARRAY 9472 + per-thread ARRAY) over 2^30 access events",
    "C3": "LLM page trace -> LFU hash (1M entries, FETCH-ADD) + ringbuf on threshold 64",
    "C4": "vector-search stream, 12-iteration bounded binary search + hash/array/per-thread helpers",
    "C5": "multi-tenant mix P1/P2/P3'/P4 via the attach table",
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def _run(self):
        """one nvidia-smi in loop mode (-lms 20) for the whole region: a sample every ~20 ms"""
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "20"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            for line in self._p.stdout:
                f = [x.strip() for x in line.strip().split(",")]
                if len(f) >= 7:
                    self.samples.append(f)
                if self._stop.is_set():
                    break
        except Exception:
            pass

    def __enter__(self):
        self._p = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)   # let the first sample land before the timed region starts
        return self

    def __exit__(self, *a):
        time.sleep(0.05)
        self._stop.set()
        if self._p is not None:
            self._p.terminate()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        busy = [float(s[0]) for s in self.samples if s[6].isdigit() and int(s[6]) > 50] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(busy)) if busy else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_rate(config, seed, n_total, budget_s=12.0):
    """The CPU oracle (as it stands, one host core) on a bounded prefix sample of the workload.
    Only interpretation is timed (SURVEY.md §8d CPU oracle timing)."""
    from gxin import configs
    from oracle.oracle import Oracle
    env = Oracle()
    s = configs.setup(env, config)
    done, t_used, chunk, i0 = 0, 0.0, 1 << 16, 0
    while t_used < budget_s and i0 < n_total:
        n = min(chunk, n_total - i0)
        ev = configs.events(config, seed, n, i0, n_total)
        t0 = time.perf_counter()
        env.run(ev, s.prog_arg, index_base=i0, want_r0=False)
        t_used += time.perf_counter() - t0
        done += n
        i0 += n
        chunk = min(chunk * 2, 1 << 20)
    return done / t_used, done, t_used


def _oracle_worker(a):
    config, seed, n_total, i0, budget_s = a
    from gxin import configs
    from oracle.oracle import Oracle
    env = Oracle()
    s = configs.setup(env, config)
    done, t_used, n = 0, 0.0, 1 << 20
    while t_used < budget_s:
        ev = configs.events(config, seed, n, i0 + done, n_total)
        t0 = time.perf_counter()
        env.run(ev, s.prog_arg, index_base=i0 + done, want_r0=False)
        t_used += time.perf_counter() - t0
        done += n
    return done, t_used


def oracle_rate_allcores(config, seed, n_total, budget_s=10.0):
    """The same oracle on every host core at once: one process per core on disjoint chunks of the
    stream (the per-event work is the same as the 1-core figure; no merge is timed)."""
    import multiprocessing as mproc
    cores = host_cores()
    span = n_total // cores // (1 << 20) * (1 << 20) or (1 << 20)
    with mproc.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_oracle_worker, [(config, seed, n_total, (k * span) % max(1, n_total - (1 << 22)), budget_s)
                                        for k in range(cores)])
    done = sum(d for d, _ in res)
    wall = max(t for _, t in res)
    return done / wall, done, cores


# SURVEY.md §8d roofline inputs per config: L2 atomics per event the method cannot avoid (A_alg):
# C1 privatised (0); C2 one record-uniform ADD per 32-event record (the 74 KiB histogram is over the
# 16 KiB privatisation budget); C3 0.69 returning FETCH-ADDs per event (prefill records key-uniform,
# a decode record holds 29.2 distinct pages: DESIGN.md §6); C4 two record-near-uniform ADDs per
# record; C5 the tenant mix (40 % P1, 30 % P2, 20 % P3', 10 % P4).
A_ALG = {"C1": 0.0, "C2": 1 / 32, "C3": 0.69, "C4": 2 / 32,
         "C5": 0.3 * (1 / 32) + 0.2 * 0.69 + 0.1 * (2 / 32)}
CONFIG_EVENTS = {"C1": 1 << 26, "C2": 1 << 30, "C3": 1 << 28, "C4": 1 << 28, "C5": 1 << 28}


def atomic_rate():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "atomics_b200.json")))["atom_add_u64_random_per_s"]
    except Exception:
        return 1.257e11


def config_records(device, args):
    """One record per config (SURVEY.md §8d result fields): device time per batch, events/s, the three
    roofline components T_hbm / T_atom / T_alu with their fractions, and a parity verdict from this
    run (a 2^16-event sample against the oracle, bit-exact, plus the full batch's event count)."""
    import torch
    import paper_2512_12615_b200 as gx
    from gxin import configs, gen_gpu
    from oracle.oracle import Oracle
    peaks = measured_peaks()[0]
    r_atom = atomic_rate()
    out = {}
    for config, n in CONFIG_EVENTS.items():
        try:
            seed = configs.SEEDS[config]
            # parity sample: the oracle and the CUDA path on the same 2^16 events
            ns = 1 << 16
            evs = configs.events(config, seed, ns)
            env = Oracle()
            so = configs.setup(env, config)
            r0o = env.run(evs, so.prog_arg)
            ost = env.stats()
            rts = gx.Runtime(device, engine=gx.GX_ENGINE_JIT)
            sg = configs.setup(rts, config)
            ret = torch.zeros(ns, dtype=torch.int64, device="cuda")
            rts.run(torch.from_numpy(evs.view(np.uint8).reshape(-1, 32)).cuda(), sg.prog_arg, ret=ret)
            torch.cuda.synchronize()
            same = bool((ret.cpu().numpy().view(np.uint64) == r0o).all())
            for key, fd in so.fds.items():
                if env.specs[fd][0] == 27:
                    same &= env.ringbuf_records(fd) == rts.ringbuf_records(sg.fds[key])
                else:
                    same &= env.dump(fd) == rts.dump(sg.fds[key])
            rts.close()
            insns = ost["insns"] / max(1, ost["events_run"])
            # the timed batch: warm maps, 3 + 5 launches
            rt = gx.Runtime(device, engine=gx.GX_ENGINE_JIT)
            s = configs.setup(rt, config)
            ev = gen_gpu.generate_device(config, seed, n, device=device)
            for _ in range(3):
                rt.run(ev, s.prog_arg)
            st0 = rt.stats()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                rt.run(ev, s.prog_arg)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            st = rt.stats()
            run_ok = st["events_run"] + st["events_skipped"] == 5 * n
            rb = st["ringbuf_bytes"] / 5 / n
            t_hbm = n * (EVENT_BYTES + rb) / (peaks["hbm_gbs"] * 1e9) * 1e3
            t_atom = n * A_ALG[config] / r_atom * 1e3
            f_sm = 1965e6
            t_alu = n / 32 * (2 * insns) / (148 * 4 * f_sm) * 1e3
            comp = {"hbm": t_hbm, "atom": t_atom, "alu": t_alu}
            bound = max(comp, key=comp.get)
            out[config] = {"events": n, "ms": ms, "events_per_s": n / (ms / 1e3), "ns_per_event": ms * 1e6 / n,
                           "t_hbm_ms": t_hbm, "t_atom_ms": t_atom, "t_alu_ms": t_alu,
                           "frac_hbm": t_hbm / ms, "frac_atom": t_atom / ms, "frac_alu": t_alu / ms,
                           "bound": bound, "frac": comp[bound] / ms, "R_atom_per_s": r_atom, "A_alg": A_ALG[config],
                           "insns_per_event": insns, "f_sm_mhz": f_sm / 1e6,
                           "parity": ("exact" if same else "mismatch") + " (2^16-event sample vs oracle)",
                           "events_accounted": bool(run_ok), "ringbuf_drops": st["ringbuf_drops"],
                           "hash_full": st["hash_full"]}
            del ev
            rt.close()
        except Exception as exc:  # pragma: no cover - box-dependent
            out[config] = {"error": str(exc)[:200]}
    return out


def multi_records(device, rank, world, args):
    """N > 1: C4 strong scaling (2^31 events in total, 2^31/N per GPU)
    and C5 (the multi-tenant mix, 2^28 events per GPU, weak), each step = the batch + gx_merge of
    every map over the library's NCCL communicator; max over ranks of the device time."""
    import torch
    import torch.distributed as dist
    import paper_2512_12615_b200 as gx
    from gxin import configs, gen_gpu
    from paper_2512_12615_b200.dist import Merger
    out = {}
    for config, n_total, scaling in (("C4", 1 << 31, "strong"), ("C5", (1 << 28) * world, "weak")):
        n = n_total // world // 32 * 32
        rt = gx.Runtime(device, engine=gx.GX_ENGINE_JIT)
        s = configs.setup(rt, config)
        ev = gen_gpu.generate_device(config, configs.SEEDS[config], n, i0=rank * n, n_total=n_total, device=device)
        m = Merger(rt, dist.group.WORLD)
        for _ in range(2):
            rt.run(ev, s.prog_arg)
            m.merge()
        torch.cuda.synchronize()
        dist.barrier()
        a, b, mb = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        for k in range(5):
            rt.run(ev, s.prog_arg)
            if k == 4:
                mb.record()
            m.merge()
        b.record()
        torch.cuda.synchronize()
        dist.barrier()
        ms = torch.tensor([a.elapsed_time(b) / 5, mb.elapsed_time(b)], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        out[config] = {"scaling": scaling, "events_total_per_step": n * world, "events_per_gpu": n,
                       "ms_per_step": float(ms[0]), "events_per_s": n * world / (float(ms[0]) / 1e3),
                       "merge_ms": float(ms[1]), "steps": 5, "merge": "every step (gx_merge after each batch)"}
        del ev
        rt.close()
    return out


def run_reference(args, rank, world):
    """--impl reference: the oracle on the host cores, rank 0 only (the base contract's reference arm)."""
    if rank != 0:
        return
    from gxin import configs
    config = args.config
    n_total = (args.events or DEFAULT_EVENTS[config]) * max(1, args.gpus)
    seed = configs.SEEDS[config]
    rates = []
    for step in range(args.warmup + args.steps):
        r, done, t = oracle_rate(config, seed, n_total, budget_s=6.0)
        if step >= args.warmup:
            rates.append((r, done, t))
    value = float(np.median([r for r, _, _ in rates]))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median([t for _, _, t in rates]) * 1e3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": WORKLOAD[config], "config": config, "events_per_gpu": n_total // max(1, args.gpus),
                       "flush": "inputs larger than L2"},
            "cpu_baseline": {"value": value, "unit": "events/s", "cores": 1, "kind": "oracle",
                             "sample": f"prefix of {rates[0][1]} events per step of the {config} stream (seed {seed}), "
                                       f"interpretation only, {cpu_model()}"},
            "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2512_12615_b200 as gx
    from gxin import configs, gen_gpu

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    config = args.config
    n = args.events or DEFAULT_EVENTS[config]
    n_total = n * world
    seed = configs.SEEDS[config]
    stream = torch.cuda.current_stream()

    engine_id = gx.GX_ENGINE_JIT if args.engine == "jit" else gx.GX_ENGINE_INTERP
    rt = gx.Runtime(local, engine=engine_id)
    s = configs.setup(rt, config)
    events = gen_gpu.generate_device(config, seed, n, i0=rank * n, n_total=n_total, device=local)
    torch.cuda.synchronize()

    merger = None
    if world > 1:
        from paper_2512_12615_b200.dist import Merger
        merger = Merger(rt, dist.group.WORLD)   # gx_comm_init on the library's NCCL communicator

    def step():
        rt.run(events, s.prog_arg, stream=stream)
        if merger is not None:
            merger.merge()

    t_compile = time.perf_counter()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t_compile = time.perf_counter() - t_compile
    launches0 = gx.gx_exec_info(rt.rt)["launches"]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_launch = []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            rt.run(events, s.prog_arg, stream=stream)
            b.record(stream)
            per_launch.append((a, b))
            if merger is not None:
                merger.merge()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    t_ms = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in per_launch]))
    launches = gx.gx_exec_info(rt.rt)["launches"] - launches0
    value = n_total * args.steps / (t_ms / 1e3)
    st = rt.stats()

    peaks, peak_kind = measured_peaks()
    alg_bytes = EVENT_BYTES * n
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    # a read-only reference measured in this run (the peak above is a read+write copy; a pure read
    # stream has no write turnaround and can exceed it): torch's int64 sum over the same event bytes
    read_ref = None
    try:
        flat = events.view(-1).view(torch.int64)
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            with torch.cuda.stream(stream):
                flat.sum()
            b.record(stream)
            torch.cuda.synchronize()
            best = a.elapsed_time(b) if best is None else min(best, a.elapsed_time(b))
        read_ref = {"gbs": alg_bytes / (best / 1e3) / 1e9, "ms": best,
                    "how": "torch int64 sum over the same event batch (read-only), best of 3, CUDA events"}
    except Exception as exc:  # pragma: no cover - box-dependent
        read_ref = {"error": str(exc)[:120]}
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{config}_{args.engine}.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("dram_bytes_per_launch")
        except Exception:
            pass
    line = {
        "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (device-generated, seeded)",
        "config": {"workload": WORKLOAD[config], "config": config, "events_per_gpu": n,
                   "global_events": n_total, "flush": "inputs (32 B x events) larger than L2",
                   "parallelism": f"dp{world}" if world > 1 else "dp1"},
        "ns_per_event": t_ms * 1e6 / (n_total * args.steps) * world,
        "gpu_launches": int(launches),
        "engine": args.engine,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                     "frac": achieved / peaks.get("hbm_gbs", 6650.0), "traffic": traffic,
                     "kernel": "gx_jit_kernel" if args.engine == "jit" else "gx_exec_kernel",
                     "alg_bytes_per_launch": alg_bytes, "peak_kind": peak_kind, "kernel_ms": kernel_ms,
                     "peak_note": "MEASURED_PEAKS hbm_gbs is a read+write copy; a read-only stream can exceed it",
                     "read_only_reference": read_ref},
        "warmup_incl_jit_s": t_compile,
        "stats": {k: int(v) // max(1, args.steps + args.warmup) for k, v in st.items()},
        "clocks": clk.summary(),
    }

    # the other engine on the same events (same maps semantics; reported, not the headline)
    if world == 1:
        other = "interp" if args.engine == "jit" else "jit"
        gx.gx_set_engine(rt.rt, gx.GX_ENGINE_INTERP if other == "interp" else gx.GX_ENGINE_JIT)
        for _ in range(2):
            rt.run(events, s.prog_arg, stream=stream)
        a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            rt.run(events, s.prog_arg, stream=stream)
        b2.record(stream)
        torch.cuda.synchronize()
        oms = a.elapsed_time(b2) / args.steps
        line["engines"] = {other: {"value": n / (oms / 1e3), "kernel_ms": oms,
                                   "hbm_frac": EVENT_BYTES * n / (oms / 1e3) / 1e9 / peaks.get("hbm_gbs", 6650.0)}}
        gx.gx_set_engine(rt.rt, engine_id)
        rt.stats()

    # end-to-end through the public API from pinned host memory (H2D inside the timed region)
    if not args.no_e2e and rank == 0 or (not args.no_e2e and world > 1):
        try:
            line["e2e"] = e2e_measure(rt, s, events, n, n_total, world, args)
        except Exception as exc:  # pragma: no cover - box-dependent
            line["e2e"] = {"value": None, "unit": "events/s", "error": str(exc)[:200]}
    if rank == 0 and not args.no_cpu and world == 1:
        r, done, t = oracle_rate(config, seed, n_total)
        line["cpu_baseline"] = {"value": r, "unit": "events/s", "cores": 1, "kind": "oracle",
                                "sample": f"prefix of {done} events of the {config} stream (seed {seed}) in "
                                          f"{t:.1f} s, interpretation only; host has {host_cores()} cores, {cpu_model()}"}
        try:
            ra, dn, cores = oracle_rate_allcores(config, seed, n_total)
            line["cpu_baseline"]["all_cores"] = {
                "value": ra, "cores": cores, "sample": f"{dn} events: disjoint 2^20-event chunks of the same stream, "
                                                      f"one oracle process per core for ~10 s (interpretation only)"}
        except Exception as exc:  # pragma: no cover - host-dependent
            line["cpu_baseline"]["all_cores"] = {"error": str(exc)[:200]}
    if rank == 0 and world == 1 and not args.no_configs:
        line["configs"] = config_records(local, args)
    if world > 1 and not args.no_configs:
        multi = multi_records(local, rank, world, args)
        if rank == 0:
            line["multi"] = multi
    if rank == 0 and world == 1 and not args.no_c1:
        try:
            line["c1"] = c1_measure(local)
        except Exception as exc:  # pragma: no cover - box-dependent
            line["c1"] = {"error": str(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.extra:
            for fn in (lambda: extra_lines(rt, args), f2_lines, f2_l2_line, f4_lines, f3_lines):
                try:
                    fn()
                except Exception as exc:  # pragma: no cover - box-dependent; the headline is printed
                    print(json.dumps({"extra_error": repr(exc)[:300]}), file=sys.stderr, flush=True)
    if world > 1:
        dist.destroy_process_group()


def c1_measure(device):
    """BASELINE.json configs[0] / the north-star target: the counter policy over 2^20-event batches.
    8 distinct batches (256 MiB > L2) are rotated so every launch streams from HBM.  Reported both
    per single launch (CUDA events around each launch) and steady state (100 back-to-back launches
    captured in one CUDA graph, SURVEY.md §8d C1 timing protocol), the latter also with the
    launches chained by programmatic dependent launch (gx_run_batch_ex GX_RUN_OVERLAP: the batches
    are resident before the graph runs, which is that flag's contract)."""
    import torch
    import paper_2512_12615_b200 as gx
    from gxin import configs, gen_gpu
    peaks = measured_peaks()[0]
    out = {}
    n, nb = 1 << 20, 8
    for config in ("C1", "C1d"):
        rt = gx.Runtime(device, engine=gx.GX_ENGINE_JIT)
        s = configs.setup(rt, config)
        bufs = [gen_gpu.generate_device(config, configs.SEEDS[config], n, i0=k * n, n_total=nb * n, device=device)
                for k in range(nb)]
        stream = torch.cuda.Stream(device)
        with torch.cuda.stream(stream):
            for k in range(3 * nb):
                rt.run(bufs[k % nb], s.prog_arg, stream=stream)
            stream.synchronize()
            times = []
            for k in range(5 * nb):
                a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                rt.run(bufs[k % nb], s.prog_arg, stream=stream)
                b2.record(stream)
                times.append((a, b2))
            stream.synchronize()
            single = float(np.median([a.elapsed_time(b2) for a, b2 in times]))
            steady = {}
            for overlap in (False, True):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for k in range(100):
                        rt.run(bufs[k % nb], s.prog_arg, stream=stream, overlap=overlap)
                g.replay()
                stream.synchronize()
                a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(5):
                    g.replay()
                b2.record(stream)
                stream.synchronize()
                steady[overlap] = a.elapsed_time(b2) / 500
                del g
            # the single-launch floor, timed the same way over the same rotating batches: a program that
            # only reads each event's addr (the whole 32-B sector streams from HBM), and a plain torch
            # reduction over the batch bytes -- what one launch of any kernel reading 32 MiB costs here
            floors = {}
            rt_floor = gx.Runtime(device, engine=gx.GX_ENGINE_JIT)
            from gxin import asm
            # the addr must stay live (an unused load is dead code to the compiler): a never-taken
            # (addresses are 8-aligned) branch to a counter update keeps every event's read
            cfd = rt_floor.create_map(gx.GX_MAP_ARRAY, 4, 8, 1)
            pf = rt_floor.load_prog(asm.assemble(
                "ldxdw r2, [r1+0]\njne r2, 1, out\nstw [r10-4], 0\nlddw r1, map:c\nmov64 r2, r10\nadd64 r2, -4\n"
                "call 1\njeq r0, 0, out\nmov64 r1, 1\natomic_add64 [r0+0], r1\nout:\nmov64 r0, 0\nexit", {"c": cfd}))
            for name, fn in (("read_only_program", lambda b: rt_floor.run(b, pf, stream=stream)),
                             ("torch_sum", lambda b: b.view(torch.int64).sum())):
                for k in range(2 * nb):
                    fn(bufs[k % nb])
                stream.synchronize()
                ts = []
                for k in range(5 * nb):
                    a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    fn(bufs[k % nb])
                    b2.record(stream)
                    ts.append((a, b2))
                stream.synchronize()
                floors[name] = float(np.median([a.elapsed_time(b2) for a, b2 in ts])) * 1e3
            rt_floor.close()
        counts = rt.array_u64(s.fds[(0, "counts")])
        runs = 3 * nb + 5 * nb + 2 * (100 + 500)
        assert int(counts.sum()) == runs * n, "counter total != events (north star invariant)"
        bw = lambda ms: EVENT_BYTES * n / (ms / 1e3) / 1e9
        out[config] = {"events": n, "single_launch_us": single * 1e3, "single_events_per_s": n / (single / 1e3),
                       "single_hbm_frac": bw(single) / peaks["hbm_gbs"],
                       "steady_us": steady[False] * 1e3, "steady_events_per_s": n / (steady[False] / 1e3),
                       "steady_hbm_frac": bw(steady[False]) / peaks["hbm_gbs"],
                       "steady_pdl_us": steady[True] * 1e3, "steady_pdl_events_per_s": n / (steady[True] / 1e3),
                       "steady_pdl_hbm_frac": bw(steady[True]) / peaks["hbm_gbs"], "counter_total_ok": True,
                       "single_launch_floor_us": floors,
                       "single_vs_floor": min(floors.values()) / (single * 1e3),
                       "flush": "8 rotating 32-MiB batches (256 MiB > L2)"}
        rt.close()
        del bufs
    return out


def e2e_measure(rt, s, events, n, n_total, world, args):
    """gx_run_batch_host over pinned host events: H2D of every step's events and D2H of the
    step's result (the stats block) inside the timed region."""
    import torch
    import paper_2512_12615_b200 as gx
    avail = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                avail = int(line.split()[1]) * 1024
    except Exception:
        pass
    ne = n
    while ne * EVENT_BYTES * 1.5 * world > avail and ne > (1 << 24):
        ne //= 2
    host = torch.empty((ne, 32), dtype=torch.uint8, pin_memory=True)
    host.copy_(events[:ne])
    torch.cuda.synchronize()
    gx.gx_run_batch_host(rt.rt, host, prog_fd=s.prog_arg)   # warm the pipeline
    gx.gx_get_stats(rt.rt)
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        gx.gx_run_batch_host(rt.rt, host, prog_fd=s.prog_arg)
        gx.gx_get_stats(rt.rt)   # D2H read of the step's result
    dt = time.perf_counter() - t0
    # the bound of this path: the pinned host->device copy bandwidth of the box (1 GiB copies)
    probe = host.view(-1)[: 1 << 30]
    dst = torch.empty(probe.numel(), dtype=torch.uint8, device="cuda")
    dst.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        dst.copy_(probe, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d_gbs = 4 * probe.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
    achieved = ne * EVENT_BYTES * steps / dt / 1e9
    return {"value": ne * world * steps / dt, "unit": "events/s", "h2d_bytes_per_step": ne * EVENT_BYTES,
            "d2h_bytes_per_step": 64, "events_per_step": ne,
            "h2d_achieved_gbs": achieved, "h2d_copy_peak_gbs": h2d_gbs, "h2d_frac": achieved / h2d_gbs,
            "note": "gx_run_batch_host: chunked pinned H2D overlapped with execution; bound = the H2D copy "
                    "bandwidth (h2d_copy_peak_gbs, torch pinned copies measured in the same run)"}


def extra_lines(rt0, args):
    """Single-GPU timings of the other configs (stderr; not the headline line)."""
    import torch
    import paper_2512_12615_b200 as gx
    from gxin import configs, gen_gpu
    for config, n, eng in [(c, n, e) for c, n in (("C1", 1 << 20), ("C1", 1 << 26), ("C1d", 1 << 26), ("C3", 1 << 28),
                                                   ("C4", 1 << 28), ("C5", 1 << 26)) for e in ("jit", "interp")]:
        rt = gx.Runtime(0, engine=gx.GX_ENGINE_JIT if eng == "jit" else gx.GX_ENGINE_INTERP)
        s = configs.setup(rt, config)
        ev = gen_gpu.generate_device(config, configs.SEEDS[config], n)
        for _ in range(3):
            rt.run(ev, s.prog_arg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            rt.run(ev, s.prog_arg)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        st = rt.stats()
        print(json.dumps({"config": config, "engine": eng, "events": n, "ms": ms, "events_per_s": n / ms * 1e3,
                          "hbm_frac": n * 32 / (ms / 1e3) / 1e9 / measured_peaks()[0]["hbm_gbs"],
                          "warp_steps_per_record": st["warp_steps"] / 8 / (n / 32),
                          "divergent_frac": st["divergent_steps"] / max(1, st["warp_steps"])}), file=sys.stderr, flush=True)
        del ev
        rt.close()


def f2_lines():
    """C6 (stride-prefetch policy, 2^28 C3-trace events) and C2 (2^30)
    with and without the runtime daemon; the daemon publishes prefetch requests / watched-map
    snapshots at every kernel-completion boundary on the batch's stream."""
    import torch
    import paper_2512_12615_b200 as gx
    from gxin import configs, gen_gpu
    for config, n, watch in (("C6", 1 << 28, ["pstat"]), ("C2", 1 << 30, ["hist", "lane_pt"])):
        ev = gen_gpu.generate_device(config, configs.SEEDS[config], n)
        for daemon in (False, True):
            rt = gx.Runtime(0, engine=gx.GX_ENGINE_JIT)
            s = configs.setup(rt, config)
            if daemon:
                for name in watch:
                    gx.gx_daemon_watch(rt.rt, s.fds[(0, name)])
                rt.daemon_start(None)
            times, nreq = [], 0
            for k in range(8):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                rt.run(ev, s.prog_arg)
                b.record()
                torch.cuda.synchronize()
                if k >= 3:
                    times.append(a.elapsed_time(b))
                if not daemon and config == "C6":   # without a daemon the host drains (outside timing)
                    nreq = len(gx.gx_prefetch_drain(rt.rt, s.fds[(0, "pfq")], 1 << 24))
            ms = float(np.mean(times))
            line = {"f2": config, "events": n, "daemon": daemon, "ms": ms, "events_per_s": n / ms * 1e3,
                    "drops": rt.stats()["ringbuf_drops"]}
            if daemon:
                rt.daemon_stop()
                line["daemon_stats"] = gx.gx_daemon_get_stats(rt.rt)
            elif config == "C6":
                line["requests_per_batch"] = nreq
            print(json.dumps(line), file=sys.stderr, flush=True)
            rt.close()
        del ev


def f2_l2_line():
    """SURVEY.md §8f f2, the device half (stderr): the paper's prefetch microbenchmark shape
    (a vector add over managed memory whose pages start on the host; device-side
    prefetch.global.L2 "trigger[s] non-blocking page faults").  c = a + b over 2^28 floats in one
    managed buffer, P7 (L2 stride prefetch, distance d ahead of every hooked load) inlined on both
    loads; controls: the kernel without hooks, and with hooks whose prefetch length is 0 (-EINVAL:
    the hook cost without any prefetch).  Pages are moved back to the host before every launch."""
    import torch
    import cuda.bindings.runtime as cr
    import paper_2512_12615_b200 as gx
    from gxin import asm, instrument
    n = 1 << 28
    err, buf = cr.cudaMallocManaged(8 * n, cr.cudaMemAttachGlobal)
    if int(err) != 0:
        print(json.dumps({"f2": "l2_uvm", "skipped": f"cudaMallocManaged: {err}"}), file=sys.stderr, flush=True)
        return
    a, b = int(buf), int(buf) + 4 * n
    c = torch.empty(n, device="cuda")
    rt = gx.Runtime(0)
    region = rt.region_map(int(buf), 8 * n)

    def timed(k, reps=4):
        out = []
        for i in range(reps + 1):
            cr.cudaMemPrefetchAsync(buf, 8 * n, -1, 0)                # back to the host (cudaCpuDeviceId)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gx.gx_kernel_launch(rt.rt, k, "vadd", ((n + 255) // 256,), (256,), [a, b, c, 0, n])
            e1.record()
            torch.cuda.synchronize()
            if i:
                out.append(e0.elapsed_time(e1))
        return float(np.median(out))

    line = {"f2": "l2_uvm", "elements": n, "bytes": 12 * n}
    k0 = gx.gx_instrument(rt.rt, rt.load_prog(asm.assemble("mov64 r0, 0\nexit")), "#define GX_HOOKS 0\n" + instrument.VADD)
    line["ms_plain"] = timed(k0)
    gx.gx_kernel_free(rt.rt, k0)
    # the first access of every 64-KiB chunk prefetches one line d ahead (a per-access prefetch
    # floods the fault handler: measured 4.3x slower than no prefetch at all)
    for dist, ln in ((0, 0), (1 << 20, 128), (4 << 20, 128), (16 << 20, 128)):
        fds = instrument.setup_l2(rt, region, dist, ln, mask=(64 << 10) - 1)
        k = gx.gx_instrument(rt.rt, rt.load_prog(asm.assemble(instrument.P7_L2_STRIDE, fds)), instrument.VADD)
        key = "ms_hooks_no_prefetch" if ln == 0 else f"ms_l2_dist_{dist >> 20}MiB"
        line[key] = timed(k)
        line[key.replace("ms_", "outcome_")] = rt.array_u64(fds["outcome"]).tolist()
        gx.gx_kernel_free(rt.rt, k)
    best = min(v for kk, v in line.items() if kk.startswith("ms_l2"))
    line["speedup_best_vs_plain"] = line["ms_plain"] / best
    line["speedup_best_vs_hooks"] = line["ms_hooks_no_prefetch"] / best
    print(json.dumps(line), file=sys.stderr, flush=True)
    rt.close()
    cr.cudaFree(buf)


def f4_lines():
    """the paper's hook-overhead microbenchmark shape (PAPER.md:466-471,
    530): c = a + b over 2^28 floats with the counter policy inlined as a hook on both loads
    (gx_instrument), against the same kernel compiled without hooks."""
    import torch
    import paper_2512_12615_b200 as gx
    from gxin import asm, instrument
    n = 1 << 28
    a = torch.randn(n, device="cuda")
    b = torch.randn(n, device="cuda")
    c = torch.empty(n, device="cuda")
    rt = gx.Runtime(0)
    counts = rt.create_map(gx.GX_MAP_ARRAY, 4, 8, 256)
    prog = rt.load_prog(asm.assemble(instrument.PI, {"counts": counts}))
    res = {}
    for hooks in (0, 1):
        k = gx.gx_instrument(rt.rt, prog, f"#define GX_HOOKS {hooks}\n" + instrument.VADD)
        launch = lambda: gx.gx_kernel_launch(rt.rt, k, "vadd", ((n + 255) // 256,), (256,), [a, b, c, 0, n])
        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            launch()
        e1.record()
        torch.cuda.synchronize()
        res[hooks] = e0.elapsed_time(e1) / 10
        gx.gx_kernel_free(rt.rt, k)
    total = int(rt.array_u64(counts).sum())
    hooks_per_launch = 2 * n
    print(json.dumps({"f4": "vadd", "elements": n, "ms_no_hooks": res[0], "ms_hooks": res[1],
                      "overhead_pct": (res[1] - res[0]) / res[0] * 100,
                      "hook_events_per_s": hooks_per_launch / (res[1] / 1e3),
                      "added_ns_per_hook": (res[1] - res[0]) * 1e6 / hooks_per_launch,
                      "counter_total_ok": total == 13 * hooks_per_launch}), file=sys.stderr, flush=True)
    rt.close()


def f3_lines():
    """the work-stealing block scheduler on 148 persistent workers
    (§6.2.1 / Fig 4 shape) -- makespan per policy and workload.  (The discrete-event
    model's makespans for the same units are test-side: tests/test_oracle_sched.py.)"""
    import paper_2512_12615_b200 as gx
    from gxin import sched
    W = 148
    for kind in ("moderate", "heavy"):
        cost, home = sched.workload(kind, W)
        budget = int(cost.sum() / W * 0.2)
        line = {"f3": kind, "workers": W, "units": len(cost), "work_us": int(cost.sum())}
        for policy in ("fixed", "greedy", "latency_budget", "max_steals"):
            rt = gx.Runtime(0)
            prog, fds = sched.setup(rt, policy, W, budget_us=budget, max_steals=2)
            r = gx.gx_sched_run(rt.rt, prog, cost, home, W, 2)
            line[policy] = {"makespan_us": r["makespan_ns"] / 1e3, "steals": int(r["steals"].sum())}
            rt.close()
        print(json.dumps(line), file=sys.stderr, flush=True)
    # CLC mode ("MaxSteals (CLC)"): one block per unit, one block resident per SM
    # (200 KiB of shared memory each); a stealing block cancels pending blocks instead of exiting
    U = 8 * W
    for kind, cost in (("equal", np.full(U, 20, dtype=np.uint32)),
                       ("heavy", sched.workload("heavy", W)[0])):
        line = {"f3": "clc_" + kind, "units": len(cost), "work_us": int(cost.sum())}
        for policy, cap in (("fixed", 0), ("max_steals", 1), ("max_steals", 4), ("greedy", 0)):
            rt = gx.Runtime(0)
            prog, fds = sched.setup(rt, policy, len(cost), max_steals=cap)
            r = gx.gx_sched_run_ex(rt.rt, prog, cost, None, 0, 0, flags=gx.GX_SCHED_CLC, smem_per_block=200 * 1024)
            name = policy if policy != "max_steals" else f"max_steals_{cap}"
            line[name] = {"makespan_us": r["makespan_ns"] / 1e3, "steals": int(r["steals"].sum()),
                          "blocks_started": int((r["end_ns"] > 0).sum())}
            rt.close()
        print(json.dumps(line), file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
