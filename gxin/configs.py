"""Config recipes C1..C5: which maps to create, their host-written
contents, which programs to load and where to attach them.

INPUT description only.  `setup` drives any object with the engine methods
    create_map(type, key_size, value_size, max_entries) -> fd
    update_map(fd, key: bytes, value: bytes, flags) -> int
    load_prog(slots: bytes) -> handle
    attach(handle, kind, tenant)
so the same recipe configures the CPU oracle (tests, bench cpu_baseline) and the
C-ABI library (tests, bench).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import gen, programs

# config -> list of (tenant, program name, attach kinds)
TENANTS = {
    "C1": [(0, "P1", (0,))],
    "C1d": [(0, "P1d", (0,))],
    "C2": [(0, "P2", (0,))],
    "C3": [(0, "P3", (0,))],
    "C4": [(0, "P4", (0,))],
    "C5": [(0, "P1", (0,)), (1, "P2", (0,)), (2, "P3f", (0, 2)), (3, "P4", (0,))],
    "C6": [(0, "P6", (0,))],
}
# C6 (f2, prefetch policy) reads the C3 LLM page trace
GEN_CONFIG = {"C1": "C1", "C1d": "C1", "C2": "C2", "C3": "C3", "C4": "C4", "C5": "C5", "C6": "C3"}


@dataclass
class Setup:
    config: str
    fds: dict = field(default_factory=dict)      # (tenant, map name) -> fd
    progs: dict = field(default_factory=dict)    # tenant -> handle
    prog_arg: object = -1                        # single program handle, or -1 = attach table


def setup(engine, config: str, threshold: int | None = None) -> Setup:
    s = Setup(config)
    for tenant, pname, kinds in TENANTS[config]:
        fds = {}
        for mname, spec in programs.maps_of(pname).items():
            fds[mname] = engine.create_map(spec.type, spec.key_size, spec.value_size, spec.max_entries)
            s.fds[(tenant, mname)] = fds[mname]
        if pname == "P4":   # host-written read-only tables
            t = gen.c4_tables()
            engine.update_map(fds["cfg"], (0).to_bytes(4, "little"), int(t["cfg"][0]).to_bytes(8, "little"), 0)
            for k, v in enumerate(t["bounds"]):
                engine.update_map(fds["bounds"], k.to_bytes(4, "little"), int(v).to_bytes(8, "little"), 0)
        kw = {"threshold": threshold} if (pname == "P3" and threshold is not None) else {}
        h = engine.load_prog(programs.build(pname, fds, **kw))
        s.progs[tenant] = h
        if config == "C5":
            for kind in kinds:
                engine.attach(h, kind, tenant)
    if config != "C5":
        s.prog_arg = s.progs[0]
    return s


def events(config: str, seed: int, n: int, i0: int = 0, n_total: int | None = None) -> np.ndarray:
    return gen.generate(GEN_CONFIG[config], seed, n, i0, n_total)


SEEDS = {"C1": 0x5EED0001, "C1d": 0x5EED0001, "C2": 0x5EED0002, "C3": 0x5EED0003,
         "C4": 0x5EED0004, "C5": 0x5EED0005, "C6": 0x5EED0003}
