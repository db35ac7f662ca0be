"""f3 inputs (F-5): the thread-block scheduling policies of PAPER.md §6.2.1
(FixedWork, Greedy, LatencyBudget, MaxSteals) as eBPF on the ENTER / EXIT / STEAL hooks, and the seeded work-unit
sets (moderate imbalance; heavy tail clustered on 10 % of the workers, "10% of blocks
perform 100--200x more work").  INPUT description only."""
from __future__ import annotations

import numpy as np

from .asm import assemble
from .gen import rnd

HOOK_ENTER, HOOK_EXIT, HOOK_STEAL = 1, 4, 5
ARRAY = 2

# every policy counts the hook kinds it sees (kcount[kind] += 1); the STEAL decision is policy-specific
_COUNT = """
    ldxw r6, [r1+16]          ; hook word: kind | stolen << 16
    ldxw r7, [r1+20]          ; worker (block_id)
    ldxw r8, [r1+28]          ; unit cost (us)
    mov64 r2, r6
    and64 r2, 255
    stxw [r10-4], r2
    lddw r1, map:kcount
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, +2
    mov64 r1, 1
    atomic_add64 [r0+0], r1
    mov64 r2, r6
    and64 r2, 255
"""

FIXED = _COUNT + """
    mov64 r0, 0               ; never steal
    exit
"""

GREEDY = _COUNT + """
    mov64 r0, 1               ; always steal
    exit
"""

# LatencyBudget ("caps per-block stealing time"): a worker may steal while the work it
# has stolen so far (stolen_us[worker], accumulated on EXIT of stolen units) is below cfg[0]
LATENCY_BUDGET = _COUNT + """
    jeq r2, 5, steal
    jne r2, 4, none           ; only EXIT accounts
    mov64 r2, r6
    rsh64 r2, 16
    and64 r2, 1
    jeq r2, 0, none           ; a home unit
    stxw [r10-8], r7
    lddw r1, map:stolen_us
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, none
    atomic_add64 [r0+0], r8
none:
    mov64 r0, 0
    exit
steal:
    stw [r10-12], 0
    lddw r1, map:cfg
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, none
    ldxdw r9, [r0+0]          ; budget (us)
    stxw [r10-8], r7
    lddw r1, map:stolen_us
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, none
    ldxdw r3, [r0+0]
    mov64 r0, 0
    jge r3, r9, +1
    mov64 r0, 1
    exit
"""

# MaxSteals ("MaxSteals (CLC)", Table 1): a worker may steal at most cfg[0] times;
# steals[worker] counts its granted STEAL decisions (only that worker's hooks touch its slot)
MAX_STEALS = _COUNT + """
    jne r2, 5, none
    stw [r10-12], 0
    lddw r1, map:cfg
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, none
    ldxdw r9, [r0+0]          ; the cap
    stxw [r10-8], r7
    lddw r1, map:steals
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, none
    ldxdw r3, [r0+0]
    jge r3, r9, none
    add64 r3, 1
    stxdw [r0+0], r3
    mov64 r0, 1
    exit
none:
    mov64 r0, 0
    exit
"""

POLICIES = {"fixed": FIXED, "greedy": GREEDY, "latency_budget": LATENCY_BUDGET, "max_steals": MAX_STEALS}
HOOK_PROBE, HOOK_RETPROBE = 6, 7


def setup(engine, policy: str, n_workers: int, budget_us: int = 0, max_steals: int = 0):
    """Creates the policy's maps on `engine` (oracle or runtime) and loads the program.  cfg[0] =
    budget_us (latency_budget) or max_steals (max_steals).  Returns (prog handle, {map name: fd})."""
    fds = {"kcount": engine.create_map(ARRAY, 4, 8, 8),
           "stolen_us": engine.create_map(ARRAY, 4, 8, max(1, n_workers)),
           "steals": engine.create_map(ARRAY, 4, 8, max(1, n_workers)),
           "cfg": engine.create_map(ARRAY, 4, 8, 1)}
    cfg = max_steals if policy == "max_steals" else budget_us
    engine.update_map(fds["cfg"], (0).to_bytes(4, "little"), int(cfg).to_bytes(8, "little"), 0)
    return engine.load_prog(assemble(POLICIES[policy], fds)), fds


def workload(kind: str, n_workers: int, units_per_worker: int = 8, seed: int = 0x5EED0F3):
    """(cost_us[U], home[U]).  'moderate': costs uniform in [25, 75] us, round-robin homes;
    'heavy': 10 % of the units cost 100-200x a 5-us base and are homed on the first 10 % of the
    workers (clustered), the rest 5 us round-robin."""
    U = n_workers * units_per_worker
    r = rnd(seed, 1, np.arange(U, dtype=np.uint64))
    if kind == "moderate":
        cost = (25 + (r % np.uint64(51))).astype(np.uint32)
        home = (np.arange(U) % n_workers).astype(np.uint32)
        return cost, home
    n_heavy = max(1, U // 10)
    hot = max(1, n_workers // 10)
    cost = np.full(U, 5, dtype=np.uint32)
    cost[:n_heavy] = (5 * (100 + (r[:n_heavy] % np.uint64(101)))).astype(np.uint32)
    home = np.empty(U, dtype=np.uint32)
    home[:n_heavy] = np.arange(n_heavy) % hot
    home[n_heavy:] = np.arange(U - n_heavy) % n_workers
    return cost, home
