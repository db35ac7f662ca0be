"""The config policies P1, P1d, P2, P3, P3', P4 as eBPF text.

These are inputs (program bytes), not semantics.  Map names are resolved to fds
by `build(name, fds)`; each entry of `MAPS` is the map spec the config creates
(type ids follow bpf.h:925-965: HASH 1, ARRAY 2, PERTHREAD ARRAY 6 (the
PERCPU_ARRAY slot), RINGBUF 27).

Event record (little endian):
    0 u64 addr | 8 u64 ts | 16 u32 hook (kind | tenant<<8 | is_write<<16)
    20 u32 block_id | 24 u16 sm_id | 26 u8 warp_id | 27 u8 lane_id | 28 u32 size
"""
from __future__ import annotations

from dataclasses import dataclass

from .asm import assemble

HASH, ARRAY, PERTHREAD_ARRAY, RINGBUF, PREFETCH_QUEUE = 1, 2, 6, 27, 64
FN_MEM_PREFETCH = 1000   # gdev_mem_prefetch (F-1)
HOOK_ACCESS, HOOK_BLOCK_ENTER, HOOK_FAULT = 0, 1, 2


@dataclass(frozen=True)
class MapSpec:
    type: int
    key_size: int
    value_size: int
    max_entries: int
    flags: int = 0


# --- C1: counter policy ("per-region access counters"; BASELINE.json configs[0]) ---
# P1: helper form, 13 insns in 14 slots: counts[(addr >> 12) & 255] += 1
P1 = """
    ldxdw r2, [r1+0]          ; addr
    rsh64 r2, 12
    and64 r2, 255             ; key = page & 255
    stxw [r10-4], r2
    lddw r1, map:counts
    mov64 r2, r10
    add64 r2, -4
    call 1                    ; bpf_map_lookup_elem
    jeq r0, 0, +2
    mov64 r1, 1
    atomic_add64 [r0+0], r1
    mov64 r0, 0
    exit
"""
P1_MAPS = {"counts": MapSpec(ARRAY, 4, 8, 256)}

# P1d: direct-value form, exactly 8 insns (9 slots); a 1-entry "global array" of 256 u64
P1D = """
    ldxdw r2, [r1+0]
    rsh64 r2, 9
    and64 r2, 0x7f8           ; ((addr >> 12) & 255) * 8
    lddw r1, mapval:counts+0  ; BPF_PSEUDO_MAP_VALUE
    add64 r1, r2
    mov64 r0, 1
    atomic_add64 [r1+0], r0
    exit
"""
P1D_MAPS = {"counts": MapSpec(ARRAY, 4, 2048, 1)}

# --- C2: per-SM / per-warp histogram + per-thread lane stats (Fig 2; 511 threadhist) ---
P2 = """
    mov64 r6, r1
    ldxh r2, [r6+24]          ; sm_id
    ldxb r3, [r6+26]          ; warp_id
    lsh64 r2, 6
    add64 r2, r3              ; key = sm_id*64 + warp_id
    stxw [r10-4], r2
    lddw r1, map:hist
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, lane
    mov64 r1, 1
    atomic_add64 [r0+0], r1
lane:
    ldxb r2, [r6+27]          ; lane_id
    stxw [r10-8], r2
    lddw r1, map:lane_pt
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, out
    ldxdw r1, [r0+0]          ; per-thread shard: plain RMW (no atomics)
    add64 r1, 1
    stxdw [r0+0], r1
    ldxw r1, [r6+28]          ; size
    ldxdw r2, [r0+8]
    add64 r2, r1
    stxdw [r0+8], r2
out:
    mov64 r0, 0
    exit
"""
P2_MAPS = {"hist": MapSpec(ARRAY, 4, 8, 148 * 64), "lane_pt": MapSpec(PERTHREAD_ARRAY, 4, 16, 32)}


# --- C3: LFU-style page counting in a 1M-entry hash + ringbuf on threshold crossing ---
def p3_text(threshold: int = 64) -> str:
    return f"""
    ldxdw r6, [r1+0]
    rsh64 r6, 12              ; page
    stxdw [r10-8], r6
    lddw r1, map:lfu
    mov64 r2, r10
    add64 r2, -8
    call 1
    jne r0, 0, have
    stdw [r10-16], 0          ; lookup-or-init: update(page, 0, BPF_NOEXIST)
    lddw r1, map:lfu
    mov64 r2, r10
    add64 r2, -8
    mov64 r3, r10
    add64 r3, -16
    mov64 r4, 1
    call 2
    lddw r1, map:lfu
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, out
have:
    mov64 r1, 1
    atomic_fetch_add64 [r0+0], r1
    add64 r1, 1
    jne r1, {threshold}, out  ; emit exactly when the count crosses T
    stxdw [r10-24], r6
    stdw [r10-16], {threshold}
    lddw r1, map:rb
    mov64 r2, r10
    add64 r2, -24
    mov64 r3, 16
    mov64 r4, 0
    call 130                  ; bpf_ringbuf_output
out:
    mov64 r0, 0
    exit
"""


P3 = p3_text(64)
P3_MAPS = {"lfu": MapSpec(HASH, 8, 8, 1 << 20), "rb": MapSpec(RINGBUF, 0, 0, 32 << 20)}

# P3': counting without a threshold; FAULT records emit {page, sm_id} unconditionally (C5 tenant 2)
P3F = """
    mov64 r7, r1
    ldxdw r6, [r7+0]
    rsh64 r6, 12
    stxdw [r10-8], r6
    lddw r1, map:lfu
    mov64 r2, r10
    add64 r2, -8
    call 1
    jne r0, 0, have
    stdw [r10-16], 0
    lddw r1, map:lfu
    mov64 r2, r10
    add64 r2, -8
    mov64 r3, r10
    add64 r3, -16
    mov64 r4, 1
    call 2
    lddw r1, map:lfu
    mov64 r2, r10
    add64 r2, -8
    call 1
    jeq r0, 0, fault
have:
    mov64 r1, 1
    atomic_add64 [r0+0], r1
fault:
    ldxw r1, [r7+16]
    and64 r1, 255
    jne r1, 2, out            ; hook kind FAULT only
    stxdw [r10-24], r6
    ldxh r1, [r7+24]
    stxdw [r10-16], r1
    lddw r1, map:rb
    mov64 r2, r10
    add64 r2, -24
    mov64 r3, 16
    mov64 r4, 0
    call 130
out:
    mov64 r0, 0
    exit
"""
# C5's FAULT records are unconditional (2 % of the events, 24 B each): 1 GiB holds the 2^28-event
# batches of a warm-up plus the timed steps without a drop (bench.py)
P3F_MAPS = {"lfu": MapSpec(HASH, 8, 8, 1 << 20), "rb": MapSpec(RINGBUF, 0, 0, 1 << 30)}

# --- C4: vector-search stream; 12-iteration bounded binary search over 4097 list bounds ---
P4 = """
    mov64 r6, r1
    ldxdw r7, [r6+0]          ; addr
    stw [r10-4], 0
    lddw r1, map:cfg
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, out0
    ldxdw r1, [r0+0]          ; cfg[0] = end of the centroid region
    jge r7, r1, search
    stw [r10-4], 0
    lddw r1, map:cstat
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, out0
    mov64 r1, 1
    atomic_add64 [r0+0], r1   ; centroid scans
out0:
    mov64 r0, 4096
    exit
search:
    mov64 r8, 0               ; lo : bounds[lo] <= addr
    mov64 r9, 4096            ; hi : addr < bounds[hi]
    stdw [r10-16], 12         ; bounded loop counter (12 = log2 4096)
loop:
    mov64 r1, r8
    add64 r1, r9
    rsh64 r1, 1               ; mid
    stxw [r10-4], r1
    lddw r1, map:bounds
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, out0
    ldxw r1, [r10-4]
    ldxdw r2, [r0+0]          ; bounds[mid]
    jgt r2, r7, left          ; lane-varying branch (relaxed SIMT mode)
    mov64 r8, r1
    ja next
left:
    mov64 r9, r1
next:
    ldxdw r1, [r10-16]
    sub64 r1, 1
    stxdw [r10-16], r1
    jne r1, 0, loop
    stxw [r10-4], r8          ; list id
    lddw r1, map:list_hits
    mov64 r2, r10
    add64 r2, -4
    call 1
    jne r0, 0, hit
    stdw [r10-24], 0
    lddw r1, map:list_hits
    mov64 r2, r10
    add64 r2, -4
    mov64 r3, r10
    add64 r3, -24
    mov64 r4, 1
    call 2
    lddw r1, map:list_hits
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, bytes
hit:
    mov64 r1, 1
    atomic_add64 [r0+0], r1
bytes:
    stxw [r10-4], r8
    lddw r1, map:list_bytes
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, pt
    ldxw r1, [r6+28]
    atomic_add64 [r0+0], r1
pt:
    stw [r10-4], 0
    lddw r1, map:scan_pt
    mov64 r2, r10
    add64 r2, -4
    call 1
    jeq r0, 0, ret
    ldxw r1, [r6+28]
    ldxdw r2, [r0+0]
    add64 r2, r1
    stxdw [r0+0], r2
ret:
    mov64 r0, r8
    exit
"""
P4_MAPS = {"cfg": MapSpec(ARRAY, 4, 8, 1), "cstat": MapSpec(ARRAY, 4, 8, 4),
           "bounds": MapSpec(ARRAY, 4, 8, 4097), "list_hits": MapSpec(HASH, 4, 8, 4096),
           "list_bytes": MapSpec(ARRAY, 4, 8, 4096), "scan_pt": MapSpec(PERTHREAD_ARRAY, 4, 8, 1)}

# --- C6: the "GPU L2 Stride Prefetch" device policy ---
# P6: when a lane touches the last 128 B of a 4-KiB page, request the next 64 KiB (16 pages)
# through gdev_mem_prefetch; the host daemon's prefetch handler receives the requests.
P6 = """
    ldxdw r6, [r1+0]          ; addr
    mov64 r2, r6
    and64 r2, 4095
    jlt r2, 3968, out         ; not in the page's last 128 B
    lddw r1, map:pfq
    mov64 r2, r6
    rsh64 r2, 12
    add64 r2, 1
    lsh64 r2, 12              ; next page
    mov64 r3, 65536           ; 16 pages ahead
    call 1000                 ; gdev_mem_prefetch(queue, addr, len)
    lddw r1, mapval:pstat+0
    mov64 r2, 1
    atomic_add64 [r1+0], r2   ; prefetch calls (a counter the host reads back)
out:
    mov64 r0, 0
    exit
"""
P6_MAPS = {"pfq": MapSpec(PREFETCH_QUEUE, 0, 0, 1 << 24), "pstat": MapSpec(ARRAY, 4, 8, 1)}

PROGRAMS = {"P1": (P1, P1_MAPS), "P1d": (P1D, P1D_MAPS), "P2": (P2, P2_MAPS),
            "P3": (P3, P3_MAPS), "P3f": (P3F, P3F_MAPS), "P4": (P4, P4_MAPS), "P6": (P6, P6_MAPS)}


def build(name: str, fds: dict, **kw) -> bytes:
    """Assemble program `name` with map names resolved through `fds`."""
    if name == "P3" and "threshold" in kw:
        return assemble(p3_text(kw["threshold"]), fds)
    return assemble(PROGRAMS[name][0], fds)


def maps_of(name: str) -> dict:
    return dict(PROGRAMS[name][1])
