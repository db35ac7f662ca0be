"""Verifier corpus on the CPU through
gx_verify_offline (the same verifier gx_verify runs), plus NVRTC compilation of the JIT kernels."""
import pytest

import paper_2512_12615_b200 as gx
from gxin import asm, programs

HASH, ARRAY, PT, RINGBUF, PFQ, REGION = 1, 2, 6, 27, 64, 65
MAPS = {0: (ARRAY, 4, 8, 16), 1: (HASH, 8, 8, 64), 2: (PT, 4, 16, 32), 3: (RINGBUF, 0, 0, 4096),
        4: (ARRAY, 4, 2048, 1), 5: (PFQ, 0, 0, 64), 6: (REGION, 0, 0, 1)}
NAMES = {"arr": 0, "h": 1, "pt": 2, "rb": 3, "g": 4, "pfq": 5, "reg": 6}


def verify(text, strict=False, **kw):
    v, rep, log = gx.gx_verify_offline(asm.assemble(text, NAMES), MAPS, strict=strict, **kw)
    return v, rep["rule"], rep, log


LOOKUP = """
    stw [r10-4], 1
    lddw r1, map:arr
    mov64 r2, r10
    add64 r2, -4
    call 1
"""

ACCEPT = {
    "const0": "mov64 r0, 0\nexit",
    "ctx_all_fields": "ldxdw r0, [r1+0]\nldxdw r2, [r1+8]\nldxw r3, [r1+16]\nldxh r4, [r1+24]\nldxb r5, [r1+27]\nexit",
    "lookup_nullcheck": LOOKUP + "jeq r0, 0, +1\nldxdw r0, [r0+0]\nexit",
    # an ARRAY key provably below max_entries (constant, or masked) cannot miss: no NULL check needed
    "lookup_key_in_range": LOOKUP + "ldxdw r0, [r0+0]\nexit",
    "lookup_masked_key_in_range": LOOKUP.replace("stw [r10-4], 1", "ldxw r2, [r1+0]\nand64 r2, 15\nstxw [r10-4], r2")
                                  + "ldxdw r0, [r0+0]\nexit",
    "bounded_loop_counter": "mov64 r0, 0\nmov64 r6, 8\nl: add64 r0, 1\nsub64 r6, 1\njne r6, 0, l\nexit",
    "stack_spill_fill_ptr": LOOKUP + "stxdw [r10-16], r0\nldxdw r1, [r10-16]\njeq r1, 0, +1\nldxdw r0, [r1+0]\nmov64 r0, 0\nexit",
    "var_offset_in_bounds": "ldxdw r2, [r1+0]\nand64 r2, 0xf8\nlddw r1, mapval:g+0\nadd64 r1, r2\nldxdw r0, [r1+0]\nexit",
    "atomic_fetch": LOOKUP + "jeq r0, 0, +4\nmov64 r1, 1\natomic_fetch_add64 [r0+0], r1\nmov64 r0, r1\nexit\nmov64 r0, 0\nexit",
    "hash_update": "stdw [r10-8], 5\nstdw [r10-16], 7\nlddw r1, map:h\nmov64 r2, r10\nadd64 r2, -8\nmov64 r3, r10\nadd64 r3, -16\nmov64 r4, 0\ncall 2\nexit",
    "mem_prefetch": "ldxdw r2, [r1+0]\nmov64 r3, 4096\nlddw r1, map:pfq\ncall 1000\nexit",
    "prefetch_l2": "ldxdw r2, [r1+0]\nmov64 r3, 128\nlddw r1, map:reg\ncall 1001\nexit",
    "mem_prefetch_policy": programs.P6.replace("map:pfq", "map:pfq").replace("mapval:pstat+0", "mapval:g+0"),
    "ringbuf": "stdw [r10-16], 1\nstdw [r10-8], 2\nlddw r1, map:rb\nmov64 r2, r10\nadd64 r2, -16\nmov64 r3, 16\nmov64 r4, 0\ncall 130\nexit",
    "percpu_rmw": "stw [r10-4], 3\nlddw r1, map:pt\nmov64 r2, r10\nadd64 r2, -4\ncall 1\njeq r0, 0, +3\nldxdw r1, [r0+8]\nadd64 r1, 1\nstxdw [r0+8], r1\nmov64 r0, 0\nexit",
    "jmp32_ok": "ldxw r2, [r1+16]\nmov64 r0, 0\njgt32 r2, 5, +1\nmov64 r0, 1\nexit",
    "sdiv_smod_movsx": "ldxdw r0, [r1+0]\nsdiv64 r0, 3\nsmod64 r0, 5\nmovsx864 r0, r0\nexit",
    "bswap_end": "ldxdw r0, [r1+0]\nbe16 r0\nbswap64 r0\nle32 r0\nexit",
    "ptr_sub_same_region": "mov64 r2, r10\nadd64 r2, -8\nmov64 r0, r10\nsub64 r0, r2\nexit",
    "uniform_branch_strict_ok": "ldxw r2, [r1+16]\nmov64 r0, 0\njeq r2, 3, +1\nmov64 r0, 1\nexit",
    "cmpxchg_stack": "stdw [r10-8], 5\nmov64 r0, 5\nmov64 r4, 9\ncmpxchg64 [r10-8], r4\nexit",
    "st_imm_map": LOOKUP + "jeq r0, 0, +1\nstdw [r0+0], 3\nmov64 r0, 0\nexit",
    "nested_loops": "mov64 r0, 0\nmov64 r6, 3\no: mov64 r7, 4\ni: add64 r0, 1\nsub64 r7, 1\njne r7, 0, i\nsub64 r6, 1\njne r6, 0, o\nexit",
    "update_noexist_lookup_again": programs.P3.replace("map:lfu", "map:h").replace("map:rb", "map:rb"),
    "ldimm64_scalar": "lddw r0, 0x123456789abcdef0\nexit",
}

REJECT = {
    # (program, strict, expected rule)
    "uninit_r0": ("exit", False, "UNINIT_READ"),
    "uninit_stack": ("ldxdw r0, [r10-8]\nexit", False, "UNINIT_READ"),
    "oob_ctx": ("ldxdw r0, [r1+32]\nexit", False, "OOB_ACCESS"),
    "ctx_write": ("stdw [r1+0], 1\nmov64 r0, 0\nexit", False, "OOB_ACCESS"),
    "oob_stack": ("stdw [r10+0], 1\nmov64 r0, 0\nexit", False, "OOB_ACCESS"),
    "oob_stack_deep": ("stdw [r10-520], 1\nmov64 r0, 0\nexit", False, "OOB_ACCESS"),
    "oob_map_value": (LOOKUP + "jeq r0, 0, +1\nldxdw r0, [r0+8]\nmov64 r0, 0\nexit", False, "OOB_ACCESS"),
    "null_deref": (LOOKUP.replace("stw [r10-4], 1", "ldxw r2, [r1+0]\nstxw [r10-4], r2") + "ldxdw r0, [r0+0]\nexit",
                   False, "NULL_DEREF"),
    "null_deref_key_out_of_range": (LOOKUP.replace("stw [r10-4], 1", "stw [r10-4], 16") + "ldxdw r0, [r0+0]\nexit",
                                    False, "NULL_DEREF"),
    "null_deref_key_range_too_wide": (LOOKUP.replace("stw [r10-4], 1", "ldxw r2, [r1+0]\nand64 r2, 31\nstxw [r10-4], r2")
                                      + "ldxdw r0, [r0+0]\nexit", False, "NULL_DEREF"),
    "misaligned": ("ldxdw r0, [r1+4]\nexit", False, "MISALIGNED"),
    "var_offset_misaligned": ("ldxdw r2, [r1+0]\nand64 r2, 0xfc\nlddw r1, mapval:g+0\nadd64 r1, r2\nldxdw r0, [r1+0]\nexit", False, "MISALIGNED"),
    "var_offset_oob": ("ldxdw r2, [r1+0]\nand64 r2, 0xff8\nlddw r1, mapval:g+0\nadd64 r1, r2\nldxdw r0, [r1+0]\nexit", False, "OOB_ACCESS"),
    "unbounded_loop": ("mov64 r0, 0\nl: add64 r0, 0\nja l", False, "UNBOUNDED_LOOP"),
    "loop_bound_from_map": (LOOKUP + "jeq r0, 0, +5\nldxdw r6, [r0+0]\nl: sub64 r6, 1\njne r6, 0, l\nmov64 r0, 0\nexit\nmov64 r0, 0\nexit", False, "BUDGET"),
    "strict_loop_bound_from_map": (LOOKUP + "jeq r0, 0, +5\nldxdw r6, [r0+0]\nl: sub64 r6, 1\njne r6, 0, l\nmov64 r0, 0\nexit\nmov64 r0, 0\nexit", True, "UNIFORM_LOOP_BOUND"),
    "return_pointer": ("mov64 r0, r10\nexit", False, "PTR_LEAK"),
    "pointer_to_map": (LOOKUP + "jeq r0, 0, +1\nstxdw [r0+0], r10\nmov64 r0, 0\nexit", False, "PTR_LEAK"),
    "pointer_mul": ("mov64 r0, r10\nmul64 r0, 2\nmov64 r0, 0\nexit", False, "PTR_LEAK"),
    "shift_range": ("mov64 r0, 1\nlsh64 r0, 64\nexit", False, "SHIFT_RANGE"),
    "shift_range32": ("mov64 r0, 1\nlsh32 r0, 32\nexit", False, "SHIFT_RANGE"),
    "bad_helper": ("call 6\nmov64 r0, 0\nexit", False, "BAD_HELPER"),
    "spin_lock": ("call 93\nmov64 r0, 0\nexit", False, "FORBIDDEN_SYNC"),
    "helper_bad_map_arg": ("mov64 r1, 1\nmov64 r2, r10\ncall 1\nmov64 r0, 0\nexit", False, "BAD_HELPER"),
    "prefetch_on_array": ("mov64 r2, 0\nmov64 r3, 64\nlddw r1, map:arr\ncall 1000\nexit", False, "BAD_HELPER"),
    "prefetch_uninit_len": ("mov64 r2, 0\nlddw r1, map:pfq\ncall 1000\nexit", False, "UNINIT_READ"),
    "prefetch_ptr_len": ("mov64 r2, 0\nmov64 r3, r10\nlddw r1, map:pfq\ncall 1000\nexit", False, "BAD_HELPER"),
    "prefetch_l2_on_queue": ("mov64 r2, 0\nmov64 r3, 64\nlddw r1, map:pfq\ncall 1001\nexit", False, "BAD_HELPER"),
    "mem_prefetch_on_region": ("mov64 r2, 0\nmov64 r3, 64\nlddw r1, map:reg\ncall 1000\nexit", False, "BAD_HELPER"),
    "prefetch_l2_uninit_len": ("mov64 r2, 0\nlddw r1, map:reg\ncall 1001\nexit", False, "UNINIT_READ"),
    "prefetch_l2_ptr_addr": ("mov64 r2, r10\nmov64 r3, 8\nlddw r1, map:reg\ncall 1001\nexit", False, "BAD_HELPER"),
    "lookup_on_region": ("stw [r10-4], 0\nlddw r1, map:reg\nmov64 r2, r10\nadd64 r2, -4\ncall 1\nmov64 r0, 0\nexit", False, "BAD_HELPER"),
    "lookup_on_prefetch_queue": ("stw [r10-4], 0\nlddw r1, map:pfq\nmov64 r2, r10\nadd64 r2, -4\ncall 1\nmov64 r0, 0\nexit", False, "BAD_HELPER"),
    "ringbuf_var_size": ("ldxdw r3, [r1+0]\nstdw [r10-8], 1\nlddw r1, map:rb\nmov64 r2, r10\nadd64 r2, -8\nmov64 r4, 0\ncall 130\nexit", False, "BAD_HELPER"),
    "bad_reg": (".raw 0xb7 11 0 0 0\nexit", False, "BAD_REG"),
    "write_r10": ("mov64 r10, 0\nmov64 r0, 0\nexit", False, "BAD_REG"),
    "ld_abs": (".raw 0x20 0 0 0 0\nmov64 r0, 0\nexit", False, "BAD_INSN"),
    "bad_jump": ("ja +5\nmov64 r0, 0\nexit", False, "BAD_JUMP"),
    "fallthrough": ("mov64 r0, 0", False, "FALLTHROUGH"),
    "unreachable": ("mov64 r0, 0\nexit\nmov64 r0, 1\nexit", False, "UNREACHABLE"),
    "div_zero_imm": ("mov64 r0, 1\ndiv64 r0, 0\nexit", False, "BAD_INSN"),
    "budget_helpers": ("mov64 r6, 70\nl: " + LOOKUP + "sub64 r6, 1\njne r6, 0, l\nmov64 r0, 0\nexit", False, "BUDGET"),
    # strict SIMT rules
    "strict_lane_branch": ("ldxdw r2, [r1+0]\nmov64 r0, 0\njeq r2, 3, +1\nmov64 r0, 1\nexit", True, "UNIFORM_BRANCH"),
    "strict_lane_loop": ("ldxdw r6, [r1+0]\nand64 r6, 7\nmov64 r0, 0\nl: add64 r0, 1\njgt r6, r0, l\nexit", True, "UNIFORM_LOOP_BOUND"),
    "strict_lane_key": ("ldxdw r2, [r1+0]\nstxdw [r10-8], r2\nstdw [r10-16], 0\nlddw r1, map:h\nmov64 r2, r10\nadd64 r2, -8\nmov64 r3, r10\nadd64 r3, -16\nmov64 r4, 0\ncall 2\nmov64 r0, 0\nexit", True, "UNIFORM_MAP_KEY"),
    "strict_lane_atomic": (programs.P1D.replace("map", "map").replace("mapval:counts", "mapval:g"), True, "NON_UNIFORM_ATOMIC"),
}


@pytest.mark.parametrize("name", sorted(ACCEPT))
def test_accept(name):
    v, rule, rep, log = verify(ACCEPT[name])
    assert v == 0, (name, rule, log)


@pytest.mark.parametrize("name", sorted(REJECT))
def test_reject(name):
    text, strict, want = REJECT[name]
    v, rule, rep, log = verify(text, strict=strict)
    assert v < 0 and rule == want, (name, v, rule, log)


def test_corpus_size_and_rule_coverage():
    """>= 20 accept and >= 20 reject programs, at least one per rule."""
    assert len(ACCEPT) >= 20 and len(REJECT) >= 20
    rules = {r for _, _, r in REJECT.values()}
    for need in ("UNIFORM_BRANCH", "UNIFORM_LOOP_BOUND", "UNIFORM_MAP_KEY", "FORBIDDEN_SYNC", "NON_UNIFORM_ATOMIC",
                 "BUDGET", "UNBOUNDED_LOOP", "OOB_ACCESS"):
        assert need in rules


def test_budget_counts():
    """SPEC.md:153-155 style hand counts: straight line of 10 -> 10; loop of 8 with one lookup."""
    v, rule, rep, _ = verify("mov64 r0, 0\n" + "add64 r0, 1\n" * 8 + "exit")
    assert v == 0 and rep["worst_insns"] == 10
    text = "mov64 r6, 8\nl: " + LOOKUP + "sub64 r6, 1\njne r6, 0, l\nmov64 r0, 0\nexit"
    v, rule, rep, _ = verify(text)
    assert v == 0 and rep["worst_helpers"] == 8 and rep["worst_insns"] == 1 + 8 * 7 + 2
    v, rule, rep, _ = verify(text, max_helpers=7)
    assert v < 0 and rule == "BUDGET"


def test_config_programs_verify_and_strict_classification():
    for name in programs.PROGRAMS:
        specs = programs.maps_of(name)
        fds = {k: i for i, k in enumerate(specs)}
        maps = {fds[k]: (s.type, s.key_size, s.value_size, s.max_entries) for k, s in specs.items()}
        v, rep, log = gx.gx_verify_offline(programs.build(name, fds), maps)
        assert v == 0, (name, log)
        assert rep["image_insns"] <= rep["n_insns"]
        # every config program has a lane-varying branch (relaxed-mode programs)
        v2, rep2, _ = gx.gx_verify_offline(programs.build(name, fds), maps, strict=True)
        assert v2 < 0


def test_p4_loop_is_bounded_by_exploration():
    specs = programs.maps_of("P4")
    fds = {k: i for i, k in enumerate(specs)}
    maps = {fds[k]: (s.type, s.key_size, s.value_size, s.max_entries) for k, s in specs.items()}
    v, rep, _ = gx.gx_verify_offline(programs.build("P4", fds), maps)
    assert v == 0 and rep["worst_insns"] > 12 * 10 and rep["processed_insns"] < 1_000_000


@pytest.mark.parametrize("name", sorted(programs.PROGRAMS))
def test_jit_compiles_offline(name):
    """f1: every config program's JIT kernel compiles with NVRTC for sm_100a (no device needed)."""
    specs = programs.maps_of(name)
    fds = {k: i for i, k in enumerate(specs)}
    maps = {fds[k]: (s.type, s.key_size, s.value_size, s.max_entries) for k, s in specs.items()}
    rc, src, log = gx.gx_jit_offline(programs.build(name, fds), maps)
    if rc == -38:  # ENOSYS: libnvrtc not loadable on this host
        pytest.skip(log)
    assert rc == 0, log
    assert "gx_jit_kernel" in src


@pytest.mark.parametrize("knobs,progs", [
    ({"GX_JIT_STAGE_MODE": "0", "GX_JIT_STAGES": "3"}, ("P2",)), ({"GX_JIT_STAGE_MODE": "1", "GX_JIT_STAGES": "2"}, ("P2",)),
    ({"GX_JIT_STAGE_MODE": "2", "GX_JIT_STAGES": "4"}, ("P2",)), ({"GX_JIT_RING_RELEASE": "mbar"}, ("P2",)),
    ({"GX_JIT_RING_CLAIM": "static", "GX_JIT_RING_RELEASE": "mbar"}, ("P2",)), ({"GX_JIT_PTCACHE": "1"}, ("P2",)),
    ({"GX_JIT_RING_RPW": "2"}, ("P2", "P3")),
    ({"GX_JIT_IFCONV": "0"}, ("P4",)), ({"GX_JIT_HASH_L1PROBE": "0"}, ("P3",)), ({"GX_JIT_HASH_L1PROBE": "1"}, ("P3",)), ({"GX_JIT_HASH_CACHE": "0"}, ("P3",)), ({"GX_JIT_PIN": "0"}, ("P2",)), ({"GX_JIT_PT_HINT": "1"}, ("P2",)), ({"GX_JIT_PT_HINT": "2"}, ("P2",)), ({"GX_JIT_BLOCK": "256"}, ("P6",))])
def test_jit_variants_compile_offline(knobs, progs, monkeypatch):
    """Every JIT code-generation variant kept for measurement (profiles/r1_jit_variants.md) still
    generates valid sm_100a code for a program that exercises it (P2 per-thread, P3 hash+ringbuf,
    P4 loop, P6 prefetch)."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    for name in progs:
        specs = programs.maps_of(name)
        fds = {k: i for i, k in enumerate(specs)}
        maps = {fds[k]: (s.type, s.key_size, s.value_size, s.max_entries) for k, s in specs.items()}
        rc, src, log = gx.gx_jit_offline(programs.build(name, fds), maps)
        if rc == -38:
            pytest.skip(log)
        assert rc == 0, (name, knobs, log[-2000:])


def _jit_source(name, **env):
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        specs = programs.maps_of(name)
        fds = {k: i for i, k in enumerate(specs)}
        maps = {fds[k]: (s.type, s.key_size, s.value_size, s.max_entries) for k, s in specs.items()}
        rc, src, log = gx.gx_jit_offline(programs.build(name, fds), maps)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    if rc == -38:
        pytest.skip(log)
    assert rc == 0, log[-2000:]
    return src


def test_codegen_decisions_offline():
    """The round-2 code-generation decisions, visible in the generated source:
    the per-thread key cache on P2's lane map (a value-start map, single program), 32-bit
    arithmetic and the PTX shift on P4's binary search (verifier intervals), the ring depth --
    4 stages, 2 for a single program that probes a hash map (P3) -- and none of it when disabled."""
    p2 = _jit_source("P2", GX_JIT_VMASK="1")
    assert "ptkc_switch<32u, 2u>" in p2 and "ptkc_flush(pkc" in p2
    assert "gx_full[4]" in p2
    assert "ptkc_switch" not in _jit_source("P2", GX_JIT_VMASK="1", GX_JIT_PTKC="0")
    p3 = _jit_source("P3", GX_JIT_VMASK="1")
    assert "gx_full[2]" in p3
    p4 = _jit_source("P4", GX_JIT_VMASK="4")
    assert "shr.b32" in p4 and "(uint64_t)(uint32_t)((uint32_t)r1 + (uint32_t)r9)" in p4
    assert "r8 = (uint64_t)(uint32_t)r8;" in p4          # block-entry re-statement at the loop head
    # the NULL test after an in-range ARRAY lookup is gone from the lookup itself
    assert "0x7f0200000000ull + (uint64_t)k * 8u;" in p4
