/*
 * gx_verifier.h -- host-side verifier + pre-decoder (internal interface of libgx).
 *
 * "We reuse Linux's eBPF verifier to enforce standard memory safety, bounded loops, and type
 * correctness. An additional verifier pass ... performs dataflow analysis on eBPF bytecode,
 * propagating warp-uniformity ... Control-flow constraints are enforced by traversing the
 * policy's CFG to reject lane-varying dependencies in branch predicates or loop bounds.
 * Map-update keys must be warp-uniform or warp-reduced." (§5.3; 282, §4.4.1)
 * The Linux verifier is not available here, so its needed subset is re-implemented:
 * SURVEY.md §8a a11 and §8c c.7 list the rules.
 */
#pragma once
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/gx.h"
#include "gx_internal.h"

struct GxMapInfo {
    bool valid = false;
    uint32_t type = 0, key_size = 0, value_size = 0, max_entries = 0;
};

/* per-map usage facts of one program (privatization and merge legality) */
struct GxMapUse {
    bool used = false;
    bool reads = false;          /* LDX, helper key/value/data reads, FETCH/XCHG/CMPXCHG */
    bool writes = false;         /* any modification */
    bool non_add_write = false;  /* a modification that is not an ATOMIC ADD */
    bool fetch_add = false;      /* ATOMIC ADD|FETCH */
    bool update_call = false;    /* bpf_map_update_elem */
    bool non_dw_atomic = false;  /* a 32-bit atomic (privatised accumulators are u64 words) */
    bool store = false;          /* a plain store or a non-ADD atomic (XCHG / CMPXCHG / OR / AND / XOR) */
    bool upd_overwrite = false;  /* an update_elem whose flags are not the constant BPF_NOEXIST */
};

struct GxVerifyResult {
    gx_verify_report report{};
    std::string log;
    std::vector<GxInsn> image;     /* pre-decoded program (same slot count) */
    std::vector<uint16_t> narrow_in; /* per image slot: registers r0..r9 holding a scalar below 2^32 on
                                        entry on every explored path (the JIT zero-extends them at
                                        block starts so the compiler keeps their upper halves known) */
    GxMapUse use[GX_MAX_MAPS];
    uint32_t stack_depth = 0;
};

/* Runs the verifier over n 8-byte slots.  Returns report.verdict. */
int gx_verify_program(const uint8_t *slots, uint32_t n, const GxMapInfo *maps, const gx_verify_opts &opts,
                      GxVerifyResult &out);

const char *gx_rule_name(uint32_t rule);
