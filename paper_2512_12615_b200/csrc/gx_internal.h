/*
 * gx_internal.h -- structures shared by the host runtime (gx_runtime.cpp, gx_verifier.cpp) and
 * the sm_100a kernels (gx_exec.cu, gx_maps.cu).  Not part of the public ABI (include/gx.h).
 */
#ifndef GX_INTERNAL_H
#define GX_INTERNAL_H

#include <stdint.h>

#define GX_MAX_MAPS 64
#define GX_MAX_PROGS 64
#define GX_MAX_LAUNCH_PROGS 16
#define GX_MAX_KINDS 8            /* attach table covers hook kinds 0..7 */
#define GX_STACK_SIZE 512
#define GX_MAX_STAGED_INSNS 2048  /* total pre-decoded slots staged in shared memory per launch */
#define GX_HASH_EMPTY 0xFFFFFFFFFFFFFFFFull
#define GX_NREGS 11
#define GX_FN_MEM_PREFETCH 1000   /* gdev_mem_prefetch helper id (F-1) */
#define GX_MAP_TYPE_PFQ 64        /* prefetch queue map type (F-2) */
#define GX_FN_PREFETCH_L2 1001    /* gdev_prefetch_l2 helper id (F-7) */
#define GX_MAP_TYPE_REGION 65     /* device region map: caller-owned device memory (F-7) */
/* request filter after a queue's records (F-2 set semantics): clamp(capacity, 2^12, 2^20) words,
 * the count carried in GxMapDesc.nshards / GxPublishItem.nshards */
#define GX_PFQ_FILTER_WORDS(cap) ((cap) < 4096u ? 4096u : (cap) > (1u << 20) ? (1u << 20) : (cap))

/* ---- pre-decoded instruction (16 B), produced by the verifier for the executor ----
 * Every field is warp-uniform on the fast path, so decode costs one broadcast LDS.128. */
struct GxInsn {
    uint8_t op;       /* handler id (GxOp) */
    uint8_t dst;      /* register index */
    uint8_t src;      /* register index */
    uint8_t flags;    /* GXF_* */
    int16_t off;      /* memory offset; ctx byte offset; stack slot index (see ops) */
    uint16_t aux;     /* branch target (absolute slot) / map fd / size code / stack byte */
    uint64_t imm;     /* immediate: sign-extended per class, merged ldimm64, relocated address */
};

/* flags */
#define GXF_X 0x01        /* source operand is a register (BPF_X) */
#define GXF_SX 0x02       /* sign-extending load (MEMSX) */
#define GXF_FETCH 0x04    /* atomic returns the old value */
#define GXF_W32 0x08      /* 32-bit atomic / memory width helper flag */
#define GXF_KEY_MAPV 0x10 /* helper key pointer is a map value (else stack slot in off) */
#define GXF_PT_VSTART 0x10 /* per-thread memory ops: the base register is a value start on every
                              path (the access is word off >> 3 of the value; JIT register cache) */
#define GXF_VAL_MAPV 0x20 /* helper value/data pointer is a map value (else stack slot) */
#define GXF_PRIV 0x40     /* atomic target map is privatized in shared memory */
#define GXF_NARROW 0x20   /* ALU64: operands and result below 2^32 on every explored path (the verifier's
                             intervals), so the 32-bit operation, zero-extended, is exact */
#define GXF_UNIFORM 0x80  /* verifier: branch operands are warp-uniform (hint) */

/* sizes: aux low bits for memory ops = log2(size) */

enum GxOp : uint8_t {
    GX_OP_NOP = 0,
    /* ALU64 (imm sign-extended; GXF_X selects register) */
    GX_ADD64, GX_SUB64, GX_MUL64, GX_DIV64, GX_SDIV64, GX_MOD64, GX_SMOD64, GX_OR64, GX_AND64,
    GX_XOR64, GX_LSH64, GX_RSH64, GX_ARSH64, GX_NEG64, GX_MOV64, GX_MOVSX64,
    /* ALU32 (imm = (u32)imm) */
    GX_ADD32, GX_SUB32, GX_MUL32, GX_DIV32, GX_SDIV32, GX_MOD32, GX_SMOD32, GX_OR32, GX_AND32,
    GX_XOR32, GX_LSH32, GX_RSH32, GX_ARSH32, GX_NEG32, GX_MOV32, GX_MOVSX32,
    GX_LE, GX_BE,                 /* END TO_LE (truncate) / TO_BE and BSWAP (swap); aux = width */
    GX_LDIMM,                     /* dst = imm (64-bit); consumes two slots */
    /* jumps: aux = absolute target */
    GX_JA,
    GX_JEQ, GX_JNE, GX_JGT, GX_JGE, GX_JLT, GX_JLE, GX_JSGT, GX_JSGE, GX_JSLT, GX_JSLE, GX_JSET,
    GX_JEQ32, GX_JNE32, GX_JGT32, GX_JGE32, GX_JLT32, GX_JLE32, GX_JSGT32, GX_JSGE32, GX_JSLT32,
    GX_JSLE32, GX_JSET32,
    GX_EXIT,
    /* loads: aux = log2(size); GXF_SX */
    GX_LDX_CTX,                   /* off = ctx byte offset */
    GX_LDX_STACK,                 /* off = stack byte address in [0,512) (constant) */
    GX_LDX_MAP,                   /* global: ea = r[src] + off */
    GX_LDX_PT,                    /* per-thread map value: logical ea = r[src] + off; imm = map fd */
    /* stores: aux = log2(size); value = r[src] (STX) or imm (ST, GXF_X clear) */
    GX_ST_STACK, GX_ST_MAP, GX_ST_PT,
    /* atomics: aux = log2(size) (2 or 3); imm = BPF atomic op code; GXF_FETCH; dst = address reg */
    GX_ATOM_STACK,                /* per-lane private: plain RMW */
    GX_ATOM_MAP,                  /* global map value: warp-aggregated atomics */
    GX_ATOM_PRIV,                 /* privatized ARRAY in shared memory; imm low byte = op, aux hi = fd */
    GX_ATOM_PT,                   /* per-thread map: plain RMW on the lane's shard */
    /* helper calls: aux = map fd; off = key stack address (or GXF_KEY_MAPV); imm = value stack
     * address (update) / data stack address + size<<32 (ringbuf) */
    GX_CALL_LOOKUP_ARRAY, GX_CALL_LOOKUP_PT, GX_CALL_LOOKUP_HASH,
    GX_CALL_UPDATE_ARRAY, GX_CALL_UPDATE_PT, GX_CALL_UPDATE_HASH,
    GX_CALL_RINGBUF_OUTPUT,
    GX_CALL_MEM_PREFETCH,         /* gdev_mem_prefetch(queue = aux, addr = r2, len = r3) (f2) */
    GX_CALL_PREFETCH_L2,          /* gdev_prefetch_l2(region = aux, addr = r2, len = r3) (f2) */
    GX_OP_COUNT
};

/* ---- device-side map descriptor ---- */
struct GxMapDesc {
    uint64_t data;         /* ARRAY: values; PT: shards [word][shard]; HASH: slots (cap+1) x 16 B;
                              RINGBUF: bytes; PREFETCH QUEUE: 16-B requests; REGION: base */
    uint64_t aux;          /* HASH: u64 counters {count}; RINGBUF: u64 {prod, used};
                              PREFETCH QUEUE: u64 {reserved}; REGION: byte length */
    uint32_t type, key_size, value_size, max_entries;
    uint32_t nshards;      /* PT: shards; PREFETCH QUEUE: request-filter words (a power of two) */
    uint32_t cap_mask;     /* HASH: capacity-1; RINGBUF: capacity-1; PREFETCH QUEUE: capacity-1 */
    uint32_t priv_off;     /* byte offset of the privatized copy in shared memory, or ~0u */
    uint32_t coherent;     /* 1: written during this launch -> loads bypass L1 */
};

struct GxProgDesc {
    uint64_t image;        /* device pointer to GxInsn[n] */
    uint32_t n;            /* slots */
    uint32_t smem_off;     /* staged offset (insns) in the shared program area */
};

struct GxLaunch {
    GxMapDesc maps[GX_MAX_MAPS];
    GxProgDesc progs[GX_MAX_LAUNCH_PROGS];
    int8_t attach[GX_MAX_KINDS][256];  /* (kind, tenant) -> launch prog slot, -1 none */
    uint32_t n_progs;
    int32_t single;                    /* launch prog slot for all events, or -1 */
    uint32_t staged_insns;             /* total slots staged in shared memory */
    uint32_t stack_slots;              /* per-lane 8-byte stack slots reserved */
    uint32_t priv_bytes;               /* privatized map bytes per block */
    uint32_t n_priv;                   /* privatized maps: indices in priv_maps */
    uint32_t priv_maps[8];
    uint32_t pad;
    uint64_t stats;                    /* device u64[8] counters (gx_batch_stats order) */
};

/* one item of a runtime-daemon publish point (gx_maps.cu publish_kernel) */
struct GxPublishItem {
    uint64_t data, aux;    /* device storage / counters of the map */
    uint64_t host_off;     /* byte offset in the host slot */
    uint64_t cap;          /* prefetch queue capacity (requests) */
    uint32_t kind;         /* 0 prefetch queue, 1 ARRAY (or a folded PERTHREAD staging copy) */
    uint32_t K, W;         /* entries, u64 words per value */
    uint32_t nshards;
};

enum { GXS_RUN = 0, GXS_SKIP, GXS_DIVERGENT, GXS_HERR, GXS_RB_BYTES, GXS_RB_DROPS, GXS_HFULL, GXS_STEPS,
       GXS_BOUNDS,             /* GX_JIT_BOUNDS=1: map accesses outside their map (redirected, counted) */
       GXS_SCRATCH = 15,       /* where a redirected access lands */
       GXS_N = 16 };

#endif
