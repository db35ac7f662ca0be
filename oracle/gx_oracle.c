/*
 * gx_oracle.c -- the CPU ORACLE for the gx device-side eBPF runtime.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with paper_2512_12615_b200/ (the CUDA path) and neither
 * includes nor links the other.
 *
 * What it computes (the plain definition):
 *     for e = 0 .. N-1 in index order (or a caller-given permutation):
 *         pick the program (prog >= 0, else the attach table on the event's hook word);
 *         run it to EXIT on ctx = &event[e] against the persistent map environment;
 *         record R0[e].
 *     outputs: R0[], the canonical state of every map, the ringbuf record multiset, stats.
 * This is PAPER.md:286's "preserving eBPF's scalar semantics": every event runs the
 * program once, sequentially, with no warp aggregation, no sharding, no blocking.
 *
 * The instruction semantics are the standard eBPF ones (PAPER.md:185, 277, 310:
 * programs come from clang/libbpf and are checked by the Linux verifier), written
 * step by step from SURVEY.md §8c O1..O10 and the readings I-1..I-28 listed in
 * DESIGN.md §3.  Each function cites the passage it follows.
 *
 * Pointer model (O7): every register and every 8-byte stack slot carries a shadow
 * tag; every memory access is bounds/alignment/initialisation checked against the
 * region it points into.  A violation is an ORACLE FAULT (the run stops, ora_fault()
 * says where): it means the verifier accepted an unsafe program.
 *
 * Parity status: pinned (tests/test_oracle_*.py) except the items of SURVEY.md §8c c.6
 * ("parity unpinned": per-shard per-thread values, helper_errors, ORDER_SENSITIVE outputs).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

#define ORA_EXPORT __attribute__((visibility("default")))

/* ---- constants from bpf.h / bpf_common.h (restated, not included) ---- */
enum { CL_LD = 0, CL_LDX = 1, CL_ST = 2, CL_STX = 3, CL_ALU = 4, CL_JMP = 5, CL_JMP32 = 6, CL_ALU64 = 7 };
enum { MAP_HASH = 1, MAP_ARRAY = 2, MAP_PT = 6, MAP_RINGBUF = 27, MAP_PFQ = 64, MAP_REGION = 65 };
/* gdev_mem_prefetch (§4.3.1 listing "Request prefetch, triggers handler in host
 * driver"), this build's helper id (reading F-1) */
enum { FN_MEM_PREFETCH = 1000 };
/* gdev_prefetch_l2 ("Device-side L2 prefetch instructions (prefetch.global.L2)"),
 * this build's helper id (reading F-7) */
enum { FN_PREFETCH_L2 = 1001 };
enum { E_NOENT = 2, E_2BIG = 7, E_AGAIN = 11, E_NOMEM = 12, E_FAULT = 14, E_EXIST = 17, E_INVAL = 22 };
#define STACK_SIZE 512
#define POISON 0xDEADBEEFDEADBEEFull
#define MAX_MAPS 64
#define MAX_PROGS 64
#define MAX_STEPS 10000000ull   /* per event; a verified program never gets close */

/* shadow tags (O7) */
enum { T_UNINIT = 0, T_SCALAR, T_CTX, T_STACK, T_MAPH, T_MAPV };

typedef struct {
    uint64_t v;      /* scalar value, or the byte offset of a pointer inside its region */
    int tag;
    int map;         /* T_MAPH / T_MAPV: map fd */
    uint8_t *base;   /* T_MAPV: start of the value region */
} reg_t;

typedef struct hnode {
    struct hnode *next;
    uint8_t *key;
    uint8_t *val;
} hnode;

typedef struct {
    int used;
    uint32_t type, key_size, value_size, max_entries;
    /* ARRAY */
    uint8_t *data;
    /* PERTHREAD ARRAY: shards[s] = max_entries*value_size bytes */
    uint8_t **shards;
    uint32_t nshards;
    /* HASH: separate chaining, nodes never move (value pointers stay valid) */
    hnode **buckets;
    uint64_t nbuckets, count;
    /* RINGBUF: Linux-style records, header {u32 len, u32 pg_off} + payload padded to 8 */
    uint8_t *rb;
    uint64_t rb_used;
    /* PREFETCH QUEUE (F-2): requests {u64 first_page, u32 npages, u32 0} in call order */
    uint64_t *pfq;          /* 2 words per request */
    uint64_t pfq_n;
    /* REGION (F-7): the device byte range [region_base, region_base + region_len) */
    uint64_t region_base, region_len;
} map_t;

typedef struct {
    int used;
    uint32_t n;          /* slots */
    uint8_t *code;       /* per slot */
    uint8_t *dst, *src;
    int16_t *off;
    int32_t *imm;
} prog_t;

typedef struct ora_env {
    map_t maps[MAX_MAPS];
    prog_t progs[MAX_PROGS];
    int attach[256][256];     /* (hook kind, tenant) -> prog, -1 none */
    uint32_t pt_shards;       /* O10 --pt-shards S */
    uint64_t stats[8];        /* events_run, events_skipped, ringbuf_drops, hash_full, helper_errors, insns */
    char fault[256];
    int faulted;
} ora_env;

enum { ST_RUN = 0, ST_SKIP, ST_DROPS, ST_HFULL, ST_HERR, ST_INSNS };

/* event i goes to per-thread shard mix64(i) mod S (SplitMix64 finalizer) */
static uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

static int fault(ora_env *env, uint64_t ev, uint32_t pc, const char *why) {
    if (!env->faulted)
        snprintf(env->fault, sizeof env->fault, "event %llu pc %u: %s", (unsigned long long)ev, pc, why);
    env->faulted = 1;
    return -1;
}

/* ------------------------------------------------------------------ environment */

ORA_EXPORT ora_env *ora_new(void) {
    ora_env *e = calloc(1, sizeof *e);
    if (!e) return NULL;
    for (int k = 0; k < 256; k++)
        for (int t = 0; t < 256; t++) e->attach[k][t] = -1;
    e->pt_shards = 1;
    return e;
}

static void map_free(map_t *m) {
    free(m->data);
    free(m->pfq);
    if (m->shards) {
        for (uint32_t s = 0; s < m->nshards; s++) free(m->shards[s]);
        free(m->shards);
    }
    if (m->buckets) {
        for (uint64_t b = 0; b < m->nbuckets; b++) {
            hnode *n = m->buckets[b];
            while (n) { hnode *nx = n->next; free(n->key); free(n->val); free(n); n = nx; }
        }
        free(m->buckets);
    }
    free(m->rb);
    memset(m, 0, sizeof *m);
}

ORA_EXPORT void ora_free(ora_env *e) {
    if (!e) return;
    for (int i = 0; i < MAX_MAPS; i++) if (e->maps[i].used) map_free(&e->maps[i]);
    for (int i = 0; i < MAX_PROGS; i++) if (e->progs[i].used) {
        prog_t *p = &e->progs[i];
        free(p->code); free(p->dst); free(p->src); free(p->off); free(p->imm);
    }
    free(e);
}

ORA_EXPORT const char *ora_fault(ora_env *e) { return e->faulted ? e->fault : ""; }
ORA_EXPORT void ora_clear_fault(ora_env *e) { e->faulted = 0; e->fault[0] = 0; }
ORA_EXPORT void ora_stats(ora_env *e, uint64_t out[8]) { memcpy(out, e->stats, sizeof e->stats); }
ORA_EXPORT void ora_reset_stats(ora_env *e) { memset(e->stats, 0, sizeof e->stats); }

/* ------------------------------------------------------------------ maps (bpf.h:925-965) */

static int pt_ensure_shards(map_t *m, uint32_t S) {
    if (m->nshards >= S) return 0;
    uint8_t **ns = realloc(m->shards, (size_t)S * sizeof *ns);
    if (!ns) return -E_NOMEM;
    m->shards = ns;
    for (uint32_t s = m->nshards; s < S; s++) {
        m->shards[s] = calloc((size_t)m->max_entries, m->value_size);
        if (!m->shards[s]) return -E_NOMEM;
    }
    m->nshards = S;
    return 0;
}

/* Map specs accepted (SURVEY.md §8b gx_map_spec comment). Returns the fd or -errno. */
ORA_EXPORT int ora_map_create(ora_env *e, uint32_t type, uint32_t key_size, uint32_t value_size,
                              uint32_t max_entries) {
    int fd = -1;
    for (int i = 0; i < MAX_MAPS; i++) if (!e->maps[i].used) { fd = i; break; }
    if (fd < 0) return -E_NOMEM;
    map_t *m = &e->maps[fd];
    memset(m, 0, sizeof *m);
    m->type = type; m->key_size = key_size; m->value_size = value_size; m->max_entries = max_entries;
    switch (type) {
    case MAP_ARRAY:
        if (key_size != 4 || value_size == 0 || value_size % 8 || max_entries == 0) return -E_INVAL;
        m->data = calloc((size_t)max_entries, value_size);
        if (!m->data) return -E_NOMEM;
        break;
    case MAP_PT:
        if (key_size != 4 || value_size == 0 || value_size % 8 || value_size > 256 || max_entries == 0)
            return -E_INVAL;
        if (pt_ensure_shards(m, e->pt_shards)) return -E_NOMEM;
        break;
    case MAP_HASH:
        if ((key_size != 4 && key_size != 8) || value_size == 0 || value_size % 8 || value_size > 256 ||
            max_entries == 0)
            return -E_INVAL;
        m->nbuckets = 1;
        while (m->nbuckets < 2ull * max_entries) m->nbuckets <<= 1;
        m->buckets = calloc(m->nbuckets, sizeof *m->buckets);
        if (!m->buckets) return -E_NOMEM;
        break;
    case MAP_RINGBUF:
        if (key_size || value_size || max_entries < 4096 || (max_entries & (max_entries - 1))) return -E_INVAL;
        m->rb = calloc(max_entries, 1);
        if (!m->rb) return -E_NOMEM;
        break;
    case MAP_PFQ:   /* capacity in requests: a power of two in [64, 2^24] (F-2) */
        if (key_size || value_size || max_entries < 64 || max_entries > (1u << 24) || (max_entries & (max_entries - 1)))
            return -E_INVAL;
        m->pfq = calloc(2 * (size_t)max_entries, sizeof(uint64_t));
        if (!m->pfq) return -E_NOMEM;
        break;
    default:
        return -E_INVAL;
    }
    m->used = 1;
    return fd;
}

static uint64_t key_u64(const map_t *m, const uint8_t *key) {
    uint64_t k = 0;
    memcpy(&k, key, m->key_size);   /* little endian host */
    return k;
}

static hnode *hash_find(map_t *m, const uint8_t *key) {
    uint64_t b = mix64(key_u64(m, key)) & (m->nbuckets - 1);
    for (hnode *n = m->buckets[b]; n; n = n->next)
        if (!memcmp(n->key, key, m->key_size)) return n;
    return NULL;
}

static hnode *hash_insert(map_t *m, const uint8_t *key) {
    uint64_t b = mix64(key_u64(m, key)) & (m->nbuckets - 1);
    hnode *n = calloc(1, sizeof *n);
    if (!n) return NULL;
    n->key = malloc(m->key_size);
    n->val = calloc(1, m->value_size);
    memcpy(n->key, key, m->key_size);
    n->next = m->buckets[b];
    m->buckets[b] = n;
    m->count++;
    return n;
}

/* bpf_map_lookup_elem (helper 1) semantics, bpf.h:1753-1760; SURVEY.md O6.  NULL if absent. */
static uint8_t *map_lookup(map_t *m, const uint8_t *key, uint32_t shard) {
    if (m->type == MAP_ARRAY || m->type == MAP_PT) {
        uint32_t k;
        memcpy(&k, key, 4);
        if (k >= m->max_entries) return NULL;
        if (m->type == MAP_ARRAY) return m->data + (uint64_t)k * m->value_size;
        return m->shards[shard] + (uint64_t)k * m->value_size;
    }
    if (m->type == MAP_HASH) {
        hnode *n = hash_find(m, key);
        return n ? n->val : NULL;
    }
    return NULL;
}

/* bpf_map_update_elem (helper 2) semantics, bpf.h:1762-1776 and 1300-1302; SURVEY.md O6.
 * ARRAY/PT: flags must be ANY(0)/NOEXIST(1)/EXIST(2); NOEXIST -> -EEXIST (elements always exist);
 * key >= max -> -E2BIG.  HASH: present+NOEXIST -> -EEXIST; absent+EXIST -> -ENOENT;
 * absent and count == max_entries -> -E2BIG (hash_full). */
static int map_update(ora_env *e, map_t *m, const uint8_t *key, const uint8_t *val, uint64_t flags,
                      uint32_t shard) {
    if (flags > 2) return -E_INVAL;
    if (m->type == MAP_ARRAY || m->type == MAP_PT) {
        uint32_t k;
        memcpy(&k, key, 4);
        if (k >= m->max_entries) return -E_2BIG;
        if (flags == 1) return -E_EXIST;
        uint8_t *dst = (m->type == MAP_ARRAY) ? m->data + (uint64_t)k * m->value_size
                                                : m->shards[shard] + (uint64_t)k * m->value_size;
        memcpy(dst, val, m->value_size);
        return 0;
    }
    if (m->type == MAP_HASH) {
        hnode *n = hash_find(m, key);
        if (n) {
            if (flags == 1) return -E_EXIST;
            memcpy(n->val, val, m->value_size);
            return 0;
        }
        if (flags == 2) return -E_NOENT;
        if (m->count >= m->max_entries) { e->stats[ST_HFULL]++; return -E_2BIG; }
        n = hash_insert(m, key);
        if (!n) return -E_NOMEM;
        memcpy(n->val, val, m->value_size);
        return 0;
    }
    return -E_INVAL;
}

/* gx_region_map: a device range for gdev_prefetch_l2 (F-7).  Returns the fd or -errno. */
ORA_EXPORT int ora_region_map(ora_env *e, uint64_t base, uint64_t len) {
    if (base == 0 || len == 0 || base + len < base) return -E_INVAL;
    int fd = -1;
    for (int i = 0; i < MAX_MAPS; i++) if (!e->maps[i].used) { fd = i; break; }
    if (fd < 0) return -E_NOMEM;
    map_t *m = &e->maps[fd];
    memset(m, 0, sizeof *m);
    m->type = MAP_REGION;
    m->max_entries = 1;
    m->region_base = base;
    m->region_len = len;
    m->used = 1;
    return fd;
}

/* gdev_prefetch_l2(region, addr, len) (F-7).  The prefetch itself is a hint
 * with no observable effect; the result is the only output: -EINVAL unless 1 <= len <= 64 KiB,
 * else -EFAULT unless region_base <= addr and addr + len <= region_base + region_len (in exact
 * 128-bit arithmetic), else 0. */
static int64_t prefetch_l2(const map_t *m, uint64_t addr, uint64_t len) {
    if (len == 0 || len > 65536) return -E_INVAL;
    if (addr < m->region_base) return -E_FAULT;
    if ((unsigned __int128)addr + len > (unsigned __int128)m->region_base + m->region_len) return -E_FAULT;
    return 0;
}

/* Host control-plane write (SURVEY.md §8b gx_update_map): per-thread maps write shard 0 and
 * zero the other shards (§8c S4). */
ORA_EXPORT int ora_map_update(ora_env *e, int fd, const void *key, const void *val, uint64_t flags) {
    if (fd < 0 || fd >= MAX_MAPS || !e->maps[fd].used) return -E_INVAL;
    map_t *m = &e->maps[fd];
    if (m->type == MAP_RINGBUF || m->type == MAP_PFQ || m->type == MAP_REGION) return -E_INVAL;
    int r = map_update(e, m, key, val, flags, 0);
    if (r == 0 && m->type == MAP_PT) {
        uint32_t k;
        memcpy(&k, key, 4);
        for (uint32_t s = 1; s < m->nshards; s++) memset(m->shards[s] + (uint64_t)k * m->value_size, 0, m->value_size);
    }
    return r;
}

/* host control plane, n entries (keys / values packed back to back): ora_map_update per entry in
 * order; stops at the first error and returns it */
ORA_EXPORT int ora_map_update_n(ora_env *e, int fd, const void *keys, const void *vals, uint64_t n, uint64_t flags) {
    if (fd < 0 || fd >= MAX_MAPS || !e->maps[fd].used) return -E_INVAL;
    const uint8_t *kp = keys, *vp = vals;
    const uint32_t ks = e->maps[fd].key_size, vs = e->maps[fd].value_size;
    for (uint64_t i = 0; i < n; i++) {
        int r = ora_map_update(e, fd, kp + i * ks, vp + i * vs, flags);
        if (r) return r;
    }
    return 0;
}

/* bpf_ringbuf_output (helper 130), bpf.h:4407-4422, 6050-6051, 6064-6066; SURVEY.md O6:
 * flags in {0, NO_WAKEUP 1, FORCE_WAKEUP 2}; rec = roundup8(8 + size); if used + rec > capacity
 * the record is dropped (-EAGAIN) else appended with header {len, pg_off}. */
static int ringbuf_output(ora_env *e, map_t *m, const uint8_t *data, uint64_t size, uint64_t flags) {
    if (flags > 2) return -E_INVAL;
    uint64_t rec = (8 + size + 7) & ~7ull;
    if (m->rb_used + rec > m->max_entries) { e->stats[ST_DROPS]++; return -E_AGAIN; }
    uint32_t hdr[2] = {(uint32_t)size, (uint32_t)(m->rb_used / 4096)};
    memcpy(m->rb + m->rb_used, hdr, 8);
    memset(m->rb + m->rb_used + 8, 0, rec - 8);
    memcpy(m->rb + m->rb_used + 8, data, size);
    m->rb_used += rec;
    return 0;
}

/* gdev_mem_prefetch(queue, addr, len) (F-1..F-3): the region is the
 * run of 4-KiB pages [addr >> 12, (addr + len - 1) >> 12] ("finer-grained 4KB pages",
 * 303 "prefetch hooks operate at page granularity"), at most 2 MiB (one UVM chunk).  len == 0,
 * len > 2 MiB or addr + len past 2^64 -> -EINVAL, nothing queued; a full queue -> -EAGAIN (the
 * request is dropped and counted); else the request {first_page, npages} is appended -> 0. */
static int mem_prefetch(ora_env *e, map_t *m, uint64_t addr, uint64_t len) {
    if (len == 0 || len > (2ull << 20) || addr + len < addr) return -E_INVAL;
    const uint64_t first = addr >> 12, last = (addr + len - 1) >> 12;
    if (m->pfq_n >= m->max_entries) { e->stats[ST_DROPS]++; return -E_AGAIN; }
    m->pfq[2 * m->pfq_n] = first;
    m->pfq[2 * m->pfq_n + 1] = last - first + 1;
    m->pfq_n++;
    return 0;
}

/* ------------------------------------------------------------------ programs (O1, O2) */

/* Copy the slots; structural decode only (the oracle does not verify).  Pseudo map
 * sources of ldimm64 are resolved at run time (O2). Returns prog id or -errno. */
ORA_EXPORT int ora_prog_load(ora_env *e, const void *slots, uint32_t n) {
    int id = -1;
    for (int i = 0; i < MAX_PROGS; i++) if (!e->progs[i].used) { id = i; break; }
    if (id < 0 || n == 0) return -E_INVAL;
    prog_t *p = &e->progs[id];
    p->n = n;
    p->code = malloc(n); p->dst = malloc(n); p->src = malloc(n);
    p->off = malloc(n * sizeof(int16_t)); p->imm = malloc(n * sizeof(int32_t));
    const uint8_t *b = slots;
    for (uint32_t i = 0; i < n; i++) {   /* struct bpf_insn, bpf.h:72-77, little endian */
        p->code[i] = b[8 * i];
        p->dst[i] = b[8 * i + 1] & 0xF;
        p->src[i] = b[8 * i + 1] >> 4;
        int16_t off; int32_t imm;
        memcpy(&off, b + 8 * i + 2, 2);
        memcpy(&imm, b + 8 * i + 4, 4);
        p->off[i] = off; p->imm[i] = imm;
    }
    p->used = 1;
    return id;
}

/* attach table (hook kind, tenant) -> program */
ORA_EXPORT int ora_attach(ora_env *e, int prog, uint32_t kind, uint32_t tenant) {
    if (kind > 255 || tenant > 255) return -E_INVAL;
    e->attach[kind][tenant] = prog;
    return 0;
}

ORA_EXPORT int ora_set_pt_shards(ora_env *e, uint32_t S) {
    if (S == 0) return -E_INVAL;
    e->pt_shards = S;
    for (int i = 0; i < MAX_MAPS; i++)
        if (e->maps[i].used && e->maps[i].type == MAP_PT && pt_ensure_shards(&e->maps[i], S)) return -E_NOMEM;
    return 0;
}

/* ------------------------------------------------------------------ interpreter (O4-O7) */

typedef struct {
    ora_env *env;
    const uint8_t *ctx;          /* 32-byte event record, read-only */
    uint8_t stack[STACK_SIZE];
    uint8_t sinit[STACK_SIZE];   /* per-byte initialised flag */
    reg_t sspill[STACK_SIZE / 8];/* per 8-byte slot: spilled pointer (tag != SCALAR) */
    reg_t r[11];
    uint64_t ev;                 /* original event index (fault reports, shard choice) */
    uint32_t shard;
} vm_t;

/* Resolve the region a pointer register addresses; check [v+off, v+off+size) and alignment.
 * Returns a host pointer to the bytes or NULL (fault). */
static uint8_t *mem_addr(vm_t *vm, const reg_t *p, int64_t off, uint32_t size, int write, uint32_t pc) {
    int64_t a = (int64_t)p->v + off;
    uint64_t lim;
    uint8_t *base;
    switch (p->tag) {
    case T_CTX:
        if (write) { fault(vm->env, vm->ev, pc, "write to ctx"); return NULL; }
        lim = 32; base = (uint8_t *)vm->ctx; break;
    case T_STACK:
        lim = STACK_SIZE; base = vm->stack; break;
    case T_MAPV:
        lim = vm->env->maps[p->map].value_size; base = p->base; break;
    default:
        fault(vm->env, vm->ev, pc, "memory access through a non-pointer");
        return NULL;
    }
    if (a < 0 || (uint64_t)a + size > lim) { fault(vm->env, vm->ev, pc, "out-of-bounds access"); return NULL; }
    if ((uint64_t)a % size) { fault(vm->env, vm->ev, pc, "misaligned access"); return NULL; }
    if (p->tag == T_STACK && !write) {
        for (uint32_t k = 0; k < size; k++)
            if (!vm->sinit[a + k]) { fault(vm->env, vm->ev, pc, "read of uninitialised stack"); return NULL; }
    }
    return base + a;
}

/* BPF_SIZE(code) = code & 0x18: W 0x00 -> 4 B, H 0x08 -> 2 B, B 0x10 -> 1 B, DW 0x18 -> 8 B
 * (bpf_common.h:17-20, bpf.h:21). */
static uint32_t size_of(uint8_t code) {
    static const uint32_t sz[4] = {4, 2, 1, 8};
    return sz[(code >> 3) & 3];
}

static uint64_t load_le(const uint8_t *p, uint32_t size) {
    uint64_t v = 0;
    memcpy(&v, p, size);
    return v;
}
static void store_le(uint8_t *p, uint32_t size, uint64_t v) { memcpy(p, &v, size); }

static uint64_t sext(uint64_t v, uint32_t bits) {
    if (bits >= 64) return v;
    uint64_t m = 1ull << (bits - 1);
    v &= (1ull << bits) - 1;
    return (v ^ m) - m;
}

static uint64_t bswap(uint64_t v, int bits) {
    uint64_t r = 0;
    for (int i = 0; i < bits / 8; i++) r |= ((v >> (8 * i)) & 0xFF) << (bits - 8 - 8 * i);
    return r;
}

/* Mark a stack write: bytes become initialised scalars; any pointer spill in a touched slot dies. */
static void stack_wrote(vm_t *vm, int64_t a, uint32_t size) {
    for (uint32_t k = 0; k < size; k++) vm->sinit[a + k] = 1;
    for (int64_t s = a / 8; s <= (int64_t)(a + size - 1) / 8; s++) vm->sspill[s].tag = T_SCALAR;
}

/* Reads `n` bytes behind a helper argument pointer (key, value, ringbuf data). */
static const uint8_t *arg_bytes(vm_t *vm, const reg_t *p, uint32_t n, uint32_t pc) {
    if (p->tag != T_STACK && p->tag != T_MAPV) { fault(vm->env, vm->ev, pc, "helper arg is not a stack/map-value pointer"); return NULL; }
    int64_t a = (int64_t)p->v;
    uint64_t lim = p->tag == T_STACK ? STACK_SIZE : vm->env->maps[p->map].value_size;
    if (a < 0 || (uint64_t)a + n > lim) { fault(vm->env, vm->ev, pc, "helper arg out of bounds"); return NULL; }
    if (p->tag == T_STACK) {
        for (uint32_t k = 0; k < n; k++) if (!vm->sinit[a + k]) { fault(vm->env, vm->ev, pc, "helper reads uninitialised stack"); return NULL; }
        for (int64_t s = a / 8; s <= (int64_t)(a + n - 1) / 8; s++)
            if (vm->sspill[s].tag != T_SCALAR) { fault(vm->env, vm->ev, pc, "helper reads a spilled pointer"); return NULL; }
        return vm->stack + a;
    }
    return p->base + a;
}

static int scalar(const reg_t *r) { return r->tag == T_SCALAR; }

/* ALU semantics, SURVEY.md §8c O5 table (RFC 9669 reading, I-3..I-6). W = 64 or 32. */
static int alu(uint32_t op, int is64, int16_t off, uint64_t d, uint64_t s, uint64_t *out) {
    uint64_t mask = is64 ? ~0ull : 0xFFFFFFFFull;
    int W = is64 ? 64 : 32;
    d &= mask; s &= mask;
    uint64_t sd = sext(d, W), ss = sext(s, W);   /* signed views as 64-bit two's complement */
    uint64_t intmin = is64 ? 0x8000000000000000ull : 0xFFFFFFFF80000000ull;
    uint64_t r;
    switch (op) {
    case 0x00: r = d + s; break;
    case 0x10: r = d - s; break;
    case 0x20: r = d * s; break;
    case 0x30:
        if (off == 0) r = s ? d / s : 0;
        else if (off == 1) {   /* SDIV (v4) */
            if (s == 0) r = 0;
            else if (sd == intmin && ss == ~0ull) r = sd;      /* INT_MIN / -1 = INT_MIN (I-4) */
            else r = (uint64_t)((int64_t)sd / (int64_t)ss);    /* C division truncates toward zero */
        } else return -1;
        break;
    case 0x90:
        if (off == 0) r = s ? d % s : d;
        else if (off == 1) {   /* SMOD (v4): sign of the dividend */
            if (s == 0) r = d;
            else if (ss == ~0ull) r = 0;
            else r = (uint64_t)((int64_t)sd % (int64_t)ss);
        } else return -1;
        break;
    case 0x40: r = d | s; break;
    case 0x50: r = d & s; break;
    case 0xA0: r = d ^ s; break;
    case 0x60: r = d << (s & (uint64_t)(W - 1)); break;
    case 0x70: r = d >> (s & (uint64_t)(W - 1)); break;
    case 0xC0: r = (uint64_t)((int64_t)sd >> (s & (uint64_t)(W - 1))); break;   /* arithmetic shift of the W-bit value */
    case 0x80: r = 0 - d; break;
    case 0xB0:
        if (off == 0) r = s;
        else if (off == 8 || off == 16 || (off == 32 && is64)) r = sext(s, (uint32_t)off);
        else return -1;
        break;
    default: return -1;
    }
    *out = r & mask;   /* ALU32 results are zero-extended (I-6) */
    return 0;
}

/* Conditional jump predicate (O5 jump table). */
static int jcond(uint32_t op, int is64, uint64_t d, uint64_t s, int *taken) {
    if (!is64) { d &= 0xFFFFFFFFull; s &= 0xFFFFFFFFull; }
    int W = is64 ? 64 : 32;
    int64_t sd = (int64_t)sext(d, W), ss = (int64_t)sext(s, W);
    switch (op) {
    case 0x10: *taken = d == s; break;
    case 0x50: *taken = d != s; break;
    case 0x20: *taken = d > s; break;
    case 0x30: *taken = d >= s; break;
    case 0xA0: *taken = d < s; break;
    case 0xB0: *taken = d <= s; break;
    case 0x60: *taken = sd > ss; break;
    case 0x70: *taken = sd >= ss; break;
    case 0xC0: *taken = sd < ss; break;
    case 0xD0: *taken = sd <= ss; break;
    case 0x40: *taken = (d & s) != 0; break;
    default: return -1;
    }
    return 0;
}

static void clobber_args(vm_t *vm) {
    for (int i = 1; i <= 5; i++) { vm->r[i].tag = T_UNINIT; vm->r[i].v = POISON; }
}

/* Runs one program on one event (O4 init, O5 loop). Returns 0 and *r0, or -1 on oracle fault. */
static int run_one(ora_env *env, prog_t *p, const uint8_t *ctx, uint64_t ev, uint64_t *r0) {
    vm_t vmv, *vm = &vmv;
    vm->env = env; vm->ctx = ctx; vm->ev = ev;
    vm->shard = env->pt_shards > 1 ? (uint32_t)(mix64(ev) % env->pt_shards) : 0;
    memset(vm->stack, 0xA5, sizeof vm->stack);       /* O4: stack poisoned, uninitialised */
    memset(vm->sinit, 0, sizeof vm->sinit);
    for (int s = 0; s < STACK_SIZE / 8; s++) vm->sspill[s].tag = T_SCALAR;
    for (int i = 0; i < 11; i++) { vm->r[i].tag = T_UNINIT; vm->r[i].v = POISON; vm->r[i].map = -1; vm->r[i].base = NULL; }
    vm->r[1].tag = T_CTX; vm->r[1].v = 0;              /* r1 = ctx */
    vm->r[10].tag = T_STACK; vm->r[10].v = STACK_SIZE; /* r10 = frame pointer (read-only) */

    uint32_t pc = 0;
    uint64_t steps = 0;
    for (;;) {
        if (pc >= p->n) return fault(env, ev, pc, "pc out of program");
        if (++steps > MAX_STEPS) return fault(env, ev, pc, "step limit (unbounded loop?)");
        env->stats[ST_INSNS]++;
        uint8_t code = p->code[pc];
        uint32_t cls = code & 7, dst = p->dst[pc], src = p->src[pc];
        int16_t off = p->off[pc];
        int32_t imm = p->imm[pc];
        if (dst > 10 || src > 10) return fault(env, ev, pc, "bad register");
        reg_t *D = &vm->r[dst], *S = &vm->r[src];

        if (cls == CL_ALU || cls == CL_ALU64) {
            int is64 = cls == CL_ALU64;
            uint32_t op = code & 0xF0;
            int x = (code & 0x08) != 0;
            if (dst == 10) return fault(env, ev, pc, "write to r10");
            if (op == 0xD0) {                                    /* END / BSWAP */
                if (!scalar(D)) return fault(env, ev, pc, "END on non-scalar");
                if (imm != 16 && imm != 32 && imm != 64) return fault(env, ev, pc, "bad END width");
                uint64_t v = D->v;
                if (is64 || x) v = bswap(v, imm);                /* BSWAP, or TO_BE on little-endian */
                else v = imm == 64 ? v : (v & ((1ull << imm) - 1));  /* TO_LE: truncate */
                if (imm < 64) v &= (1ull << imm) - 1;
                D->v = v;
                pc++;
                continue;
            }
            reg_t sv;
            if (op == 0x80) { sv.tag = T_SCALAR; sv.v = 0; }     /* NEG has no source */
            else if (x) sv = *S;
            else { sv.tag = T_SCALAR; sv.v = is64 ? (uint64_t)(int64_t)imm : (uint64_t)(uint32_t)imm; sv.map = -1; sv.base = NULL; }
            if (sv.tag == T_UNINIT) return fault(env, ev, pc, "read of uninitialised register");
            if (op == 0xB0 && off == 0) {                        /* MOV: copies pointers too */
                if (!is64 && sv.tag != T_SCALAR) return fault(env, ev, pc, "32-bit mov of a pointer");
                *D = sv;
                if (!is64) D->v &= 0xFFFFFFFFull;
                pc++;
                continue;
            }
            if (D->tag == T_UNINIT) return fault(env, ev, pc, "read of uninitialised register");
            int dptr = D->tag != T_SCALAR, sptr = sv.tag != T_SCALAR;
            if (dptr || sptr) {                                  /* O7: only ptr +- scalar, ptr - ptr */
                if (!is64) return fault(env, ev, pc, "32-bit ALU on a pointer");
                if (op == 0x00 && dptr != sptr) {
                    reg_t P = dptr ? *D : sv;
                    uint64_t k = dptr ? sv.v : D->v;
                    if (P.tag == T_MAPH) return fault(env, ev, pc, "arithmetic on a map handle");
                    P.v += k;
                    *D = P;
                } else if (op == 0x10 && dptr && !sptr) {
                    if (D->tag == T_MAPH) return fault(env, ev, pc, "arithmetic on a map handle");
                    D->v -= sv.v;
                } else if (op == 0x10 && dptr && sptr && D->tag == sv.tag &&
                           (D->tag == T_STACK || (D->tag == T_MAPV && D->base == sv.base))) {
                    D->v = D->v - sv.v; D->tag = T_SCALAR; D->base = NULL; D->map = -1;
                } else return fault(env, ev, pc, "illegal pointer arithmetic");
                pc++;
                continue;
            }
            uint64_t r;
            if (alu(op, is64, off, D->v, sv.v, &r)) return fault(env, ev, pc, "bad ALU instruction");
            D->v = r; D->tag = T_SCALAR;
            pc++;
            continue;
        }

        if (cls == CL_JMP || cls == CL_JMP32) {
            uint32_t op = code & 0xF0;
            int is64 = cls == CL_JMP;
            if (op == 0x00) {                                    /* JA */
                if (!is64) return fault(env, ev, pc, "gotol unsupported");
                pc = pc + 1 + off;
                continue;
            }
            if (op == 0x90) {                                    /* EXIT */
                if (!is64) return fault(env, ev, pc, "bad exit");
                if (vm->r[0].tag != T_SCALAR) return fault(env, ev, pc, "r0 at exit is not an initialised scalar");
                *r0 = vm->r[0].v;
                return 0;
            }
            if (op == 0x80) {                                    /* CALL helper imm (O6) */
                if (!is64 || src != 0) return fault(env, ev, pc, "bpf-to-bpf / kfunc calls unsupported");
                reg_t *R1 = &vm->r[1], *R2 = &vm->r[2], *R3 = &vm->r[3], *R4 = &vm->r[4];
                int64_t ret;
                if (imm == 1 || imm == 2 || imm == 130 || imm == FN_MEM_PREFETCH || imm == FN_PREFETCH_L2) {
                    if (R1->tag != T_MAPH) return fault(env, ev, pc, "helper r1 is not a map handle");
                }
                if (imm == 1) {
                    map_t *m = &env->maps[R1->map];
                    if (m->type == MAP_RINGBUF || m->type == MAP_PFQ || m->type == MAP_REGION)
                        return fault(env, ev, pc, "lookup on ringbuf / prefetch queue / region");
                    const uint8_t *key = arg_bytes(vm, R2, m->key_size, pc);
                    if (!key) return -1;
                    uint8_t *v = map_lookup(m, key, vm->shard);
                    clobber_args(vm);
                    if (v) { vm->r[0].tag = T_MAPV; vm->r[0].map = R1->map; vm->r[0].base = v; vm->r[0].v = 0; }
                    else { vm->r[0].tag = T_SCALAR; vm->r[0].v = 0; }
                    pc++;
                    continue;
                } else if (imm == 2) {
                    map_t *m = &env->maps[R1->map];
                    if (m->type == MAP_RINGBUF || m->type == MAP_PFQ || m->type == MAP_REGION)
                        return fault(env, ev, pc, "update on ringbuf / prefetch queue / region");
                    const uint8_t *key = arg_bytes(vm, R2, m->key_size, pc);
                    if (!key) return -1;
                    const uint8_t *val = arg_bytes(vm, R3, m->value_size, pc);
                    if (!val) return -1;
                    if (!scalar(R4)) return fault(env, ev, pc, "flags not a scalar");
                    uint8_t kb[8], vb[256];
                    memcpy(kb, key, m->key_size);
                    memcpy(vb, val, m->value_size);
                    ret = map_update(env, m, kb, vb, R4->v, vm->shard);
                } else if (imm == 130) {
                    map_t *m = &env->maps[R1->map];
                    if (m->type != MAP_RINGBUF) return fault(env, ev, pc, "ringbuf_output on a non-ringbuf map");
                    if (!scalar(R3) || !scalar(R4)) return fault(env, ev, pc, "size/flags not scalar");
                    if (R3->v == 0 || R3->v > 256) return fault(env, ev, pc, "ringbuf size out of [1,256]");
                    const uint8_t *data = arg_bytes(vm, R2, (uint32_t)R3->v, pc);
                    if (!data) return -1;
                    ret = ringbuf_output(env, m, data, R3->v, R4->v);
                } else if (imm == FN_MEM_PREFETCH) {
                    map_t *m = &env->maps[R1->map];
                    if (m->type != MAP_PFQ) return fault(env, ev, pc, "mem_prefetch on a non-prefetch-queue map");
                    if (!scalar(R2) || !scalar(R3)) return fault(env, ev, pc, "prefetch addr/len not scalar");
                    ret = mem_prefetch(env, m, R2->v, R3->v);
                } else if (imm == FN_PREFETCH_L2) {
                    map_t *m = &env->maps[R1->map];
                    if (m->type != MAP_REGION) return fault(env, ev, pc, "prefetch_l2 on a non-region map");
                    if (!scalar(R2) || !scalar(R3)) return fault(env, ev, pc, "prefetch addr/len not scalar");
                    ret = prefetch_l2(m, R2->v, R3->v);
                } else {
                    return fault(env, ev, pc, "unknown or forbidden helper");
                }
                if (ret < 0) env->stats[ST_HERR]++;
                clobber_args(vm);
                vm->r[0].tag = T_SCALAR; vm->r[0].v = (uint64_t)ret;
                pc++;
                continue;
            }
            /* conditional jumps */
            int x = (code & 0x08) != 0;
            if (D->tag == T_UNINIT || (x && S->tag == T_UNINIT)) return fault(env, ev, pc, "read of uninitialised register");
            uint64_t sv = x ? S->v : (is64 ? (uint64_t)(int64_t)imm : (uint64_t)(uint32_t)imm);
            int taken;
            if (D->tag != T_SCALAR || (x && S->tag != T_SCALAR)) {
                /* O7: only JEQ/JNE ptr, 0 (a NULL-able map value is compared with 0). */
                if (x || !(op == 0x10 || op == 0x50) || imm != 0 || !is64) return fault(env, ev, pc, "pointer comparison");
                taken = (op == 0x50);   /* a live pointer is never NULL */
            } else if (jcond(op, is64, D->v, sv, &taken)) return fault(env, ev, pc, "bad jump op");
            pc = taken ? pc + 1 + off : pc + 1;
            continue;
        }

        if (cls == CL_LD) {                                      /* only ldimm64 (O5) */
            if (code != 0x18 || pc + 1 >= p->n) return fault(env, ev, pc, "bad LD");
            if (p->code[pc + 1] || p->dst[pc + 1] || p->src[pc + 1] || p->off[pc + 1]) return fault(env, ev, pc, "bad ldimm64 second slot");
            if (dst == 10) return fault(env, ev, pc, "write to r10");
            uint64_t lo = (uint32_t)imm, hi = (uint32_t)p->imm[pc + 1];
            if (src == 0) { D->tag = T_SCALAR; D->v = lo | (hi << 32); }
            else if (src == 1 || src == 2) {                     /* O2 relocation */
                if (imm < 0 || imm >= MAX_MAPS || !env->maps[imm].used) return fault(env, ev, pc, "bad map fd");
                if (src == 1) { D->tag = T_MAPH; D->map = imm; D->v = 0; D->base = NULL; }
                else {
                    map_t *m = &env->maps[imm];
                    if (m->type != MAP_ARRAY) return fault(env, ev, pc, "map_value on a non-array");
                    if (hi >= m->value_size) return fault(env, ev, pc, "map_value offset out of range");
                    D->tag = T_MAPV; D->map = imm; D->base = m->data; D->v = hi;
                }
            } else return fault(env, ev, pc, "unsupported pseudo source");
            pc += 2;
            continue;
        }

        if (cls == CL_LDX) {
            uint32_t mode = code & 0xE0, size = size_of(code);
            if (dst == 10) return fault(env, ev, pc, "write to r10");
            if (mode != 0x60 && mode != 0x80) return fault(env, ev, pc, "bad LDX mode");
            if (mode == 0x80 && size == 8) return fault(env, ev, pc, "bad MEMSX size");
            if (S->tag == T_UNINIT) return fault(env, ev, pc, "read of uninitialised register");
            uint8_t *a = mem_addr(vm, S, off, size, 0, pc);
            if (!a) return -1;
            if (S->tag == T_STACK) {
                int64_t so = (int64_t)S->v + off;
                reg_t *spill = &vm->sspill[so / 8];
                if (spill->tag != T_SCALAR) {                    /* fill of a spilled pointer */
                    if (size != 8 || mode != 0x60) return fault(env, ev, pc, "partial read of a spilled pointer");
                    *D = *spill;
                    pc++;
                    continue;
                }
            }
            uint64_t v = load_le(a, size);
            if (mode == 0x80) v = sext(v, size * 8);
            D->tag = T_SCALAR; D->v = v; D->base = NULL; D->map = -1;
            pc++;
            continue;
        }

        if (cls == CL_ST || cls == CL_STX) {
            uint32_t mode = code & 0xE0, size = size_of(code);
            if (D->tag == T_UNINIT) return fault(env, ev, pc, "read of uninitialised register");
            if (cls == CL_STX && S->tag == T_UNINIT) return fault(env, ev, pc, "read of uninitialised register");
            if (mode == 0x60) {
                uint8_t *a = mem_addr(vm, D, off, size, 1, pc);
                if (!a) return -1;
                if (cls == CL_STX && S->tag != T_SCALAR) {       /* pointer spill: stack only, 8 bytes */
                    if (D->tag != T_STACK || size != 8) return fault(env, ev, pc, "pointer stored outside the stack (leak)");
                    int64_t so = (int64_t)D->v + off;
                    store_le(a, 8, S->v);
                    stack_wrote(vm, so, 8);
                    vm->sspill[so / 8] = *S;
                    pc++;
                    continue;
                }
                uint64_t v = cls == CL_ST ? (uint64_t)(int64_t)imm : S->v;
                store_le(a, size, v);
                if (D->tag == T_STACK) stack_wrote(vm, (int64_t)D->v + off, size);
                pc++;
                continue;
            }
            if (mode == 0xC0 && cls == CL_STX) {                 /* atomics, bpf.h:23, 49-51 */
                if (size != 4 && size != 8) return fault(env, ev, pc, "B/H atomics unsupported");
                if (S->tag != T_SCALAR) return fault(env, ev, pc, "atomic operand is a pointer");
                uint8_t *a = mem_addr(vm, D, off, size, 1, pc);
                if (!a) return -1;
                if (D->tag == T_STACK) {
                    int64_t so = (int64_t)D->v + off;
                    for (uint32_t k = 0; k < size; k++)
                        if (!vm->sinit[so + k]) return fault(env, ev, pc, "atomic on uninitialised stack");
                    if (vm->sspill[so / 8].tag != T_SCALAR) return fault(env, ev, pc, "atomic on a spilled pointer");
                }
                uint64_t mask = size == 8 ? ~0ull : 0xFFFFFFFFull;
                uint64_t old = load_le(a, size), sv = S->v & mask, nv;
                int fetch = imm & 1;
                switch (imm) {
                case 0x00: case 0x01: nv = old + sv; break;
                case 0x40: case 0x41: nv = old | sv; break;
                case 0x50: case 0x51: nv = old & sv; break;
                case 0xA0: case 0xA1: nv = old ^ sv; break;
                case 0xE1: nv = sv; break;                                       /* XCHG */
                case 0xF1: {                                                     /* CMPXCHG */
                    if (vm->r[0].tag != T_SCALAR) return fault(env, ev, pc, "cmpxchg r0 not a scalar");
                    nv = (old == (vm->r[0].v & mask)) ? sv : old;
                    store_le(a, size, nv);
                    vm->r[0].v = old;                                            /* W: zero-extended */
                    pc++;
                    continue;
                }
                default: return fault(env, ev, pc, "bad atomic op");
                }
                store_le(a, size, nv & mask);
                if (fetch) { S->v = old; S->tag = T_SCALAR; }
                pc++;
                continue;
            }
            return fault(env, ev, pc, "bad store mode");
        }
        return fault(env, ev, pc, "bad instruction class");
    }
}

/* O3 batch loop.  `order` (nullable) is a permutation of [0,n) (O10 --perm); R0 is written
 * at the original index.  Returns 0, or -1 on an oracle fault. */
ORA_EXPORT int ora_run(ora_env *e, const void *events, uint64_t n, int prog, uint64_t *r0_out,
                       const uint64_t *order, uint64_t index_base) {
    const uint8_t *evb = events;
    for (uint64_t k = 0; k < n; k++) {
        uint64_t i = order ? order[k] : k;
        const uint8_t *ctx = evb + 32 * i;
        uint32_t hook;
        memcpy(&hook, ctx + 16, 4);
        int p = prog >= 0 ? prog : e->attach[hook & 0xFF][(hook >> 8) & 0xFF];
        if (p < 0 || p >= MAX_PROGS || !e->progs[p].used) { e->stats[ST_SKIP]++; if (r0_out) r0_out[i] = 0; continue; }
        uint64_t r0;
        if (run_one(e, &e->progs[p], ctx, index_base + i, &r0)) return -1;
        e->stats[ST_RUN]++;
        if (r0_out) r0_out[i] = r0;
    }
    return 0;
}

/* ------------------------------------------------------------------ f3: block scheduling
 * The work-stealing thread-block scheduler of PAPER.md §4.3.2 ("Return whether to steal work (TB
 * scheduler)", should_try_steal) and §6.2.1 (persistent workers pull work units; FixedWork /
 * Greedy / LatencyBudget), as the discrete-event simulation of SPEC.md:374-424 (F-5):
 *   every worker pops its own deque from the head: ENTER hook, cost_us of work, EXIT hook;
 *   when its deque is empty it fires the STEAL hook: R0 == 0 -> the worker retires; else it steals
 *   the TAIL unit of the worker with the largest deque (lowest id on ties), paying steal_cost_us,
 *   and runs it (ENTER/EXIT with the stolen bit); no victim -> it retires.
 * Workers advance on one simulated clock: the next step is taken by the worker with the smallest
 * time (lowest id on ties).  Hook records: addr = unit id (STEAL: 0), ts = simulated ns,
 * hook = kind | stolen << 16, block_id = worker, size = cost_us (STEAL: 0). */
enum { HK_ENTER = 1, HK_EXIT = 4, HK_STEAL = 5 };

static int sched_hook(ora_env *e, int prog, uint32_t kind, uint32_t stolen, uint32_t worker, uint64_t unit,
                      uint64_t t_us, uint32_t cost, uint64_t seq, uint64_t *r0) {
    uint8_t ctx[32] = {0};
    const uint64_t ts = t_us * 1000;
    const uint32_t hook = kind | (stolen << 16);
    memcpy(ctx + 0, &unit, 8);
    memcpy(ctx + 8, &ts, 8);
    memcpy(ctx + 16, &hook, 4);
    memcpy(ctx + 20, &worker, 4);
    memcpy(ctx + 28, &cost, 4);
    if (run_one(e, &e->progs[prog], ctx, seq, r0)) return -1;
    e->stats[ST_RUN]++;
    return 0;
}

ORA_EXPORT int ora_sched_run(ora_env *e, int prog, uint32_t n_units, const uint32_t *cost_us, const uint32_t *home,
                             uint32_t n_workers, uint32_t steal_cost_us, uint32_t *executed_by, uint8_t *stolen,
                             uint64_t *busy_us, uint64_t *end_us, uint32_t *steals, uint64_t *makespan_us) {
    if (prog < 0 || prog >= MAX_PROGS || !e->progs[prog].used || !n_workers) return -E_INVAL;
    uint32_t *cnt = calloc(n_workers + 1, sizeof *cnt), *off = calloc(n_workers + 1, sizeof *off);
    uint32_t *seg = malloc((n_units + 1) * sizeof *seg), *head = calloc(n_workers, sizeof *head),
             *tail = calloc(n_workers, sizeof *tail), *fill = calloc(n_workers, sizeof *fill);
    uint64_t *t = calloc(n_workers, sizeof *t);
    uint8_t *done = calloc(n_workers, 1);
    for (uint32_t u = 0; u < n_units; u++) cnt[home[u]]++;
    for (uint32_t w = 0; w < n_workers; w++) off[w + 1] = off[w] + cnt[w];
    for (uint32_t u = 0; u < n_units; u++) seg[off[home[u]] + fill[home[u]]++] = u;   /* deque in unit order */
    for (uint32_t w = 0; w < n_workers; w++) { head[w] = off[w]; tail[w] = off[w + 1]; busy_us[w] = 0; steals[w] = 0; }
    uint64_t seq = 0;
    int rc = 0;
    for (;;) {
        int w = -1;
        for (uint32_t k = 0; k < n_workers; k++)
            if (!done[k] && (w < 0 || t[k] < t[w])) w = (int)k;
        if (w < 0) break;
        uint32_t u, st = 0;
        if (head[w] < tail[w]) {
            u = seg[head[w]++];
        } else {
            uint64_t r0;
            if (sched_hook(e, prog, HK_STEAL, 0, (uint32_t)w, 0, t[w], 0, seq++, &r0)) { rc = -1; break; }
            if (r0 == 0) { done[w] = 1; continue; }
            int v = -1;
            for (uint32_t k = 0; k < n_workers; k++)
                if (tail[k] > head[k] && (v < 0 || tail[k] - head[k] > tail[v] - head[v])) v = (int)k;
            if (v < 0) { done[w] = 1; continue; }
            u = seg[--tail[v]];
            st = 1;
            t[w] += steal_cost_us;
            steals[w]++;
        }
        uint64_t r0;
        if (sched_hook(e, prog, HK_ENTER, st, (uint32_t)w, u, t[w], cost_us[u], seq++, &r0)) { rc = -1; break; }
        t[w] += cost_us[u];
        busy_us[w] += cost_us[u];
        if (sched_hook(e, prog, HK_EXIT, st, (uint32_t)w, u, t[w], cost_us[u], seq++, &r0)) { rc = -1; break; }
        executed_by[u] = (uint32_t)w;
        stolen[u] = (uint8_t)st;
    }
    uint64_t ms = 0;
    for (uint32_t w = 0; w < n_workers; w++) { end_us[w] = t[w]; if (t[w] > ms) ms = t[w]; }
    *makespan_us = ms;
    free(cnt); free(off); free(seg); free(head); free(tail); free(fill); free(t); free(done);
    return rc;
}

/* ------------------------------------------------------------------ canonical dumps (O8) */

/* hash dump order: keys (at most 8 bytes) as unsigned little-endian integers; the sort key travels
 * with each entry (no global: environments may be dumped from several threads at once) */
typedef struct { uint64_t k; const hnode *n; } hsort_t;
static int hcmp(const void *x, const void *y) {
    const hsort_t *a = x, *b = y;
    return a->k < b->k ? -1 : a->k > b->k ? 1 : 0;
}

/* ARRAY: max*vs bytes.  PT: per key, per 8-byte word, the SUM over shards (S4).  HASH: entries
 * (key || value) sorted by key as an unsigned LE integer.  *n_out = bytes written (ARRAY/PT)
 * or entries (HASH). */
ORA_EXPORT int ora_map_dump(ora_env *e, int fd, void *buf, uint64_t cap, uint64_t *n_out) {
    if (fd < 0 || fd >= MAX_MAPS || !e->maps[fd].used) return -E_INVAL;
    map_t *m = &e->maps[fd];
    uint8_t *out = buf;
    if (m->type == MAP_ARRAY) {
        uint64_t sz = (uint64_t)m->max_entries * m->value_size;
        if (sz > cap) return -E_2BIG;
        memcpy(out, m->data, sz);
        *n_out = sz;
        return 0;
    }
    if (m->type == MAP_PT) {
        uint64_t sz = (uint64_t)m->max_entries * m->value_size;
        if (sz > cap) return -E_2BIG;
        for (uint64_t w = 0; w < sz / 8; w++) {
            uint64_t acc = 0;
            for (uint32_t s = 0; s < m->nshards; s++) acc += load_le(m->shards[s] + 8 * w, 8);
            store_le(out + 8 * w, 8, acc);
        }
        *n_out = sz;
        return 0;
    }
    if (m->type == MAP_HASH) {
        uint64_t es = m->key_size + m->value_size;
        if (m->count * es > cap) return -E_2BIG;
        hsort_t *all = malloc((m->count + 1) * sizeof *all);
        uint64_t c = 0;
        for (uint64_t b = 0; b < m->nbuckets; b++)
            for (hnode *n = m->buckets[b]; n; n = n->next) {
                all[c].k = load_le(n->key, m->key_size);
                all[c++].n = n;
            }
        qsort(all, c, sizeof *all, hcmp);
        for (uint64_t i = 0; i < c; i++) {
            memcpy(out + i * es, all[i].n->key, m->key_size);
            memcpy(out + i * es + m->key_size, all[i].n->val, m->value_size);
        }
        free(all);
        *n_out = c;
        return 0;
    }
    return -E_INVAL;
}

typedef struct { const uint8_t *p; uint32_t len; } rec_t;
static int rcmp(const void *x, const void *y) {
    const rec_t *a = x, *b = y;
    uint32_t n = a->len < b->len ? a->len : b->len;
    int c = memcmp(a->p, b->p, n);
    if (c) return c;
    return a->len < b->len ? -1 : (a->len > b->len);
}

/* RINGBUF multiset (O8): records sorted lexicographically by payload; written as
 * u32 len || payload (unpadded).  *n_rec = records, *n_bytes = bytes written. */
ORA_EXPORT int ora_ringbuf_dump(ora_env *e, int fd, void *buf, uint64_t cap, uint64_t *n_rec, uint64_t *n_bytes) {
    if (fd < 0 || fd >= MAX_MAPS || !e->maps[fd].used || e->maps[fd].type != MAP_RINGBUF) return -E_INVAL;
    map_t *m = &e->maps[fd];
    uint64_t cnt = 0;
    for (uint64_t o = 0; o < m->rb_used; o += (8 + load_le(m->rb + o, 4) + 7) & ~7ull) cnt++;
    rec_t *r = malloc((cnt + 1) * sizeof *r);
    uint64_t k = 0;
    for (uint64_t o = 0; o < m->rb_used; o += (8 + load_le(m->rb + o, 4) + 7) & ~7ull) {
        r[k].len = (uint32_t)load_le(m->rb + o, 4);
        r[k].p = m->rb + o + 8;
        k++;
    }
    qsort(r, cnt, sizeof *r, rcmp);
    uint64_t w = 0;
    for (uint64_t i = 0; i < cnt; i++) {
        if (w + 4 + r[i].len > cap) { free(r); return -E_2BIG; }
        memcpy((uint8_t *)buf + w, &r[i].len, 4);
        memcpy((uint8_t *)buf + w + 4, r[i].p, r[i].len);
        w += 4 + r[i].len;
    }
    free(r);
    *n_rec = cnt;
    *n_bytes = w;
    return 0;
}

ORA_EXPORT uint64_t ora_ringbuf_used(ora_env *e, int fd) { return e->maps[fd].rb_used; }

/* PREFETCH QUEUE canonical content (F-2): the SET of requests -- prefetching a region
 * twice is the same as once, so implementations may merge identical requests -- sorted by
 * (first_page, npages), 2 u64 words each; *n = distinct requests, *n_calls = appended requests. */
static int pcmp(const void *a, const void *b) {
    const uint64_t *x = a, *y = b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : x[1] > y[1];
}
ORA_EXPORT int ora_pfq_dump(ora_env *e, int fd, uint64_t *buf, uint64_t cap, uint64_t *n, uint64_t *n_calls) {
    if (fd < 0 || fd >= MAX_MAPS || !e->maps[fd].used || e->maps[fd].type != MAP_PFQ) return -E_INVAL;
    map_t *m = &e->maps[fd];
    uint64_t *t = malloc((2 * m->pfq_n + 2) * sizeof *t);
    memcpy(t, m->pfq, 2 * m->pfq_n * sizeof *t);
    qsort(t, m->pfq_n, 2 * sizeof *t, pcmp);
    uint64_t k = 0;
    for (uint64_t i = 0; i < m->pfq_n; i++) {
        if (k && t[2 * (k - 1)] == t[2 * i] && t[2 * (k - 1) + 1] == t[2 * i + 1]) continue;
        t[2 * k] = t[2 * i];
        t[2 * k + 1] = t[2 * i + 1];
        k++;
    }
    if (k > cap) { free(t); return -E_2BIG; }
    memcpy(buf, t, 2 * k * sizeof *t);
    free(t);
    *n = k;
    *n_calls = m->pfq_n;
    return 0;
}
/* drain: the host handler consumed the queue (gx_prefetch_drain / the runtime daemon) */
ORA_EXPORT int ora_pfq_reset(ora_env *e, int fd) {
    if (fd < 0 || fd >= MAX_MAPS || !e->maps[fd].used || e->maps[fd].type != MAP_PFQ) return -E_INVAL;
    e->maps[fd].pfq_n = 0;
    return 0;
}

/* ------------------------------------------------------------------ shards (O10 --shards G, S3) */

/* Deep copy of an environment (maps, programs, attach table, settings); stats reset. */
ORA_EXPORT ora_env *ora_clone(ora_env *src) {
    ora_env *e = ora_new();
    if (!e) return NULL;
    memcpy(e->attach, src->attach, sizeof e->attach);
    e->pt_shards = src->pt_shards;
    for (int i = 0; i < MAX_MAPS; i++) {
        map_t *s = &src->maps[i], *d = &e->maps[i];
        if (!s->used) continue;
        *d = *s;
        d->data = NULL; d->shards = NULL; d->buckets = NULL; d->rb = NULL; d->nshards = 0; d->count = 0;
        if (s->type == MAP_ARRAY) {
            d->data = malloc((size_t)s->max_entries * s->value_size);
            memcpy(d->data, s->data, (size_t)s->max_entries * s->value_size);
        } else if (s->type == MAP_PT) {
            pt_ensure_shards(d, s->nshards);
            for (uint32_t k = 0; k < s->nshards; k++)
                memcpy(d->shards[k], s->shards[k], (size_t)s->max_entries * s->value_size);
        } else if (s->type == MAP_HASH) {
            d->buckets = calloc(s->nbuckets, sizeof *d->buckets);
            for (uint64_t b = 0; b < s->nbuckets; b++)
                for (hnode *n = s->buckets[b]; n; n = n->next) {
                    hnode *c = hash_insert(d, n->key);
                    memcpy(c->val, n->val, s->value_size);
                }
        } else if (s->type == MAP_RINGBUF) {
            d->rb = calloc(s->max_entries, 1);
            memcpy(d->rb, s->rb, s->rb_used);
        } else if (s->type == MAP_PFQ) {
            d->pfq = calloc(2 * (size_t)s->max_entries, sizeof(uint64_t));
            memcpy(d->pfq, s->pfq, 2 * s->pfq_n * sizeof(uint64_t));
        }
    }
    for (int i = 0; i < MAX_PROGS; i++) {
        prog_t *s = &src->progs[i];
        if (!s->used) continue;
        prog_t *d = &e->progs[i];   /* same program id in the clone */
        d->n = s->n;
        d->code = malloc(s->n); d->dst = malloc(s->n); d->src = malloc(s->n);
        d->off = malloc(s->n * sizeof(int16_t)); d->imm = malloc(s->n * sizeof(int32_t));
        memcpy(d->code, s->code, s->n); memcpy(d->dst, s->dst, s->n); memcpy(d->src, s->src, s->n);
        memcpy(d->off, s->off, s->n * sizeof(int16_t)); memcpy(d->imm, s->imm, s->n * sizeof(int32_t));
        d->used = 1;
    }
    return e;
}

/* S3 snapshot-and-merge:
 * `init` holds the state every shard started from and receives the canonical result.
 * ARRAY / PT (folded): canon = init + sum_g (local_g - init) per u64 word (mod 2^64).
 * HASH: union of keys; value = init (0 if new) + sum_g (local_g - init) per word;
 *       a union larger than max_entries -> hash_full, -E2BIG.
 * RINGBUF: multiset union (records appended in shard order; capacity drops counted).
 * Stats are summed.  Returns 0 or -errno. */
ORA_EXPORT int ora_merge(ora_env *init, ora_env **locals, int G) {
    int rc = 0;
    for (int i = 0; i < MAX_MAPS; i++) {
        map_t *m = &init->maps[i];
        if (!m->used) continue;
        if (m->type == MAP_ARRAY || m->type == MAP_PT) {
            uint64_t words = (uint64_t)m->max_entries * m->value_size / 8;
            uint64_t *acc = calloc(words, 8), *base = calloc(words, 8);
            for (uint64_t w = 0; w < words; w++) {               /* init (folded) */
                if (m->type == MAP_ARRAY) base[w] = load_le(m->data + 8 * w, 8);
                else for (uint32_t s = 0; s < m->nshards; s++) base[w] += load_le(m->shards[s] + 8 * w, 8);
                acc[w] = base[w];
            }
            for (int g = 0; g < G; g++) {
                map_t *l = &locals[g]->maps[i];
                for (uint64_t w = 0; w < words; w++) {
                    uint64_t lv = 0;
                    if (l->type == MAP_ARRAY) lv = load_le(l->data + 8 * w, 8);
                    else for (uint32_t s = 0; s < l->nshards; s++) lv += load_le(l->shards[s] + 8 * w, 8);
                    acc[w] += lv - base[w];
                }
            }
            if (m->type == MAP_ARRAY) memcpy(m->data, acc, words * 8);
            else {
                for (uint32_t s = 0; s < m->nshards; s++) memset(m->shards[s], 0, words * 8);
                memcpy(m->shards[0], acc, words * 8);
            }
            free(acc); free(base);
        } else if (m->type == MAP_HASH) {
            uint32_t vw = m->value_size / 8;
            /* start from a snapshot of init values, then add every shard's delta */
            ora_env *snap = ora_clone(init);
            for (int g = 0; g < G; g++) {
                map_t *l = &locals[g]->maps[i];
                for (uint64_t b = 0; b < l->nbuckets; b++)
                    for (hnode *n = l->buckets[b]; n; n = n->next) {
                        hnode *iv = hash_find(&snap->maps[i], n->key);
                        hnode *dst = hash_find(m, n->key);
                        if (!dst) {
                            if (m->count >= m->max_entries) { init->stats[ST_HFULL]++; rc = -E_2BIG; continue; }
                            dst = hash_insert(m, n->key);
                        }
                        for (uint32_t w = 0; w < vw; w++) {
                            uint64_t d = load_le(n->val + 8 * w, 8) - (iv ? load_le(iv->val + 8 * w, 8) : 0);
                            store_le(dst->val + 8 * w, 8, load_le(dst->val + 8 * w, 8) + d);
                        }
                    }
            }
            ora_free(snap);
        } else if (m->type == MAP_RINGBUF) {
            uint64_t start = m->rb_used;   /* records present at init are in every local copy */
            for (int g = 0; g < G; g++) {
                map_t *l = &locals[g]->maps[i];
                for (uint64_t o = start; o < l->rb_used; o += (8 + load_le(l->rb + o, 4) + 7) & ~7ull) {
                    uint32_t len = (uint32_t)load_le(l->rb + o, 4);
                    ringbuf_output(init, m, l->rb + o + 8, len, 0);
                }
            }
        } else if (m->type == MAP_PFQ) {   /* union of the shards' requests (F-2: a set) */
            uint64_t start = m->pfq_n;
            for (int g = 0; g < G; g++) {
                map_t *l = &locals[g]->maps[i];
                for (uint64_t r = start; r < l->pfq_n; r++) {
                    if (m->pfq_n >= m->max_entries) { init->stats[ST_DROPS]++; rc = -E_AGAIN; continue; }
                    m->pfq[2 * m->pfq_n] = l->pfq[2 * r];
                    m->pfq[2 * m->pfq_n + 1] = l->pfq[2 * r + 1];
                    m->pfq_n++;
                }
            }
        }
    }
    for (int g = 0; g < G; g++)
        for (int k = 0; k < 8; k++) init->stats[k] += locals[g]->stats[k];
    return rc;
}
