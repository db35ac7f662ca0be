/*
 * gx_runtime.cpp -- implementation of the C ABI in include/gx.h (host side).
 *
 * Owns the per-device runtime: map memory and descriptors, loaded programs and their verified
 * pre-decoded images, the attach table, launch descriptors, stats, and the chunked host->device
 * pipeline of gx_run_batch_host.  Every device-side step is one of the kernels in gx_exec.cu /
 * gx_maps.cu; nothing here computes on events.
 */
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <errno.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <thread>
#include <memory>
#include <string>
#include <vector>

#include "../../include/gx.h"
#include "gx_internal.h"
#include "gx_jit.h"
#include "gx_verifier.h"

#include <cuda.h>
#include <nccl.h> /* types only: libnccl is dlopen'ed at gx_comm_init (no link-time dependency) */
#include <nvtx3/nvToolsExt.h> /* header-only: ranges reach a profiler only when one injects itself */
#include <chrono>

extern "C" {
int gx_launch_exec(const GxLaunch *d_launch, const void *d_events, uint64_t n, uint64_t *d_ret, uint32_t grid,
                   uint32_t smem, cudaStream_t stream);
int gx_exec_occupancy(uint32_t smem, int *blocks_per_sm);
uint32_t gx_exec_block_threads();
int gx_k_pt_fold(const uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, uint64_t *out, cudaStream_t s);
int gx_k_nsmid(uint32_t *out_host);
int gx_k_pt_set(uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, uint32_t k, const uint64_t *vals,
                cudaStream_t s);
int gx_k_pt_store_canonical(uint64_t *data, uint32_t nshards, uint32_t K, uint32_t W, const uint64_t *vals,
                            cudaStream_t s);
int gx_k_hash_init(uint64_t *slots, uint64_t cap, cudaStream_t s);
int gx_k_publish(const GxPublishItem *items, uint32_t n_items, uint8_t *host_slot, cudaStream_t s);
int gx_k_hash_host_update(const GxMapDesc *m, const uint64_t *keys, const uint64_t *vals, uint64_t n, uint64_t flags,
                          int64_t *rc, unsigned long long *full, cudaStream_t s);
int gx_k_sub(const uint64_t *a, const uint64_t *b, uint64_t *out, uint64_t n, cudaStream_t s);
int gx_k_add(const uint64_t *a, const uint64_t *b, uint64_t *out, uint64_t n, cudaStream_t s);
int gx_k_hash_export(const GxMapDesc *m, const GxMapDesc *base, uint32_t nranks, int32_t owner, int pass,
                     unsigned long long *counts, unsigned long long *offsets, uint64_t *keys, uint64_t *deltas,
                     uint64_t cap_out, cudaStream_t s);
int gx_k_hash_accumulate(const GxMapDesc *m, const uint64_t *keys, const uint64_t *deltas, uint64_t n,
                         unsigned long long *full, cudaStream_t s);
}

namespace {

constexpr uint32_t kBlocksPerSmMax = 4;        /* 4 x 256 threads = 1024 executor lanes per SM */
constexpr uint32_t kPrivMaxBytes = 16 * 1024;  /* shared-memory privatisation budget per block */
constexpr uint64_t kHostChunk = 1ull << 22;    /* events per chunk of gx_run_batch_host (128 MiB) */

struct Map {
    bool valid = false;
    gx_map_spec spec{};
    void *data = nullptr;   /* device */
    void *aux = nullptr;    /* device counters */
    uint64_t data_bytes = 0;
    uint32_t nshards = 0;
    uint64_t cap = 0;       /* HASH slots / RINGBUF bytes */
    void *base = nullptr;   /* merge snapshot (ARRAY/PT canonical words, HASH slot copy) */
    void *base_aux = nullptr;
};

struct Prog {
    bool valid = false;
    uint32_t hook = 0;
    std::vector<uint8_t> slots;
    bool verified = false;
    GxVerifyResult vr;
    GxInsn *d_image = nullptr;
};

struct LaunchKey {
    int prog;
    std::vector<int> attach_progs;
    uint64_t version;
    bool operator<(const LaunchKey &o) const {
        if (prog != o.prog) return prog < o.prog;
        if (version != o.version) return version < o.version;
        return attach_progs < o.attach_progs;
    }
};

struct LaunchCfg {
    GxLaunch *d = nullptr;
    GxLaunch h;              /* host copy (the JIT bakes it into the generated kernel) */
    std::vector<int> progs;  /* launch slot -> prog fd */
    uint32_t smem = 0;
    uint32_t grid = 0;
    /* JIT engine: one module per launch variant (GX_JIT_V_*: ring / register ingest x R0 off / on),
     * compiled on the variant's first launch */
    struct JitVar {
        bool tried = false;
        CUmodule mod = nullptr;
        CUfunction fn = nullptr;
        unsigned smem = 0;        /* dynamic shared bytes (the ring stages; fixed at compile) */
        uint32_t grid = 0, block = 256;
    } jv[4];
    bool ring_ok = true;
    bool jit_failed = false;   /* the JIT could not compile this configuration: interpreter launches */
    std::string jit_log;
    double jit_ms = 0;
};

/* driver entry points through the runtime (no link-time dependency on libcuda) */
struct Drv {
    bool ok = false;
    CUresult (*moduleLoadData)(CUmodule *, const void *) = nullptr;
    CUresult (*moduleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void **, void **) = nullptr;
    CUresult (*occupancy)(int *, CUfunction, int, size_t) = nullptr;
    CUresult (*moduleUnload)(CUmodule) = nullptr;
    CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*launchKernelEx)(const CUlaunchConfig *, CUfunction, void **, void **) = nullptr;
};
Drv &drv() {
    static Drv d;
    static bool init = false;
    if (!init) {
        init = true;
        cudaDriverEntryPointQueryResult q;
        bool ok = true;
        ok &= cudaGetDriverEntryPoint("cuModuleLoadData", (void **)&d.moduleLoadData, cudaEnableDefault, &q) == cudaSuccess;
        ok &= cudaGetDriverEntryPoint("cuModuleGetFunction", (void **)&d.moduleGetFunction, cudaEnableDefault, &q) == cudaSuccess;
        ok &= cudaGetDriverEntryPoint("cuLaunchKernel", (void **)&d.launchKernel, cudaEnableDefault, &q) == cudaSuccess;
        ok &= cudaGetDriverEntryPoint("cuOccupancyMaxActiveBlocksPerMultiprocessor", (void **)&d.occupancy,
                                      cudaEnableDefault, &q) == cudaSuccess;
        ok &= cudaGetDriverEntryPoint("cuModuleUnload", (void **)&d.moduleUnload, cudaEnableDefault, &q) == cudaSuccess;
        ok &= cudaGetDriverEntryPoint("cuFuncSetAttribute", (void **)&d.funcSetAttribute, cudaEnableDefault, &q) == cudaSuccess;
        if (cudaGetDriverEntryPoint("cuLaunchKernelEx", (void **)&d.launchKernelEx, cudaEnableDefault, &q) != cudaSuccess)
            d.launchKernelEx = nullptr;
        d.ok = ok && d.moduleLoadData && d.moduleGetFunction && d.launchKernel;
    }
    return d;
}

}  // namespace

/* runtime daemon (include/gx.h) */
struct DaemonSlot {
    uint8_t *host = nullptr;   /* pinned, device-mapped */
    cudaEvent_t ev = nullptr;
    bool busy = false;
};
struct Daemon {
    static constexpr int kSlots = 4;
    bool running = false, stopping = false;
    gx_prefetch_handler fn = nullptr;
    void *user = nullptr;
    std::thread th;
    std::mutex mu;
    std::condition_variable cv_work, cv_free;
    std::deque<int> pending;
    DaemonSlot slots[kSlots];
    uint64_t slot_bytes = 0;
    std::vector<int> watched;              /* map fds, in watch order */
    std::vector<GxPublishItem> items;      /* frozen layout at start */
    std::vector<int> item_fd;
    GxPublishItem *d_items = nullptr;
    struct Fold { const uint64_t *data; uint32_t nshards, K, W; uint64_t *staging; };
    std::vector<Fold> folds;                /* watched per-thread maps: SUM fold before publishing */
    std::map<int, std::vector<uint8_t>> snap; /* latest published canonical snapshots */
    uint64_t version = 0;
    gx_daemon_stats st{};
    uint64_t managed_ptr = 0, managed_bytes = 0; /* default handler's prefetchable range */
    cudaStream_t s_prefetch = nullptr;
};

/* ---- multi-GPU transport of gx_merge: NCCL (dlopen'ed; device buffers over
 * NVLink / NVSwitch), or caller-supplied host callbacks (several ranks sharing one device in tests). */
struct GxComm {
    int nranks = 1, rank = 0;
    virtual ~GxComm() {}
    virtual bool device_buffers() const = 0;
    /* in-place u64 SUM over ranks (wraparound: exactly the S3 delta arithmetic) */
    virtual int allreduce_sum_u64(uint64_t *buf, uint64_t n, cudaStream_t s) = 0;
    /* every rank sends send_bytes[g] bytes from send + soff[g] to rank g and receives recv_bytes[g]
     * bytes from rank g at recv + roff[g] */
    virtual int alltoallv(const uint8_t *send, const uint64_t *send_bytes, const uint64_t *soff, uint8_t *recv,
                          const uint64_t *recv_bytes, const uint64_t *roff, cudaStream_t s) = 0;
    /* recv[g * bytes .. ] = rank g's send[0 .. bytes) */
    virtual int allgather(const void *send, void *recv, uint64_t bytes, cudaStream_t s) = 0;
    virtual const char *error() const { return ""; }
};

struct MergeScratch {
    uint64_t *d = nullptr; /* device scratch (packed deltas, hash exchange buffers) */
    uint64_t words = 0;
    std::vector<uint64_t> h; /* host staging for host transports */
};

struct gx_rt {
    int dev = 0;
    int nsm = 0;
    uint32_t max_shards = 0;
    Map maps[GX_MAX_MAPS];
    Prog progs[GX_MAX_PROGS];
    int attach[GX_MAX_KINDS][256];
    uint64_t version = 1;               /* bumps whenever maps / programs / attach change */
    std::map<LaunchKey, LaunchCfg> launches;
    unsigned long long *d_stats = nullptr;
    uint32_t last_grid = 0, last_block = 0, last_smem = 0;
    int engine = GX_ENGINE_JIT;
    uint64_t n_launches = 0;
    std::string err;
    /* gx_run_batch_host pipeline */
    cudaStream_t s_copy = nullptr, s_exec = nullptr;
    void *d_chunk[2] = {nullptr, nullptr};
    uint64_t *d_rchunk[2] = {nullptr, nullptr};
    cudaEvent_t ev_copied[2], ev_done[2];
    bool pipe_init = false;
    Daemon dmn;
    /* batch order across streams (order_after_last) */
    cudaEvent_t ev_order = nullptr;
    cudaStream_t order_stream = nullptr;
    bool order_valid = false;
    /* gx_comm_init / gx_merge */
    std::unique_ptr<GxComm> comm;
    MergeScratch ms;
    uint64_t merges = 0;
};

namespace {

/* GX_LOG_LEVEL: 0 silent (default), 1 errors (every -errno with its text),
 * 2 + JIT compiles (variant, block, grid, shared memory, milliseconds) and merges, 3 + every launch. */
int log_level() {
    static const int lv = getenv("GX_LOG_LEVEL") ? atoi(getenv("GX_LOG_LEVEL")) : 0;
    return lv;
}
void gx_log(int level, const char *fmt, ...) {
    if (level > log_level()) return;
    char buf[768];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    fprintf(stderr, "[gx:%d] %s\n", level, buf);
}
/* NVTX range for the duration of a public call (no-op unless a profiler injects NVTX) */
struct NvtxScope {
    explicit NvtxScope(const char *name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};

int set_err(gx_rt *rt, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (rt) rt->err = buf;
    gx_log(1, "error %d: %s", code, buf);
    return code;
}

int cuda_err(gx_rt *rt, cudaError_t e, const char *what) {
    return set_err(rt, -EFAULT, "%s: %s", what, cudaGetErrorString(e));
}
#define CK(call, what)                                    \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) return cuda_err(rt, _e, what); \
    } while (0)

GxMapDesc make_desc(const Map &m) {
    GxMapDesc d{};
    d.data = (uint64_t)m.data;
    d.aux = (uint64_t)m.aux;
    d.type = m.spec.type;
    d.key_size = m.spec.key_size;
    d.value_size = m.spec.value_size;
    d.max_entries = m.spec.max_entries;
    d.nshards = m.nshards;
    d.cap_mask = (uint32_t)(m.cap ? m.cap - 1 : 0);
    d.priv_off = 0xFFFFFFFFu;
    d.coherent = 0;
    if (m.spec.type == GX_MAP_REGION) d.aux = m.data_bytes; /* [data, data + aux): caller-owned */
    return d;
}

GxMapDesc make_base_desc(const Map &m) {
    GxMapDesc d = make_desc(m);
    d.data = (uint64_t)m.base;
    d.aux = (uint64_t)m.base_aux;
    return d;
}

bool check_map(gx_rt *rt, int fd) { return rt && fd >= 0 && fd < GX_MAX_MAPS && rt->maps[fd].valid; }
bool check_prog(gx_rt *rt, int fd) { return rt && fd >= 0 && fd < GX_MAX_PROGS && rt->progs[fd].valid; }

uint32_t smem_bytes(uint32_t staged, uint32_t stack_slots, uint32_t priv_bytes) {
    uint32_t per_warp = (GX_NREGS + 4 + stack_slots) * 32 * 8;
    return staged * (uint32_t)sizeof(GxInsn) + GX_MAX_MAPS * (uint32_t)sizeof(GxMapDesc) + GX_MAX_KINDS * 256 +
           priv_bytes + 64 + per_warp * (gx_exec_block_threads() / 32);
}

/* builds (or reuses) the device launch descriptor for one run configuration */
int get_launch(gx_rt *rt, int prog_fd, LaunchCfg *&out) {
    LaunchKey key;
    key.prog = prog_fd;
    key.version = rt->version;
    std::vector<int> plist;
    if (prog_fd >= 0) plist.push_back(prog_fd);
    else {
        for (int k = 0; k < GX_MAX_KINDS; k++)
            for (int t = 0; t < 256; t++)
                if (rt->attach[k][t] >= 0 && std::find(plist.begin(), plist.end(), rt->attach[k][t]) == plist.end())
                    plist.push_back(rt->attach[k][t]);
        key.attach_progs = plist;
    }
    auto it = rt->launches.find(key);
    if (it != rt->launches.end()) {
        out = &it->second;
        return 0;
    }
    if (plist.size() > GX_MAX_LAUNCH_PROGS) return set_err(rt, -E2BIG, "more than %d programs in one launch", GX_MAX_LAUNCH_PROGS);
    GxLaunch h;
    memset(&h, 0, sizeof h);
    memset(h.attach, -1, sizeof h.attach);
    for (int i = 0; i < GX_MAX_MAPS; i++)
        if (rt->maps[i].valid) h.maps[i] = make_desc(rt->maps[i]);
    uint32_t staged = 0, stack = 8;
    for (size_t q = 0; q < plist.size(); q++) {
        Prog &p = rt->progs[plist[q]];
        if (!p.verified) return set_err(rt, -EPERM, "program %d has not passed gx_verify", plist[q]);
        h.progs[q].image = (uint64_t)p.d_image;
        h.progs[q].n = (uint32_t)p.vr.image.size();
        h.progs[q].smem_off = staged;
        staged += h.progs[q].n;
        stack = std::max(stack, p.vr.stack_depth);
    }
    if (staged > GX_MAX_STAGED_INSNS) return set_err(rt, -E2BIG, "launch stages %u instructions (max %d)", staged, GX_MAX_STAGED_INSNS);
    h.n_progs = (uint32_t)plist.size();
    h.single = prog_fd >= 0 ? 0 : -1;
    if (prog_fd < 0)
        for (int k = 0; k < GX_MAX_KINDS; k++)
            for (int t = 0; t < 256; t++)
                if (rt->attach[k][t] >= 0)
                    h.attach[k][t] = (int8_t)(std::find(plist.begin(), plist.end(), rt->attach[k][t]) - plist.begin());
    h.staged_insns = staged;
    h.stack_slots = (stack + 7) / 8;
    /* map facts across the launch: coherent (written by any program) and privatisable
     * (write-only commutative ADD accumulator in every program that uses it: SURVEY.md §8c c.7) */
    uint32_t priv = 0;
    for (int m = 0; m < GX_MAX_MAPS; m++) {
        if (!rt->maps[m].valid) continue;
        bool written = false, accum = true, used = false;
        for (int q : plist) {
            const GxMapUse &u = rt->progs[q].vr.use[m];
            if (!u.used) continue;
            used = true;
            written |= u.writes;
            if (u.reads || u.non_add_write || u.fetch_add || u.update_call || u.non_dw_atomic) accum = false;
        }
        h.maps[m].coherent = written ? 1 : 0;
        const Map &mm = rt->maps[m];
        uint64_t bytes = (uint64_t)mm.spec.max_entries * mm.spec.value_size;
        if (used && written && accum && mm.spec.type == GX_MAP_ARRAY && h.n_priv < 8 && priv + bytes <= kPrivMaxBytes &&
            !getenv("GX_NO_PRIV")) {
            h.maps[m].priv_off = priv;
            h.priv_maps[h.n_priv++] = m;
            priv += (uint32_t)((bytes + 15) & ~15ull);
        }
    }
    h.priv_bytes = priv;
    h.stats = (uint64_t)rt->d_stats;
    LaunchCfg cfg;
    cfg.smem = smem_bytes(staged, h.stack_slots, priv);
    if (cfg.smem > 227 * 1024) return set_err(rt, -E2BIG, "launch needs %u bytes of shared memory", cfg.smem);
    int bps = 0;
    int e = gx_exec_occupancy(cfg.smem, &bps);
    if (e) return cuda_err(rt, (cudaError_t)e, "occupancy");
    if (bps < 1) return set_err(rt, -E2BIG, "executor does not fit on an SM (%u B shared)", cfg.smem);
    cfg.grid = (uint32_t)rt->nsm * (uint32_t)std::min<int>(bps, (int)kBlocksPerSmMax);
    cfg.h = h;
    cfg.progs = plist;
    CK(cudaMalloc(&cfg.d, sizeof(GxLaunch)), "cudaMalloc launch");
    CK(cudaMemcpy(cfg.d, &h, sizeof h, cudaMemcpyHostToDevice), "cudaMemcpy launch");
    auto res = rt->launches.emplace(key, cfg);
    out = &res.first->second;
    return 0;
}

/* compiles (once) the JIT kernel of launch variant `k` of a configuration */
int jit_prepare(gx_rt *rt, LaunchCfg &cfg, int k) {
    LaunchCfg::JitVar &V = cfg.jv[k];
    if (V.fn) return 0;
    if (V.tried) return set_err(rt, -ENOSYS, "JIT unavailable: %s", cfg.jit_log.c_str());
    V.tried = true;
    if (getenv("GX_JIT_INJECT_FAILURE") && atoi(getenv("GX_JIT_INJECT_FAILURE")) != 0) { /* fault injection (tests) */
        cfg.jit_log = "injected failure (GX_JIT_INJECT_FAILURE)";
        return set_err(rt, -ENOSYS, "JIT unavailable: %s", cfg.jit_log.c_str());
    }
    Drv &d = drv();
    if (!d.ok) {
        cfg.jit_log = "driver entry points unavailable";
        return set_err(rt, -ENOSYS, "JIT unavailable: %s", cfg.jit_log.c_str());
    }
    auto t0 = std::chrono::steady_clock::now();
    std::vector<const GxInsn *> images;
    std::vector<uint32_t> sizes;
    std::vector<const uint16_t *> nin;
    for (int q : cfg.progs) {
        const GxVerifyResult &vr = rt->progs[q].vr;
        images.push_back(vr.image.data());
        sizes.push_back((uint32_t)vr.image.size());
        nin.push_back(vr.narrow_in.size() == vr.image.size() ? vr.narrow_in.data() : nullptr);
    }
    const bool ring = k < 2;
    /* fewer, larger blocks keep the per-block privatised-shard flush small; one 1024-thread block
     * per SM measured fastest on every config (profiles/r1_jit_variants.md); 256-thread blocks only
     * if the 1024-thread kernel cannot be resident at all */
    for (int B : {gx_jit_block(), 256}) {
        std::string src = gx_jit_source(cfg.h, images, sizes, B, 1u << k, &nin);
        if (const char *dump = getenv("GX_JIT_DUMP")) {
            if (FILE *f = fopen(dump, "w")) {
                fputs(src.c_str(), f);
                fclose(f);
            }
        }
        std::vector<char> cubin;
        if (gx_jit_compile(src, cubin, cfg.jit_log)) return set_err(rt, -ENOSYS, "JIT compile failed: %s", cfg.jit_log.c_str());
        CUmodule mod = nullptr;
        if (d.moduleLoadData(&mod, cubin.data()) != CUDA_SUCCESS) return set_err(rt, -EFAULT, "cuModuleLoadData failed");
        CUfunction fn = nullptr;
        if (d.moduleGetFunction(&fn, mod, gx_jit_kernel_name(k)) != CUDA_SUCCESS)
            return set_err(rt, -EFAULT, "cuModuleGetFunction(%s) failed", gx_jit_kernel_name(k));
        const unsigned smem = ring ? gx_jit_smem(B, gx_jit_stages_for(images, sizes)) : 0u;
        if (ring && d.funcSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem) != CUDA_SUCCESS)
            return set_err(rt, -EFAULT, "cuFuncSetAttribute(%u B dynamic shared) failed", smem);
        /* shared-memory carve-out preference (GX_JIT_CARVEOUT percent; -1 = the driver's choice): a
         * hint -- the driver still picks a configuration that fits the ring -- so 0 asks for the
         * smallest carve-out, leaving the rest of the SM's 256 KiB to L1 */
        if (const char *e = getenv("GX_JIT_CARVEOUT")) {
            const int pct = atoi(e);
            if (pct >= 0 && pct <= 100) d.funcSetAttribute(fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, pct);
        }
        int bps = 2048 / B; /* per-thread shards: at most 2048 resident threads per SM */
        {
            int b = 0;
            if (!d.occupancy || d.occupancy(&b, fn, B, smem) != CUDA_SUCCESS || b < 1) b = 1;
            bps = std::min(bps, b);
        }
        if (bps * B < 1024 && B != 256) {
            if (d.moduleUnload) d.moduleUnload(mod);
            continue;
        }
        V.mod = mod;
        V.fn = fn;
        V.smem = smem;
        V.block = (uint32_t)B;
        V.grid = (uint32_t)rt->nsm * (uint32_t)bps;
        break;
    }
    /* every large batch takes the ring (round 1 kept ALU-heavy single programs -- a bounded loop,
     * > 64 instructions on the worst path -- on register ingest; after round 2's code-generation
     * changes the ring wins for them too: C4 4.08 -> 4.01 ms, profiles/r2_stages.md) */
    cfg.ring_ok = true;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    cfg.jit_ms += ms;
    gx_log(2, "JIT variant %d (%s ingest%s): %zu program(s), block %u, grid %u, %u B dynamic shared, %.1f ms", k,
           ring ? "ring" : "register", (k & 1) ? ", R0" : "", cfg.progs.size(), V.block, V.grid, V.smem, ms);
    return 0;
}

/* the launch variant a batch takes: the TMA ring for large batches (>= 2^22 events) of light
 * programs, per-lane register loads otherwise (GX_JIT_INGEST=ring|reg forces one;
 * profiles/r1_jit_variants.md) */
int jit_variant(const LaunchCfg &cfg, uint64_t n, bool want_ret) {
    const char *fe = getenv("GX_JIT_INGEST");
    const int force = !fe ? 0 : strcmp(fe, "ring") == 0 ? 1 : strcmp(fe, "reg") == 0 ? 2 : 0;
    const bool ring = force == 1 || (force == 0 && cfg.ring_ok && n >= (1ull << 22));
    return (ring ? 0 : 2) + (want_ret ? 1 : 0);
}

/* a publish point on `stream` after the batch's kernel: take a free slot (wait for the daemon if
 * none: backpressure), write the prefetch queues and watched snapshots into it, record its event */
int daemon_publish(gx_rt *rt, cudaStream_t stream) {
    Daemon &D = rt->dmn;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
        return set_err(rt, -EBUSY, "the runtime daemon cannot follow batches captured into a CUDA graph");
    int slot = -1;
    {
        std::unique_lock<std::mutex> lk(D.mu);
        for (;;) {
            for (int k = 0; k < Daemon::kSlots; k++)
                if (!D.slots[k].busy) {
                    slot = k;
                    break;
                }
            if (slot >= 0) break;
            D.st.backpressure++;
            D.cv_free.wait(lk);
        }
        D.slots[slot].busy = true;
    }
    for (const Daemon::Fold &f : D.folds) {
        int e = gx_k_pt_fold(f.data, f.nshards, f.K, f.W, f.staging, stream);
        if (e) return cuda_err(rt, (cudaError_t)e, "daemon fold");
    }
    int e = gx_k_publish(D.d_items, (uint32_t)D.items.size(), D.slots[slot].host, stream);
    if (e) return cuda_err(rt, (cudaError_t)e, "daemon publish");
    CK(cudaEventRecord(D.slots[slot].ev, stream), "daemon event");
    {
        std::lock_guard<std::mutex> lk(D.mu);
        D.pending.push_back(slot);
    }
    D.cv_work.notify_one();
    return 0;
}

/* default prefetch handler: requests inside the registered managed range are prefetched to the
 * device (cudaMemPrefetchAsync, "host-side callbacks extend prefetching"); all are
 * counted */
void default_prefetch(gx_rt *rt, const uint64_t *reqs, uint64_t n) {
    Daemon &D = rt->dmn;
    if (!D.managed_bytes) return;
    const uint64_t lo = D.managed_ptr, hi = D.managed_ptr + D.managed_bytes;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t a = reqs[2 * i] << 12, b = a + ((reqs[2 * i + 1] & 0xFFFFFFFFull) << 12);
        a = std::max(a, lo);
        b = std::min(b, hi);
        if (a >= b) continue;
#if CUDART_VERSION >= 13000
        cudaMemLocation loc{cudaMemLocationTypeDevice, rt->dev};
        if (cudaMemPrefetchAsync((void *)a, b - a, loc, 0, D.s_prefetch) == cudaSuccess) D.st.managed_prefetches++;
#else
        if (cudaMemPrefetchAsync((void *)a, b - a, rt->dev, D.s_prefetch) == cudaSuccess) D.st.managed_prefetches++;
#endif
    }
}

void daemon_main(gx_rt *rt) {
    Daemon &D = rt->dmn;
    cudaSetDevice(rt->dev);
    for (;;) {
        int slot;
        {
            std::unique_lock<std::mutex> lk(D.mu);
            D.cv_work.wait(lk, [&] { return !D.pending.empty() || D.stopping; });
            if (D.pending.empty()) return; /* stopping and drained */
            slot = D.pending.front();
            D.pending.pop_front();
        }
        cudaEventSynchronize(D.slots[slot].ev);
        const uint8_t *h = D.slots[slot].host;
        uint64_t nreq = 0;
        for (size_t i = 0; i < D.items.size(); i++) {
            const GxPublishItem &it = D.items[i];
            const uint64_t *w = reinterpret_cast<const uint64_t *>(h + it.host_off);
            if (it.kind == 0) {
                const uint64_t n = w[0];
                nreq += n;
                if (n) {
                    if (D.fn) D.fn(D.user, D.item_fd[i], w + 1, n);
                    else default_prefetch(rt, w + 1, n);
                }
            }
        }
        {
            std::lock_guard<std::mutex> lk(D.mu);
            D.version++;
            for (size_t i = 0; i < D.items.size(); i++) {
                const GxPublishItem &it = D.items[i];
                if (it.kind == 0) continue;
                const uint8_t *src = h + it.host_off;
                D.snap[D.item_fd[i]].assign(src, src + 8ull * it.K * it.W);
                D.st.snapshots++;
            }
            D.st.batches++;
            D.st.requests += nreq;
            D.slots[slot].busy = false;
        }
        D.cv_free.notify_all();
    }
}

/* Batches of one runtime run in submission order whatever streams they are given: per-thread
 * shards are plain read-modify-writes keyed by the resident thread, and the privatised and
 * hash-cache flushes assume one batch at a time.  Every batch records an event right after its
 * kernel on its own stream (while that stream surely exists -- a caller's stream may be gone by
 * the next batch); a batch on a different stream first waits on it.  Same-stream order is free. */
int order_after_last(gx_rt *rt, cudaStream_t stream) {
    if (rt->order_valid && rt->order_stream != stream) CK(cudaStreamWaitEvent(stream, rt->ev_order, 0), "order wait");
    return 0;
}
int order_record(gx_rt *rt, cudaStream_t stream) {
    CK(cudaEventRecord(rt->ev_order, stream), "order event");
    rt->order_stream = stream;
    rt->order_valid = true;
    return 0;
}

int launch_cfg(gx_rt *rt, LaunchCfg &cfg, const void *d_events, uint64_t n, uint64_t *d_ret, cudaStream_t stream,
               uint32_t flags = 0) {
    if (int rc = order_after_last(rt, stream)) return rc;
    gx_log(3, "batch %llu: %llu events, %s engine, stream %p", (unsigned long long)rt->n_launches, (unsigned long long)n,
           rt->engine == GX_ENGINE_JIT ? "jit" : "interp", (void *)stream);
    /* a launch configuration the JIT cannot compile (e.g. an NVRTC resource limit) runs on the
     * interpreter -- the same semantics on the same GPU -- and says so at GX_LOG_LEVEL 1 */
    bool jit_ok = rt->engine == GX_ENGINE_JIT && !cfg.jit_failed;
    int vk = 0;
    if (jit_ok) {
        vk = jit_variant(cfg, n, d_ret != nullptr);
        int rc = jit_prepare(rt, cfg, vk);
        if (rc == -ENOSYS) {
            cfg.jit_failed = true;
            jit_ok = false;
            gx_log(1, "JIT variant %d unavailable (%s): this launch configuration runs on the interpreter", vk,
                   rt->err.c_str());
        } else if (rc) {
            return rc;
        }
    }
    if (jit_ok) {
        const LaunchCfg::JitVar &V = cfg.jv[vk];
        const void *ev = d_events;
        uint64_t nn = n;
        uint64_t *rp = d_ret;
        unsigned long long *st = rt->d_stats;
        void *args[] = {(void *)&ev, (void *)&nn, (void *)&rp, (void *)&st};
        /* small batches: fewer, fuller blocks (>= 8 events per thread) so block set-up and the
         * privatised-shard flush do not dominate; large batches: the resident grid */
        static const uint64_t per_thread = getenv("GX_JIT_EPT") ? strtoull(getenv("GX_JIT_EPT"), nullptr, 10) : 8;
        static const uint64_t cap = getenv("GX_JIT_GRID") ? strtoull(getenv("GX_JIT_GRID"), nullptr, 10) : ~0ull;
        const uint64_t B = V.block;
        uint64_t want = (n + B * per_thread - 1) / (B * per_thread);
        if (want * 2 >= V.grid) want = V.grid; /* past half the resident grid: every SM streams */
        want = std::min<uint64_t>(cap, want);
        uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(V.grid, want));
        CUfunction fnl = V.fn;
        const unsigned smem = V.smem;
        if ((flags & GX_RUN_OVERLAP) && drv().launchKernelEx) {
            /* programmatic dependent launch: the grid may start while the previous kernel on the
             * stream drains; it stages its first records, then griddepcontrol.wait holds every map
             * access until that kernel has completed and flushed (gx_jit.cpp) */
            CUlaunchAttribute at[1];
            at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
            at[0].value.programmaticStreamSerializationAllowed = 1;
            CUlaunchConfig lc = {};
            lc.gridDimX = grid;
            lc.gridDimY = lc.gridDimZ = 1;
            lc.blockDimX = (unsigned)B;
            lc.blockDimY = lc.blockDimZ = 1;
            lc.sharedMemBytes = smem;
            lc.hStream = (CUstream)stream;
            lc.attrs = at;
            lc.numAttrs = 1;
            if (drv().launchKernelEx(&lc, fnl, args, nullptr) != CUDA_SUCCESS)
                return set_err(rt, -EFAULT, "JIT kernel launch (PDL) failed");
        } else if (drv().launchKernel(fnl, grid, 1, 1, (unsigned)B, 1, 1, smem, (CUstream)stream, args, nullptr) !=
                   CUDA_SUCCESS) {
            return set_err(rt, -EFAULT, "JIT kernel launch failed");
        }
        rt->last_grid = grid;
        rt->last_block = (uint32_t)B;
        rt->last_smem = smem;
    } else {
        int e = gx_launch_exec(cfg.d, d_events, n, d_ret, cfg.grid, cfg.smem, stream);
        if (e) return cuda_err(rt, (cudaError_t)e, "executor launch");
        rt->last_grid = cfg.grid;
        rt->last_block = gx_exec_block_threads();
        rt->last_smem = cfg.smem;
    }
    rt->n_launches++;
    if (rt->dmn.running) /* the publish point belongs to this batch: the order event follows it */
        if (int rc = daemon_publish(rt, stream)) return rc;
    return order_record(rt, stream);
}

int sync(gx_rt *rt) {
    CK(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    return 0;
}

}  // namespace

extern "C" {

int gx_open(int cuda_device, gx_rt **out) {
    if (!out) return -EINVAL;
    *out = nullptr;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, cuda_device);
    if (e != cudaSuccess) return -EFAULT;
    if (prop.major != 10) return -EFAULT; /* sm_100a code only */
    e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) return -EFAULT;
    gx_rt *rt = new gx_rt();
    rt->dev = cuda_device;
    if (cudaEventCreateWithFlags(&rt->ev_order, cudaEventDisableTiming) != cudaSuccess) {
        delete rt;
        return -EFAULT;
    }
    rt->nsm = prop.multiProcessorCount;
    /* one shard per resident thread slot (2048 / SM); f4 hooks key shards by (%smid, %warpid, lane),
     * and %smid ranges over [0, %nsmid), which may exceed the SM count */
    {
        uint32_t nsmid = 0;
        if (gx_k_nsmid(&nsmid) != 0) nsmid = 0;
        rt->max_shards = (uint32_t)std::max<int>(rt->nsm, (int)nsmid) * 2048;
    }
    if (const char *e = getenv("GX_ENGINE")) rt->engine = strcmp(e, "interp") == 0 ? GX_ENGINE_INTERP : GX_ENGINE_JIT;
    for (auto &row : rt->attach)
        for (int &x : row) x = -1;
    if (cudaMalloc(&rt->d_stats, GXS_N * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(rt->d_stats, 0, GXS_N * sizeof(unsigned long long)) != cudaSuccess) {
        delete rt;
        return -ENOMEM;
    }
    *out = rt;
    return 0;
}

void gx_close(gx_rt *rt) {
    if (!rt) return;
    cudaSetDevice(rt->dev);
    gx_daemon_stop(rt);
    cudaDeviceSynchronize();
    for (auto &m : rt->maps) {
        if (m.spec.type != GX_MAP_REGION) cudaFree(m.data);   /* a region's memory is the caller's */
        cudaFree(m.aux);
        cudaFree(m.base);
        cudaFree(m.base_aux);
    }
    for (auto &p : rt->progs) cudaFree(p.d_image);
    for (auto &kv : rt->launches) {
        cudaFree(kv.second.d);
        for (auto &v : kv.second.jv)
            if (v.mod && drv().moduleUnload) drv().moduleUnload(v.mod);
    }
    cudaFree(rt->d_stats);
    if (rt->ev_order) cudaEventDestroy(rt->ev_order);
    rt->comm.reset();
    cudaFree(rt->ms.d);
    if (rt->pipe_init) {
        for (int b = 0; b < 2; b++) {
            cudaFree(rt->d_chunk[b]);
            cudaFree(rt->d_rchunk[b]);
            cudaEventDestroy(rt->ev_copied[b]);
            cudaEventDestroy(rt->ev_done[b]);
        }
        cudaStreamDestroy(rt->s_copy);
        cudaStreamDestroy(rt->s_exec);
    }
    delete rt;
}

const char *gx_last_error(gx_rt *rt) { return rt ? rt->err.c_str() : "no runtime"; }

int gx_create_map(gx_rt *rt, const gx_map_spec *spec, int *map_fd) {
    if (!rt || !spec || !map_fd) return -EINVAL;
    const gx_map_spec s = *spec;
    if (s.flags) return set_err(rt, -EINVAL, "map flags must be 0");
    int fd = -1;
    for (int i = 0; i < GX_MAX_MAPS; i++)
        if (!rt->maps[i].valid) {
            fd = i;
            break;
        }
    if (fd < 0) return set_err(rt, -ENOMEM, "too many maps");
    Map m;
    m.spec = s;
    switch (s.type) {
    case GX_MAP_ARRAY:
        if (s.key_size != 4 || !s.value_size || s.value_size % 8 || s.value_size > 65536 || !s.max_entries)
            return set_err(rt, -EINVAL, "bad ARRAY spec");
        m.data_bytes = (uint64_t)s.max_entries * s.value_size;
        break;
    case GX_MAP_PERTHREAD_ARRAY:
        if (s.key_size != 4 || s.value_size < 8 || s.value_size > 256 || (s.value_size & (s.value_size - 1)) ||
            !s.max_entries || (uint64_t)s.max_entries * s.value_size > 4096)
            return set_err(rt, -EINVAL, "bad PERTHREAD_ARRAY spec (value_size a power of two in [8,256], "
                                        "max_entries*value_size <= 4096)");
        m.nshards = rt->max_shards;
        m.data_bytes = (uint64_t)s.max_entries * s.value_size * m.nshards;
        break;
    case GX_MAP_HASH: {
        if ((s.key_size != 4 && s.key_size != 8) || s.value_size != 8 || !s.max_entries)
            return set_err(rt, -EINVAL, "bad HASH spec (key 4 or 8 bytes, value 8 bytes)");
        uint64_t cap = 16;
        while (cap < 2ull * s.max_entries) cap <<= 1;
        m.cap = cap;
        m.data_bytes = (cap + 2) * 16; /* key words, then value words (gx_device.cuh) */
        break;
    }
    case GX_MAP_RINGBUF:
        if (s.key_size || s.value_size || s.max_entries < 4096 || (s.max_entries & (s.max_entries - 1)))
            return set_err(rt, -EINVAL, "bad RINGBUF spec (byte capacity: power of two >= 4096)");
        m.cap = s.max_entries;
        m.data_bytes = s.max_entries;
        break;
    case GX_MAP_PREFETCH_QUEUE:
        if (s.key_size || s.value_size || s.max_entries < 64 || s.max_entries > (1u << 24) ||
            (s.max_entries & (s.max_entries - 1)))
            return set_err(rt, -EINVAL, "bad PREFETCH_QUEUE spec (capacity in requests: power of two in [64, 2^24])");
        m.cap = s.max_entries;
        m.nshards = GX_PFQ_FILTER_WORDS(s.max_entries);
        m.data_bytes = 16ull * s.max_entries + 8ull * m.nshards; /* records + request filter */
        break;
    default:
        return set_err(rt, -EINVAL, "unknown map type %u", s.type);
    }
    if (cudaMalloc(&m.data, m.data_bytes) != cudaSuccess) return set_err(rt, -ENOMEM, "cudaMalloc map %llu B", (unsigned long long)m.data_bytes);
    cudaMalloc(&m.aux, 64);
    cudaMemset(m.aux, 0, 64);
    if (s.type == GX_MAP_HASH) {
        int e = gx_k_hash_init((uint64_t *)m.data, m.cap, 0);
        if (e) return cuda_err(rt, (cudaError_t)e, "hash init");
    } else {
        CK(cudaMemset(m.data, 0, m.data_bytes), "cudaMemset map");
    }
    CK(cudaDeviceSynchronize(), "map init");
    m.valid = true;
    rt->maps[fd] = m;
    rt->version++;
    *map_fd = fd;
    return 0;
}

int gx_region_map(gx_rt *rt, const void *dev_ptr, uint64_t len, int *map_fd) {
    if (!rt || !map_fd) return -EINVAL;
    if (!dev_ptr || !len || (uint64_t)(uintptr_t)dev_ptr + len < (uint64_t)(uintptr_t)dev_ptr)
        return set_err(rt, -EINVAL, "bad device region");
    int fd = -1;
    for (int i = 0; i < GX_MAX_MAPS; i++)
        if (!rt->maps[i].valid) {
            fd = i;
            break;
        }
    if (fd < 0) return set_err(rt, -ENOMEM, "too many maps");
    Map m;
    m.spec.type = GX_MAP_REGION;
    m.spec.max_entries = 1;
    m.data = const_cast<void *>(dev_ptr);
    m.data_bytes = len;
    m.valid = true;
    rt->maps[fd] = m;
    rt->version++;
    *map_fd = fd;
    return 0;
}

int gx_update_map(gx_rt *rt, int fd, const void *keys, const void *vals, uint64_t n, uint64_t flags) {
    if (!check_map(rt, fd)) return -ENOENT;
    if (n == 0) return 0;
    if (!keys || !vals) return -EINVAL;
    Map &m = rt->maps[fd];
    const gx_map_spec &s = m.spec;
    int rc0 = sync(rt);
    if (rc0) return rc0;
    const uint8_t *kb = (const uint8_t *)keys, *vb = (const uint8_t *)vals;
    if (s.type == GX_MAP_RINGBUF || s.type == GX_MAP_PREFETCH_QUEUE || s.type == GX_MAP_REGION)
        return set_err(rt, -EINVAL, "ring buffers, prefetch queues and regions have no keys");
    if (flags > 2) return -EINVAL;
    if (s.type == GX_MAP_ARRAY || s.type == GX_MAP_PERTHREAD_ARRAY) {
        int first = 0;
        std::vector<uint8_t> img;
        bool whole = s.type == GX_MAP_ARRAY && n > 8;
        if (whole) {
            img.resize(m.data_bytes);
            CK(cudaMemcpy(img.data(), m.data, m.data_bytes, cudaMemcpyDeviceToHost), "read array");
        }
        uint64_t *dv = nullptr;
        if (s.type == GX_MAP_PERTHREAD_ARRAY) CK(cudaMalloc(&dv, s.value_size), "cudaMalloc");
        for (uint64_t i = 0; i < n; i++) {
            uint32_t k;
            memcpy(&k, kb + 4 * i, 4);
            int rc = 0;
            if (k >= s.max_entries) rc = -E2BIG;
            else if (flags == 1) rc = -EEXIST;
            if (rc) {
                if (!first) first = rc;
                continue;
            }
            const uint8_t *v = vb + (uint64_t)s.value_size * i;
            if (whole) memcpy(img.data() + (uint64_t)k * s.value_size, v, s.value_size);
            else if (s.type == GX_MAP_ARRAY)
                CK(cudaMemcpy((uint8_t *)m.data + (uint64_t)k * s.value_size, v, s.value_size, cudaMemcpyHostToDevice), "write array");
            else {
                CK(cudaMemcpy(dv, v, s.value_size, cudaMemcpyHostToDevice), "write pt");
                int e = gx_k_pt_set((uint64_t *)m.data, m.nshards, s.max_entries, s.value_size / 8, k, dv, 0);
                if (e) return cuda_err(rt, (cudaError_t)e, "pt set");
                CK(cudaDeviceSynchronize(), "pt set");
            }
        }
        if (whole) CK(cudaMemcpy(m.data, img.data(), m.data_bytes, cudaMemcpyHostToDevice), "write array");
        cudaFree(dv);
        return first;
    }
    /* HASH */
    std::vector<uint64_t> hk(n), hv(n);
    for (uint64_t i = 0; i < n; i++) {
        uint64_t k = 0;
        memcpy(&k, kb + s.key_size * i, s.key_size);
        hk[i] = k;
        memcpy(&hv[i], vb + 8 * i, 8);
    }
    uint64_t *dk, *dvv;
    int64_t *drc;
    unsigned long long *dfull;
    CK(cudaMalloc(&dk, 8 * n), "cudaMalloc");
    CK(cudaMalloc(&dvv, 8 * n), "cudaMalloc");
    CK(cudaMalloc(&drc, 8 * n), "cudaMalloc");
    CK(cudaMalloc(&dfull, 8), "cudaMalloc");
    cudaMemset(dfull, 0, 8);
    cudaMemcpy(dk, hk.data(), 8 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dvv, hv.data(), 8 * n, cudaMemcpyHostToDevice);
    GxMapDesc d = make_desc(m);
    int e = gx_k_hash_host_update(&d, dk, dvv, n, flags, drc, dfull, 0);
    if (e) return cuda_err(rt, (cudaError_t)e, "hash update");
    std::vector<int64_t> rc(n);
    CK(cudaMemcpy(rc.data(), drc, 8 * n, cudaMemcpyDeviceToHost), "hash update rc");
    cudaFree(dk);
    cudaFree(dvv);
    cudaFree(drc);
    cudaFree(dfull);
    for (auto r : rc)
        if (r) return (int)r;
    return 0;
}

int gx_read_map(gx_rt *rt, int fd, void *keys, void *vals, uint64_t cap, uint64_t *n_out) {
    if (!check_map(rt, fd)) return -ENOENT;
    if (!vals || !n_out) return -EINVAL;
    Map &m = rt->maps[fd];
    const gx_map_spec &s = m.spec;
    int rc0 = sync(rt);
    if (rc0) return rc0;
    if (s.type == GX_MAP_ARRAY || s.type == GX_MAP_PERTHREAD_ARRAY) {
        if (cap < s.max_entries) return -E2BIG;
        uint64_t bytes = (uint64_t)s.max_entries * s.value_size;
        if (s.type == GX_MAP_ARRAY) {
            CK(cudaMemcpy(vals, m.data, bytes, cudaMemcpyDeviceToHost), "read array");
        } else {
            uint64_t *tmp;
            CK(cudaMalloc(&tmp, bytes), "cudaMalloc");
            int e = gx_k_pt_fold((const uint64_t *)m.data, m.nshards, s.max_entries, s.value_size / 8, tmp, 0);
            if (e) return cuda_err(rt, (cudaError_t)e, "pt fold");
            CK(cudaMemcpy(vals, tmp, bytes, cudaMemcpyDeviceToHost), "read pt");
            cudaFree(tmp);
        }
        if (keys)
            for (uint32_t k = 0; k < s.max_entries; k++) memcpy((uint8_t *)keys + 4 * k, &k, 4);
        *n_out = s.max_entries;
        return 0;
    }
    if (s.type == GX_MAP_HASH) {
        /* key words K[0 .. cap+1], then value words V (gx_device.cuh); K[cap] / K[cap+1] are the
         * presence states of the all-ones and the all-ones - 1 key */
        std::vector<uint64_t> w(2 * (m.cap + 2));
        CK(cudaMemcpy(w.data(), m.data, m.data_bytes, cudaMemcpyDeviceToHost), "read hash");
        const uint64_t *K = w.data(), *V = w.data() + m.cap + 2;
        std::vector<std::pair<uint64_t, uint64_t>> ent;
        for (uint64_t i = 0; i < m.cap; i++)
            if (K[i] < GX_HASH_EMPTY - 1) ent.push_back({K[i], V[i]});
        if (K[m.cap] == 1) ent.push_back({GX_HASH_EMPTY, V[m.cap]});
        if (K[m.cap + 1] == 1) ent.push_back({GX_HASH_EMPTY - 1, V[m.cap + 1]});
        std::sort(ent.begin(), ent.end());
        if (ent.size() > cap) return -E2BIG;
        for (size_t i = 0; i < ent.size(); i++) {
            if (keys) memcpy((uint8_t *)keys + s.key_size * i, &ent[i].first, s.key_size);
            memcpy((uint8_t *)vals + 8 * i, &ent[i].second, 8);
        }
        *n_out = ent.size();
        return 0;
    }
    return -EINVAL;
}

int gx_ringbuf_drain(gx_rt *rt, int fd, void *buf, uint64_t cap, uint64_t *n_bytes) {
    if (!check_map(rt, fd)) return -ENOENT;
    Map &m = rt->maps[fd];
    if (m.spec.type != GX_MAP_RINGBUF || !n_bytes) return -EINVAL;
    int rc0 = sync(rt);
    if (rc0) return rc0;
    uint64_t ctr[2];
    CK(cudaMemcpy(ctr, m.aux, 16, cudaMemcpyDeviceToHost), "ringbuf counters");
    uint64_t used = std::min<uint64_t>(ctr[1], m.cap);
    if (used > cap || (used && !buf)) {
        *n_bytes = used;
        return -E2BIG;
    }
    if (used) CK(cudaMemcpy(buf, m.data, used, cudaMemcpyDeviceToHost), "ringbuf data");
    CK(cudaMemset(m.aux, 0, 16), "ringbuf reset");
    *n_bytes = used;
    return 0;
}

int gx_prefetch_drain(gx_rt *rt, int fd, uint64_t *reqs, uint64_t cap, uint64_t *n_req) {
    if (!check_map(rt, fd)) return -ENOENT;
    Map &m = rt->maps[fd];
    if (m.spec.type != GX_MAP_PREFETCH_QUEUE || !n_req) return -EINVAL;
    int rc0 = sync(rt);
    if (rc0) return rc0;
    uint64_t reserved = 0;
    CK(cudaMemcpy(&reserved, m.aux, 8, cudaMemcpyDeviceToHost), "prefetch queue counter");
    const uint64_t n = std::min<uint64_t>(reserved, m.cap);
    if (n > cap || (n && !reqs)) {
        *n_req = n;
        return -E2BIG;
    }
    if (n) CK(cudaMemcpy(reqs, m.data, 16 * n, cudaMemcpyDeviceToHost), "prefetch queue data");
    CK(cudaMemset(m.aux, 0, 8), "prefetch queue reset");
    CK(cudaMemset((uint8_t *)m.data + 16 * m.cap, 0, 8ull * m.nshards), "prefetch filter reset");
    for (uint64_t i = 0; i < n; i++) reqs[2 * i + 1] &= 0xFFFFFFFFull; /* {first_page, npages} */
    *n_req = n;
    return 0;
}

int gx_load_prog(gx_rt *rt, uint32_t hook, const void *insn_slots, uint32_t n_slots, int *prog_fd) {
    if (!rt || !insn_slots || !prog_fd || n_slots == 0) return -EINVAL;
    if (n_slots > 4096) return set_err(rt, -E2BIG, "program has %u slots (max 4096)", n_slots);
    int fd = -1;
    for (int i = 0; i < GX_MAX_PROGS; i++)
        if (!rt->progs[i].valid) {
            fd = i;
            break;
        }
    if (fd < 0) return set_err(rt, -ENOMEM, "too many programs");
    Prog &p = rt->progs[fd];
    p = Prog();
    p.valid = true;
    p.hook = hook;
    p.slots.assign((const uint8_t *)insn_slots, (const uint8_t *)insn_slots + 8ull * n_slots);
    *prog_fd = fd;
    return 0;
}

int gx_verify(gx_rt *rt, int prog_fd, const gx_verify_opts *opts, gx_verify_report *report, char *log,
              uint64_t log_len) {
    NvtxScope nv("gx_verify");
    if (!check_prog(rt, prog_fd)) return -ENOENT;
    Prog &p = rt->progs[prog_fd];
    GxMapInfo mi[GX_MAX_MAPS];
    for (int i = 0; i < GX_MAX_MAPS; i++) {
        const Map &m = rt->maps[i];
        mi[i].valid = m.valid;
        mi[i].type = m.spec.type;
        mi[i].key_size = m.spec.key_size;
        mi[i].value_size = m.spec.value_size;
        mi[i].max_entries = m.spec.max_entries;
    }
    gx_verify_opts o{};
    if (opts) o = *opts;
    int v = gx_verify_program(p.slots.data(), (uint32_t)(p.slots.size() / 8), mi, o, p.vr);
    if (report) *report = p.vr.report;
    if (log && log_len) {
        size_t k = std::min<size_t>(log_len - 1, p.vr.log.size());
        memcpy(log, p.vr.log.data(), k);
        log[k] = 0;
    }
    if (v != 0) {
        p.verified = false;
        rt->err = p.vr.log;
        return v;
    }
    cudaFree(p.d_image);
    p.d_image = nullptr;
    CK(cudaMalloc(&p.d_image, p.vr.image.size() * sizeof(GxInsn)), "cudaMalloc image");
    CK(cudaMemcpy(p.d_image, p.vr.image.data(), p.vr.image.size() * sizeof(GxInsn), cudaMemcpyHostToDevice), "upload image");
    p.verified = true;
    rt->version++;
    return 0;
}

int gx_verify_offline(const void *insn_slots, uint32_t n_slots, const gx_map_spec *maps, uint32_t n_maps,
                      const gx_verify_opts *opts, gx_verify_report *report, char *log, uint64_t log_len) {
    if (!insn_slots || n_maps > GX_MAX_MAPS || (n_maps && !maps)) return -EINVAL;
    GxMapInfo mi[GX_MAX_MAPS];
    for (uint32_t i = 0; i < n_maps; i++) {
        mi[i].valid = maps[i].type != 0;
        mi[i].type = maps[i].type;
        mi[i].key_size = maps[i].key_size;
        mi[i].value_size = maps[i].value_size;
        mi[i].max_entries = maps[i].max_entries;
    }
    gx_verify_opts o{};
    if (opts) o = *opts;
    GxVerifyResult vr;
    int v = gx_verify_program((const uint8_t *)insn_slots, n_slots, mi, o, vr);
    if (report) *report = vr.report;
    if (log && log_len) {
        size_t k = std::min<size_t>(log_len - 1, vr.log.size());
        memcpy(log, vr.log.data(), k);
        log[k] = 0;
    }
    return v;
}

int gx_jit_offline(const void *insn_slots, uint32_t n_slots, const gx_map_spec *maps, uint32_t n_maps, char *src,
                   uint64_t src_len, char *log, uint64_t log_len) {
    if (!insn_slots || n_maps > GX_MAX_MAPS || (n_maps && !maps)) return -EINVAL;
    GxMapInfo mi[GX_MAX_MAPS];
    GxLaunch h;
    memset(&h, 0, sizeof h);
    memset(h.attach, -1, sizeof h.attach);
    for (uint32_t i = 0; i < n_maps; i++) {
        mi[i].valid = maps[i].type != 0;
        mi[i].type = maps[i].type;
        mi[i].key_size = maps[i].key_size;
        mi[i].value_size = maps[i].value_size;
        mi[i].max_entries = maps[i].max_entries;
        GxMapDesc &d = h.maps[i];
        d.data = 0x7f0000000000ull + ((uint64_t)i << 32);
        d.aux = d.data - 4096;
        d.type = maps[i].type;
        d.key_size = maps[i].key_size;
        d.value_size = maps[i].value_size;
        d.max_entries = maps[i].max_entries;
        d.nshards = maps[i].type == GX_MAP_PREFETCH_QUEUE ? GX_PFQ_FILTER_WORDS(maps[i].max_entries) : 303104;
        d.cap_mask = (maps[i].type == GX_MAP_RINGBUF || maps[i].type == GX_MAP_PREFETCH_QUEUE) ? maps[i].max_entries - 1
                                                                                              : 2 * maps[i].max_entries - 1;
        d.priv_off = 0xFFFFFFFFu;
        d.coherent = 1;
    }
    gx_verify_opts o{};
    GxVerifyResult vr;
    int v = gx_verify_program((const uint8_t *)insn_slots, n_slots, mi, o, vr);
    if (v) return v;
    h.n_progs = 1;
    h.single = 0;
    std::vector<const GxInsn *> images{vr.image.data()};
    std::vector<uint32_t> sizes{(uint32_t)vr.image.size()};
    std::vector<const uint16_t *> nin{vr.narrow_in.size() == vr.image.size() ? vr.narrow_in.data() : nullptr};
    unsigned vmask = GX_JIT_V_ALL; /* GX_JIT_VMASK: the launch variants to generate (GX_JIT_V_* bits) */
    if (const char *e = getenv("GX_JIT_VMASK")) vmask = (unsigned)strtoul(e, nullptr, 0) & GX_JIT_V_ALL;
    std::string s = gx_jit_source(h, images, sizes, gx_jit_block(), vmask ? vmask : GX_JIT_V_ALL, &nin);
    if (src && src_len) {
        size_t k = std::min<size_t>(src_len - 1, s.size());
        memcpy(src, s.data(), k);
        src[k] = 0;
    }
    std::vector<char> cubin;
    std::string lg;
    int rc = gx_jit_compile(s, cubin, lg);
    if (log && log_len) {
        size_t k = std::min<size_t>(log_len - 1, lg.size());
        memcpy(log, lg.data(), k);
        log[k] = 0;
    }
    return rc ? -ENOSYS : 0;
}

int gx_attach(gx_rt *rt, int prog_fd, uint32_t kind, uint32_t tenant) {
    if (!rt || kind >= GX_MAX_KINDS || tenant > 255) return -EINVAL;
    if (prog_fd >= 0 && !check_prog(rt, prog_fd)) return -ENOENT;
    rt->attach[kind][tenant] = prog_fd < 0 ? -1 : prog_fd;
    rt->version++;
    return 0;
}

int gx_run_batch(gx_rt *rt, const void *d_events, uint64_t n, int prog_fd, uint64_t *d_ret, void *stream) {
    NvtxScope nv("gx_run_batch");
    return gx_run_batch_ex(rt, d_events, n, prog_fd, d_ret, stream, 0);
}

int gx_run_batch_ex(gx_rt *rt, const void *d_events, uint64_t n, int prog_fd, uint64_t *d_ret, void *stream, uint32_t flags) {
    if (!rt) return -EINVAL;
    if (flags & ~(uint32_t)GX_RUN_OVERLAP) return set_err(rt, -EINVAL, "unknown run flags 0x%x", flags);
    if (n == 0) return 0;
    if (!d_events || ((uintptr_t)d_events & 31)) return set_err(rt, -EINVAL, "events must be 32-byte aligned device memory");
    if (prog_fd >= 0 && !check_prog(rt, prog_fd)) return -ENOENT;
    LaunchCfg *cfg;
    int rc = get_launch(rt, prog_fd, cfg);
    if (rc) return rc;
    return launch_cfg(rt, *cfg, d_events, n, d_ret, (cudaStream_t)stream, flags);
}

int gx_run_batch_host(gx_rt *rt, const void *h_events, uint64_t n, int prog_fd, uint64_t *h_ret) {
    NvtxScope nv("gx_run_batch_host");
    if (!rt || (!h_events && n)) return -EINVAL;
    if (n == 0) return 0;
    if (prog_fd >= 0 && !check_prog(rt, prog_fd)) return -ENOENT;
    LaunchCfg *cfg;
    int rc = get_launch(rt, prog_fd, cfg);
    if (rc) return rc;
    if (!rt->pipe_init) {
        CK(cudaStreamCreateWithFlags(&rt->s_copy, cudaStreamNonBlocking), "stream");
        CK(cudaStreamCreateWithFlags(&rt->s_exec, cudaStreamNonBlocking), "stream");
        for (int b = 0; b < 2; b++) {
            CK(cudaMalloc(&rt->d_chunk[b], kHostChunk * 32), "cudaMalloc chunk");
            CK(cudaMalloc(&rt->d_rchunk[b], kHostChunk * 8), "cudaMalloc chunk");
            CK(cudaEventCreateWithFlags(&rt->ev_copied[b], cudaEventDisableTiming), "event");
            CK(cudaEventCreateWithFlags(&rt->ev_done[b], cudaEventDisableTiming), "event");
            CK(cudaEventRecord(rt->ev_done[b], rt->s_exec), "event");
        }
        rt->pipe_init = true;
    }
    /* copies of chunk i+1 overlap the execution of chunk i; kernels stay serialised on s_exec
     * (per-thread shards are not shared between concurrent launches) */
    const uint8_t *src = (const uint8_t *)h_events;
    uint64_t nchunks = (n + kHostChunk - 1) / kHostChunk;
    for (uint64_t c = 0; c < nchunks; c++) {
        int b = (int)(c & 1);
        uint64_t i0 = c * kHostChunk, cnt = std::min(kHostChunk, n - i0);
        CK(cudaStreamWaitEvent(rt->s_copy, rt->ev_done[b], 0), "wait");
        CK(cudaMemcpyAsync(rt->d_chunk[b], src + 32 * i0, 32 * cnt, cudaMemcpyHostToDevice, rt->s_copy), "H2D");
        CK(cudaEventRecord(rt->ev_copied[b], rt->s_copy), "record");
        CK(cudaStreamWaitEvent(rt->s_exec, rt->ev_copied[b], 0), "wait");
        rc = launch_cfg(rt, *cfg, rt->d_chunk[b], cnt, h_ret ? rt->d_rchunk[b] : nullptr, rt->s_exec);
        if (rc) return rc;
        if (h_ret) CK(cudaMemcpyAsync(h_ret + i0, rt->d_rchunk[b], 8 * cnt, cudaMemcpyDeviceToHost, rt->s_exec), "D2H");
        CK(cudaEventRecord(rt->ev_done[b], rt->s_exec), "record");
    }
    CK(cudaStreamSynchronize(rt->s_exec), "sync");
    return 0;
}

int gx_daemon_watch(gx_rt *rt, int fd) {
    if (!rt || !check_map(rt, fd)) return -ENOENT;
    const uint32_t t = rt->maps[fd].spec.type;
    if (t != GX_MAP_ARRAY && t != GX_MAP_PERTHREAD_ARRAY)
        return set_err(rt, -EINVAL, "only ARRAY and PERTHREAD_ARRAY maps are snapshotted");
    if (rt->dmn.running) return set_err(rt, -EBUSY, "watch maps before gx_daemon_start");
    for (int w : rt->dmn.watched)
        if (w == fd) return 0;
    rt->dmn.watched.push_back(fd);
    return 0;
}

int gx_daemon_prefetch_range(gx_rt *rt, void *managed_ptr, uint64_t bytes) {
    if (!rt) return -EINVAL;
    rt->dmn.managed_ptr = (uint64_t)managed_ptr;
    rt->dmn.managed_bytes = managed_ptr ? bytes : 0;
    return 0;
}

int gx_daemon_start(gx_rt *rt, gx_prefetch_handler handler, void *user) {
    if (!rt) return -EINVAL;
    Daemon &D = rt->dmn;
    if (D.running) return set_err(rt, -EBUSY, "daemon already running");
    D.items.clear();
    D.item_fd.clear();
    D.folds.clear();
    uint64_t off = 0;
    for (int fd = 0; fd < GX_MAX_MAPS; fd++) {
        const Map &m = rt->maps[fd];
        if (!m.valid || m.spec.type != GX_MAP_PREFETCH_QUEUE) continue;
        GxPublishItem it{};
        it.data = (uint64_t)m.data;
        it.aux = (uint64_t)m.aux;
        it.cap = m.cap;
        it.nshards = m.nshards;
        it.kind = 0;
        it.host_off = off;
        off += 8 + 16 * m.cap;
        D.items.push_back(it);
        D.item_fd.push_back(fd);
    }
    for (int fd : D.watched) {
        const Map &m = rt->maps[fd];
        if (!m.valid) continue;
        GxPublishItem it{};
        it.data = (uint64_t)m.data;
        it.kind = 1;
        it.K = m.spec.max_entries;
        it.W = m.spec.value_size / 8;
        it.nshards = m.nshards;
        if (m.spec.type == GX_MAP_PERTHREAD_ARRAY) { /* folded into a staging copy first */
            uint64_t *stg = nullptr;
            CK(cudaMalloc(&stg, 8ull * it.K * it.W), "daemon fold staging");
            D.folds.push_back({(const uint64_t *)m.data, m.nshards, it.K, it.W, stg});
            it.data = (uint64_t)stg;
        }
        it.host_off = off;
        off += 8ull * it.K * it.W;
        D.items.push_back(it);
        D.item_fd.push_back(fd);
    }
    D.slot_bytes = std::max<uint64_t>(off, 64);
    for (auto &sl : D.slots) {
        CK(cudaHostAlloc((void **)&sl.host, D.slot_bytes, cudaHostAllocMapped), "daemon slot");
        CK(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming), "daemon event");
        sl.busy = false;
    }
    if (!D.items.empty()) {
        CK(cudaMalloc(&D.d_items, sizeof(GxPublishItem) * D.items.size()), "daemon items");
        CK(cudaMemcpy(D.d_items, D.items.data(), sizeof(GxPublishItem) * D.items.size(), cudaMemcpyHostToDevice), "daemon items");
    }
    CK(cudaStreamCreateWithFlags(&D.s_prefetch, cudaStreamNonBlocking), "daemon stream");
    D.fn = handler;
    D.user = user;
    D.stopping = false;
    D.pending.clear();
    D.snap.clear();
    D.version = 0;
    D.st = gx_daemon_stats{};
    D.running = true;
    D.th = std::thread(daemon_main, rt);
    return 0;
}

int gx_daemon_stop(gx_rt *rt) {
    if (!rt) return -EINVAL;
    Daemon &D = rt->dmn;
    if (!D.running) return 0;
    {
        std::lock_guard<std::mutex> lk(D.mu);
        D.stopping = true;
    }
    D.cv_work.notify_all();
    D.th.join();
    D.running = false;
    cudaStreamSynchronize(D.s_prefetch);
    cudaStreamDestroy(D.s_prefetch);
    for (auto &sl : D.slots) {
        cudaFreeHost(sl.host);
        cudaEventDestroy(sl.ev);
        sl = DaemonSlot{};
    }
    cudaFree(D.d_items);
    D.d_items = nullptr;
    for (auto &f : D.folds) cudaFree(f.staging);
    D.folds.clear();
    return 0;
}

int gx_snapshot_read(gx_rt *rt, int fd, void *buf, uint64_t cap, uint64_t *version) {
    if (!rt || !version) return -EINVAL;
    Daemon &D = rt->dmn;
    std::lock_guard<std::mutex> lk(D.mu);
    bool watched = false;
    for (int w : D.watched) watched |= w == fd;
    if (!watched) return -ENOENT;
    auto it = D.snap.find(fd);
    *version = it == D.snap.end() ? 0 : D.version;
    if (it == D.snap.end()) return 0;
    if (cap < it->second.size() || !buf) return -E2BIG;
    memcpy(buf, it->second.data(), it->second.size());
    return 0;
}

int gx_daemon_get_stats(gx_rt *rt, gx_daemon_stats *out) {
    if (!rt || !out) return -EINVAL;
    std::lock_guard<std::mutex> lk(rt->dmn.mu);
    *out = rt->dmn.st;
    return 0;
}

struct gx_kernel {
    CUmodule mod = nullptr;
    std::string log;
};

int gx_instrument(gx_rt *rt, int prog_fd, const char *user_src, gx_kernel **out, char *log, uint64_t log_len) {
    if (!rt || !user_src || !out) return -EINVAL;
    *out = nullptr;
    if (!check_prog(rt, prog_fd)) return -ENOENT;
    LaunchCfg *cfg;
    int rc = get_launch(rt, prog_fd, cfg);
    if (rc) return rc;
    Drv &d = drv();
    if (!d.ok) return set_err(rt, -ENOSYS, "driver entry points unavailable");
    GxLaunch h = cfg->h; /* no shared-memory privatisation inside a user kernel */
    for (auto &m : h.maps) m.priv_off = 0xFFFFFFFFu;
    h.n_priv = 0;
    h.priv_bytes = 0;
    const Prog &p = rt->progs[prog_fd];
    std::string src = gx_jit_instrument_source(h, p.vr.image.data(), (uint32_t)p.vr.image.size(), user_src);
    if (const char *dump = getenv("GX_JIT_DUMP")) {
        if (FILE *f = fopen(dump, "w")) {
            fputs(src.c_str(), f);
            fclose(f);
        }
    }
    std::vector<char> cubin;
    std::string lg;
    const int crc = gx_jit_compile(src, cubin, lg);
    if (log && log_len) {
        size_t k = std::min<size_t>(log_len - 1, lg.size());
        memcpy(log, lg.data(), k);
        log[k] = 0;
    }
    if (crc) return set_err(rt, -EINVAL, "instrumented module does not compile: %s", lg.c_str());
    gx_kernel *k = new gx_kernel();
    if (d.moduleLoadData(&k->mod, cubin.data()) != CUDA_SUCCESS) {
        delete k;
        return set_err(rt, -EFAULT, "cuModuleLoadData failed");
    }
    k->log = lg;
    *out = k;
    return 0;
}

int gx_kernel_launch(gx_rt *rt, gx_kernel *k, const char *name, const uint32_t grid[3], const uint32_t block[3],
                     uint32_t smem, void **args, void *stream) {
    if (!rt || !k || !name || !grid || !block) return -EINVAL;
    CUfunction fn = nullptr;
    if (drv().moduleGetFunction(&fn, k->mod, name) != CUDA_SUCCESS)
        return set_err(rt, -ENOENT, "no kernel '%s' in the instrumented module", name);
    if (smem > 48 * 1024 && drv().funcSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem) != CUDA_SUCCESS)
        return set_err(rt, -EINVAL, "cuFuncSetAttribute(%u B dynamic shared) failed", smem);
    if (drv().launchKernel(fn, grid[0], grid[1], grid[2], block[0], block[1], block[2], smem, (CUstream)stream, args,
                           nullptr) != CUDA_SUCCESS)
        return set_err(rt, -EFAULT, "instrumented kernel launch failed");
    rt->n_launches++;
    return 0;
}

/* f3: the thread-block scheduler of PAPER.md §4.3.2 / §6.2.1 (F-5, F-6) in two modes,
 * both driven by lane 0 of each block calling the policy through the inline hooks (gx_instrument):
 *  - DEQUE: persistent workers, one per block.  Deques are [head, tail) index pairs packed in one
 *    u64 per worker: the owner pops the head, thieves pop the tail, each with one CAS.
 *  - CLC: one block per unit (the plain grid), and "steal" is Blackwell cluster launch control
 *    ("MaxSteals (CLC)"): after its unit, a block whose should_try_steal says yes
 *    cancels a not-yet-launched block with clusterlaunchcontrol.try_cancel and runs that block's
 *    unit itself; a failed cancel (no block left to launch) or R0 == 0 ends the block.
 * Every hook call can be logged ({record, R0, worker, per-worker sequence number}) so that the
 * policy's decisions can be replayed through the oracle worker by worker. */
static const char *kSchedSrc = R"CUDA(
struct GxHookLog { unsigned rec[8]; unsigned long long r0; unsigned worker, seq; };
__device__ __forceinline__ unsigned long long gx_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void gx_spin_ns(unsigned long long ns) {
    const unsigned long long a = gx_now();
    while (gx_now() - a < ns) { }
}
struct GxSchedCtx {
    unsigned w, seq;
    GxHookLog *log;
    unsigned long long log_cap, *log_n;
    __device__ __forceinline__ unsigned long long hook(unsigned long long addr, unsigned kind, unsigned size) {
        unsigned rec[8];
        const unsigned long long r = gx_hook_event(1u, addr, kind, size, log ? rec : nullptr);
        if (log) {
            const unsigned long long i = atomicAdd(log_n, 1ull);
            if (i < log_cap) {
                GxHookLog *e = &log[i];
                for (int k = 0; k < 8; k++) e->rec[k] = rec[k];
                e->r0 = r;
                e->worker = w;
                e->seq = seq;
            }
        }
        seq++;
        return r;
    }
    /* one work unit: ENTER, [PROBE], the unit's body (a globaltimer spin), [RETPROBE], EXIT */
    __device__ __forceinline__ unsigned long long unit(unsigned u, unsigned st, unsigned cost_us, bool probes) {
        hook(u, 1u | (st << 16), cost_us);
        if (probes) hook(1ull, 6u, 0u);                 /* device function 1 = the unit body */
        const unsigned long long a = gx_now();
        gx_spin_ns(1000ull * cost_us);
        const unsigned long long b = gx_now() - a;
        if (probes) hook(1ull, 7u, u);                  /* its return value: the unit id */
        hook(u, 4u | (st << 16), cost_us);
        return b;
    }
};
extern "C" __global__ void gx_sched_worker(const unsigned *seg, const unsigned *off, unsigned long long *ht, unsigned W,
                                           const unsigned *cost_us, unsigned steal_cost_us, unsigned probes,
                                           unsigned *executed_by, unsigned char *stolen, unsigned long long *busy_ns,
                                           unsigned long long *start_ns, unsigned long long *end_ns, unsigned *steals,
                                           GxHookLog *log, unsigned long long log_cap, unsigned long long *log_n) {
    if (threadIdx.x != 0) return;      /* lane 0 is the worker; hooks run for the group {lane 0} */
    GxSchedCtx x{blockIdx.x, 0u, log, log_cap, log_n};
    const unsigned w = blockIdx.x;
    start_ns[w] = gx_now();
    unsigned long long busy = 0;
    unsigned nst = 0;
    for (;;) {
        unsigned u = 0, st = 0;
        bool got = false;
        for (;;) {                     /* own deque: pop the head */
            const unsigned long long old = *(volatile unsigned long long *)&ht[w];
            const unsigned h = (unsigned)old, t = (unsigned)(old >> 32);
            if (h >= t) break;
            if (atomicCAS(&ht[w], old, (unsigned long long)(h + 1) | ((unsigned long long)t << 32)) == old) {
                u = seg[off[w] + h];
                got = true;
                break;
            }
        }
        if (!got) {
            if (x.hook(0ull, 5u, 0u) == 0) break;      /* should_try_steal -> no */
            for (;;) {                 /* victim: largest deque, lowest id; take its tail */
                int v = -1;
                unsigned best = 0;
                unsigned long long vold = 0;
                for (unsigned k = 0; k < W; k++) {
                    const unsigned long long o = *(volatile unsigned long long *)&ht[k];
                    const unsigned len = (unsigned)(o >> 32) - (unsigned)o;
                    if ((unsigned)(o >> 32) > (unsigned)o && len > best) { best = len; v = (int)k; vold = o; }
                }
                if (v < 0) break;
                const unsigned h = (unsigned)vold, t = (unsigned)(vold >> 32);
                if (atomicCAS(&ht[v], vold, (unsigned long long)h | ((unsigned long long)(t - 1) << 32)) == vold) {
                    u = seg[off[v] + t - 1];
                    got = true;
                    break;
                }
            }
            if (!got) break;
            gx_spin_ns(1000ull * steal_cost_us);
            st = 1;
            nst++;
        }
        busy += x.unit(u, st, cost_us[u], probes != 0);
        executed_by[u] = w;
        stolen[u] = (unsigned char)st;
    }
    busy_ns[w] = busy;
    steals[w] = nst;
    end_ns[w] = gx_now();
}
extern "C" __global__ void gx_sched_clc(const unsigned *cost_us, unsigned steal_cost_us, unsigned probes,
                                        unsigned *executed_by, unsigned char *stolen, unsigned long long *busy_ns,
                                        unsigned long long *start_ns, unsigned long long *end_ns, unsigned *steals,
                                        GxHookLog *log, unsigned long long log_cap, unsigned long long *log_n) {
    __shared__ __align__(16) unsigned long long resp[2];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x != 0) return;
    const unsigned bar_a = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned resp_a = (unsigned)__cvta_generic_to_shared(resp);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar_a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    GxSchedCtx x{blockIdx.x, 0u, log, log_cap, log_n};
    const unsigned w = blockIdx.x;
    start_ns[w] = gx_now();
    unsigned long long busy = 0;
    unsigned nst = 0, u = w, st = 0, phase = 0;
    for (;;) {
        busy += x.unit(u, st, cost_us[u], probes != 0);
        executed_by[u] = w;
        stolen[u] = (unsigned char)st;
        if (x.hook(0ull, 5u, 0u) == 0) break;          /* should_try_steal -> no */
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" :: "r"(bar_a) : "memory");
        asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
                     :: "r"(resp_a), "r"(bar_a) : "memory");
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar_a), "r"(phase) : "memory");
        phase ^= 1u;
        unsigned ok = 0, cx = 0, cy, cz;
        asm volatile("{ .reg .pred p; .reg .b128 r; ld.shared.b128 r, [%4];\n"
                     "  clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n"
                     "  selp.u32 %3, 1, 0, p;\n"
                     "  @p clusterlaunchcontrol.query_cancel.get_first_ctaid.v4.b32.b128 {%0, %1, %2, _}, r; }"
                     : "=r"(cx), "=r"(cy), "=r"(cz), "=r"(ok) : "r"(resp_a) : "memory");
        if (!ok) break;                /* nothing left to launch: a later try_cancel would be undefined */
        u = cx;
        st = 1;
        nst++;
        gx_spin_ns(1000ull * steal_cost_us);
    }
    busy_ns[w] = busy;
    steals[w] = nst;
    end_ns[w] = gx_now();
}
)CUDA";

int gx_sched_run_ex(gx_rt *rt, int prog_fd, uint32_t flags, uint32_t n_units, const uint32_t *cost_us,
                    const uint32_t *home, uint32_t n_workers, uint32_t steal_cost_us, uint32_t smem_per_block,
                    uint32_t *executed_by, uint8_t *stolen, uint64_t *busy_ns, uint64_t *end_ns, uint32_t *steals,
                    uint64_t *makespan_ns, gx_hook_log *log, uint64_t log_cap, uint64_t *log_n) {
    if (!rt || !cost_us || !n_units || !executed_by || !stolen || !busy_ns || !end_ns || !steals || !makespan_ns)
        return -EINVAL;
    if (flags & ~(uint32_t)(GX_SCHED_CLC | GX_SCHED_PROBES)) return set_err(rt, -EINVAL, "unknown sched flags 0x%x", flags);
    if ((log_cap && !log) || (log && !log_n)) return set_err(rt, -EINVAL, "hook log needs log and log_n");
    const bool clc = flags & GX_SCHED_CLC;
    if (clc) {
        if (home) return set_err(rt, -EINVAL, "GX_SCHED_CLC: unit u is block u's (home must be NULL)");
        n_workers = n_units;
    } else {
        if (!home || !n_workers) return -EINVAL;
        for (uint32_t u = 0; u < n_units; u++)
            if (home[u] >= n_workers) return set_err(rt, -EINVAL, "unit %u homed on worker %u >= %u", u, home[u], n_workers);
    }
    gx_kernel *k = nullptr;
    int rc = gx_instrument(rt, prog_fd, kSchedSrc, &k, nullptr, 0);
    if (rc) return rc;
    const uint32_t W = n_workers;
    std::vector<uint32_t> off(W + 1, 0), seg(n_units), fill(W, 0);
    std::vector<unsigned long long> ht(W);
    if (!clc) {
        for (uint32_t u = 0; u < n_units; u++) off[home[u] + 1]++;
        for (uint32_t w = 0; w < W; w++) off[w + 1] += off[w];
        for (uint32_t u = 0; u < n_units; u++) seg[off[home[u]] + fill[home[u]]++] = u; /* deque in unit order */
        for (uint32_t w = 0; w < W; w++) ht[w] = (unsigned long long)(off[w + 1] - off[w]) << 32;
    }
    uint32_t *d_seg, *d_off, *d_cost, *d_exec, *d_steals;
    unsigned long long *d_ht, *d_busy, *d_start, *d_end, *d_logn;
    uint8_t *d_stolen;
    void *d_log = nullptr;
    CK(cudaMalloc(&d_seg, 4ull * n_units), "sched");
    CK(cudaMalloc(&d_off, 4ull * (W + 1)), "sched");
    CK(cudaMalloc(&d_cost, 4ull * n_units), "sched");
    CK(cudaMalloc(&d_exec, 4ull * n_units), "sched");
    CK(cudaMalloc(&d_stolen, n_units), "sched");
    CK(cudaMalloc(&d_steals, 4ull * W), "sched");
    CK(cudaMalloc(&d_ht, 8ull * W), "sched");
    CK(cudaMalloc(&d_busy, 8ull * W), "sched");
    CK(cudaMalloc(&d_start, 8ull * W), "sched");
    CK(cudaMalloc(&d_end, 8ull * W), "sched");
    CK(cudaMalloc(&d_logn, 8), "sched");
    if (log_cap) CK(cudaMalloc(&d_log, sizeof(gx_hook_log) * log_cap), "sched log");
    CK(cudaMemcpy(d_seg, seg.data(), 4ull * n_units, cudaMemcpyHostToDevice), "sched");
    CK(cudaMemcpy(d_off, off.data(), 4ull * (W + 1), cudaMemcpyHostToDevice), "sched");
    CK(cudaMemcpy(d_cost, cost_us, 4ull * n_units, cudaMemcpyHostToDevice), "sched");
    CK(cudaMemcpy(d_ht, ht.data(), 8ull * W, cudaMemcpyHostToDevice), "sched");
    CK(cudaMemset(d_exec, 0xFF, 4ull * n_units), "sched");
    CK(cudaMemset(d_stolen, 0, n_units), "sched");
    CK(cudaMemset(d_steals, 0, 4ull * W), "sched");
    CK(cudaMemset(d_busy, 0, 8ull * W), "sched");
    CK(cudaMemset(d_start, 0xFF, 8ull * W), "sched");   /* blocks cancelled by CLC never start */
    CK(cudaMemset(d_end, 0, 8ull * W), "sched");
    CK(cudaMemset(d_logn, 0, 8), "sched");
    uint32_t probes = (flags & GX_SCHED_PROBES) ? 1u : 0u;
    const uint32_t block[3] = {32, 1, 1};
    if (clc) {
        void *args[] = {&d_cost, &steal_cost_us, &probes, &d_exec, &d_stolen, &d_busy, &d_start, &d_end, &d_steals,
                        &d_log, &log_cap, &d_logn};
        const uint32_t grid[3] = {n_units, 1, 1};
        rc = gx_kernel_launch(rt, k, "gx_sched_clc", grid, block, smem_per_block, args, nullptr);
    } else {
        void *args[] = {&d_seg, &d_off, &d_ht, (void *)&W, &d_cost, &steal_cost_us, &probes, &d_exec, &d_stolen, &d_busy,
                        &d_start, &d_end, &d_steals, &d_log, &log_cap, &d_logn};
        const uint32_t grid[3] = {W, 1, 1};
        rc = gx_kernel_launch(rt, k, "gx_sched_worker", grid, block, smem_per_block, args, nullptr);
    }
    if (!rc) {
        CK(cudaDeviceSynchronize(), "sched run");
        std::vector<unsigned long long> st(W), en(W), bu(W);
        unsigned long long ln = 0;
        CK(cudaMemcpy(executed_by, d_exec, 4ull * n_units, cudaMemcpyDeviceToHost), "sched");
        CK(cudaMemcpy(stolen, d_stolen, n_units, cudaMemcpyDeviceToHost), "sched");
        CK(cudaMemcpy(steals, d_steals, 4ull * W, cudaMemcpyDeviceToHost), "sched");
        CK(cudaMemcpy(st.data(), d_start, 8ull * W, cudaMemcpyDeviceToHost), "sched");
        CK(cudaMemcpy(en.data(), d_end, 8ull * W, cudaMemcpyDeviceToHost), "sched");
        CK(cudaMemcpy(bu.data(), d_busy, 8ull * W, cudaMemcpyDeviceToHost), "sched");
        CK(cudaMemcpy(&ln, d_logn, 8, cudaMemcpyDeviceToHost), "sched");
        if (log_cap) CK(cudaMemcpy(log, d_log, sizeof(gx_hook_log) * std::min<uint64_t>(ln, log_cap), cudaMemcpyDeviceToHost), "sched");
        if (log_n) *log_n = ln;
        const unsigned long long t0 = *std::min_element(st.begin(), st.end());
        unsigned long long t1 = 0;
        for (uint32_t w = 0; w < W; w++) {
            busy_ns[w] = bu[w];
            end_ns[w] = en[w] ? en[w] - t0 : 0;              /* 0: a block cancelled before it started */
            t1 = std::max(t1, en[w]);
        }
        *makespan_ns = t1 - t0;
        if (log && ln > log_cap) rc = set_err(rt, -ENOSPC, "hook log: %llu hooks ran, %llu fit", ln, (unsigned long long)log_cap);
    }
    cudaFree(d_seg); cudaFree(d_off); cudaFree(d_cost); cudaFree(d_exec); cudaFree(d_stolen); cudaFree(d_steals);
    cudaFree(d_ht); cudaFree(d_busy); cudaFree(d_start); cudaFree(d_end); cudaFree(d_logn);
    if (d_log) cudaFree(d_log);
    gx_kernel_free(rt, k);
    return rc;
}

int gx_sched_run(gx_rt *rt, int prog_fd, uint32_t n_units, const uint32_t *cost_us, const uint32_t *home, uint32_t n_workers,
                 uint32_t steal_cost_us, uint32_t *executed_by, uint8_t *stolen, uint64_t *busy_ns, uint64_t *end_ns,
                 uint32_t *steals, uint64_t *makespan_ns) {
    if (!home) return -EINVAL;
    return gx_sched_run_ex(rt, prog_fd, 0, n_units, cost_us, home, n_workers, steal_cost_us, 0, executed_by, stolen,
                           busy_ns, end_ns, steals, makespan_ns, nullptr, 0, nullptr);
}

void gx_kernel_free(gx_rt *rt, gx_kernel *k) {
    (void)rt;
    if (!k) return;
    if (k->mod && drv().moduleUnload) drv().moduleUnload(k->mod);
    delete k;
}

int gx_get_stats(gx_rt *rt, gx_batch_stats *out) {
    if (!rt || !out) return -EINVAL;
    int rc0 = sync(rt);
    if (rc0) return rc0;
    unsigned long long h[GXS_N];
    CK(cudaMemcpy(h, rt->d_stats, sizeof h, cudaMemcpyDeviceToHost), "stats");
    CK(cudaMemset(rt->d_stats, 0, sizeof h), "stats reset");
    out->events_run = h[GXS_RUN];
    out->events_skipped = h[GXS_SKIP];
    out->divergent_steps = h[GXS_DIVERGENT];
    out->helper_errors = h[GXS_HERR];
    out->ringbuf_bytes = h[GXS_RB_BYTES];
    out->ringbuf_drops = h[GXS_RB_DROPS];
    out->hash_full = h[GXS_HFULL];
    out->warp_steps = h[GXS_STEPS];
    out->bounds_violations = h[GXS_BOUNDS];
    return 0;
}

int gx_set_engine(gx_rt *rt, int engine) {
    if (!rt || (engine != GX_ENGINE_INTERP && engine != GX_ENGINE_JIT)) return -EINVAL;
    rt->engine = engine;
    return 0;
}

int gx_get_engine(gx_rt *rt) { return rt ? rt->engine : -EINVAL; }

int gx_exec_info(gx_rt *rt, uint32_t *grid, uint32_t *block, uint32_t *smem, uint64_t *launches) {
    if (!rt) return -EINVAL;
    if (grid) *grid = rt->last_grid;
    if (block) *block = rt->last_block;
    if (smem) *smem = rt->last_smem;
    if (launches) *launches = rt->n_launches;
    return 0;
}

/* ------------------------------------------------------------------ merge (S3) */

int gx_merge_words(gx_rt *rt, int fd, uint64_t *words) {
    if (!check_map(rt, fd) || !words) return -EINVAL;
    const Map &m = rt->maps[fd];
    if (m.spec.type != GX_MAP_ARRAY && m.spec.type != GX_MAP_PERTHREAD_ARRAY) return -EINVAL;
    *words = (uint64_t)m.spec.max_entries * m.spec.value_size / 8;
    return 0;
}

static int ensure_base(gx_rt *rt, Map &m, bool retake = false) {
    if (m.base && !retake) return 0;
    if (m.base && retake) {
        CK(cudaDeviceSynchronize(), "snapshot");
        if (m.spec.type == GX_MAP_HASH) {
            CK(cudaMemcpy(m.base, m.data, m.data_bytes, cudaMemcpyDeviceToDevice), "base");
            CK(cudaMemcpy(m.base_aux, m.aux, 64, cudaMemcpyDeviceToDevice), "base");
        } else {
            uint64_t bytes = (uint64_t)m.spec.max_entries * m.spec.value_size;
            if (m.spec.type == GX_MAP_ARRAY) CK(cudaMemcpy(m.base, m.data, bytes, cudaMemcpyDeviceToDevice), "base");
            else {
                int e = gx_k_pt_fold((const uint64_t *)m.data, m.nshards, m.spec.max_entries, m.spec.value_size / 8,
                                     (uint64_t *)m.base, 0);
                if (e) return cuda_err(rt, (cudaError_t)e, "base fold");
            }
        }
        CK(cudaDeviceSynchronize(), "snapshot");
        return 0;
    }
    CK(cudaDeviceSynchronize(), "snapshot");
    if (m.spec.type == GX_MAP_HASH) {
        CK(cudaMalloc(&m.base, m.data_bytes), "cudaMalloc base");
        CK(cudaMalloc(&m.base_aux, 64), "cudaMalloc base");
        CK(cudaMemcpy(m.base, m.data, m.data_bytes, cudaMemcpyDeviceToDevice), "base");
        CK(cudaMemcpy(m.base_aux, m.aux, 64, cudaMemcpyDeviceToDevice), "base");
        return 0;
    }
    uint64_t bytes = (uint64_t)m.spec.max_entries * m.spec.value_size;
    CK(cudaMalloc(&m.base, bytes), "cudaMalloc base");
    if (m.spec.type == GX_MAP_ARRAY) CK(cudaMemcpy(m.base, m.data, bytes, cudaMemcpyDeviceToDevice), "base");
    else {
        int e = gx_k_pt_fold((const uint64_t *)m.data, m.nshards, m.spec.max_entries, m.spec.value_size / 8,
                             (uint64_t *)m.base, 0);
        if (e) return cuda_err(rt, (cudaError_t)e, "base fold");
    }
    CK(cudaDeviceSynchronize(), "base");
    return 0;
}

int gx_merge_snapshot(gx_rt *rt, int fd) {
    if (!check_map(rt, fd)) return -ENOENT;
    Map &m = rt->maps[fd];
    if (m.spec.type == GX_MAP_RINGBUF || m.spec.type == GX_MAP_PREFETCH_QUEUE || m.spec.type == GX_MAP_REGION) return -EINVAL;
    return ensure_base(rt, m, true);
}

int gx_merge_export(gx_rt *rt, int fd, uint64_t *d_delta, void *stream) {
    if (!check_map(rt, fd) || !d_delta) return -EINVAL;
    Map &m = rt->maps[fd];
    if (m.spec.type != GX_MAP_ARRAY && m.spec.type != GX_MAP_PERTHREAD_ARRAY) return -EINVAL;
    int rc = ensure_base(rt, m);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t words = (uint64_t)m.spec.max_entries * m.spec.value_size / 8;
    int e;
    if (m.spec.type == GX_MAP_ARRAY) {
        e = gx_k_sub((const uint64_t *)m.data, (const uint64_t *)m.base, d_delta, words, s);
    } else {
        e = gx_k_pt_fold((const uint64_t *)m.data, m.nshards, m.spec.max_entries, m.spec.value_size / 8, d_delta, s);
        if (!e) e = gx_k_sub(d_delta, (const uint64_t *)m.base, d_delta, words, s);
    }
    if (e) return cuda_err(rt, (cudaError_t)e, "merge export");
    return 0;
}

int gx_merge_apply(gx_rt *rt, int fd, const uint64_t *d_sum, void *stream) {
    if (!check_map(rt, fd) || !d_sum) return -EINVAL;
    Map &m = rt->maps[fd];
    if (m.spec.type != GX_MAP_ARRAY && m.spec.type != GX_MAP_PERTHREAD_ARRAY) return -EINVAL;
    int rc = ensure_base(rt, m);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t words = (uint64_t)m.spec.max_entries * m.spec.value_size / 8;
    /* base = base + sum; local = base */
    int e = gx_k_add((const uint64_t *)m.base, d_sum, (uint64_t *)m.base, words, s);
    if (!e) {
        if (m.spec.type == GX_MAP_ARRAY) {
            cudaError_t ce = cudaMemcpyAsync(m.data, m.base, words * 8, cudaMemcpyDeviceToDevice, s);
            if (ce != cudaSuccess) return cuda_err(rt, ce, "merge apply");
        } else {
            e = gx_k_pt_store_canonical((uint64_t *)m.data, m.nshards, m.spec.max_entries, m.spec.value_size / 8,
                                        (const uint64_t *)m.base, s);
        }
    }
    if (e) return cuda_err(rt, (cudaError_t)e, "merge apply");
    return 0;
}

int gx_hash_export(gx_rt *rt, int fd, uint32_t nranks, int32_t owner, uint64_t *d_keys, uint64_t *d_vals,
                   uint64_t cap, uint64_t *h_counts) {
    if (!check_map(rt, fd) || !h_counts || nranks == 0 || nranks > 4096 || owner >= (int32_t)nranks) return -EINVAL;
    Map &m = rt->maps[fd];
    if (m.spec.type != GX_MAP_HASH) return -EINVAL;
    int rc = ensure_base(rt, m);
    if (rc) return rc;
    unsigned long long *cnt, *off;
    CK(cudaMalloc(&cnt, 16ull * nranks), "cudaMalloc");
    off = cnt + nranks;
    CK(cudaMemset(cnt, 0, 16ull * nranks), "memset");
    GxMapDesc d = make_desc(m), b = make_base_desc(m);
    int e = gx_k_hash_export(&d, &b, nranks, owner, 0, cnt, off, d_keys, d_vals, cap, 0);
    if (e) return cuda_err(rt, (cudaError_t)e, "hash export");
    std::vector<unsigned long long> c(nranks), o(nranks);
    CK(cudaMemcpy(c.data(), cnt, 8ull * nranks, cudaMemcpyDeviceToHost), "hash export counts");
    uint64_t total = 0;
    for (uint32_t g = 0; g < nranks; g++) {
        o[g] = total;
        total += c[g];
        h_counts[g] = c[g];
    }
    if (total > cap) {
        cudaFree(cnt);
        return set_err(rt, -E2BIG, "hash export needs %llu entries (cap %llu)", (unsigned long long)total,
                       (unsigned long long)cap);
    }
    if (total) {
        CK(cudaMemcpy(off, o.data(), 8ull * nranks, cudaMemcpyHostToDevice), "hash export offsets");
        e = gx_k_hash_export(&d, &b, nranks, owner, 1, cnt, off, d_keys, d_vals, cap, 0);
        if (e) return cuda_err(rt, (cudaError_t)e, "hash export");
    }
    CK(cudaDeviceSynchronize(), "hash export");
    cudaFree(cnt);
    return 0;
}

int gx_hash_apply(gx_rt *rt, int fd, const uint64_t *d_keys, const uint64_t *d_vals, uint64_t n, uint32_t flags,
                  void *stream) {
    if (!check_map(rt, fd) || (n && (!d_keys || !d_vals)) || (flags & ~3u)) return -EINVAL;
    Map &m = rt->maps[fd];
    if (m.spec.type != GX_MAP_HASH) return -EINVAL;
    int rc = ensure_base(rt, m);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (flags & GX_MERGE_RESTORE) {
        CK(cudaMemcpyAsync(m.data, m.base, m.data_bytes, cudaMemcpyDeviceToDevice, s), "hash restore");
        CK(cudaMemcpyAsync(m.aux, m.base_aux, 64, cudaMemcpyDeviceToDevice, s), "hash restore");
    }
    unsigned long long *full;
    CK(cudaMalloc(&full, 8), "cudaMalloc");
    CK(cudaMemsetAsync(full, 0, 8, s), "memset");
    GxMapDesc d = make_desc(m);
    if (n) {
        int e = gx_k_hash_accumulate(&d, d_keys, d_vals, n, full, s);
        if (e) return cuda_err(rt, (cudaError_t)e, "hash accumulate");
    }
    if (flags & GX_MERGE_COMMIT) {
        CK(cudaMemcpyAsync(m.base, m.data, m.data_bytes, cudaMemcpyDeviceToDevice, s), "hash commit");
        CK(cudaMemcpyAsync(m.base_aux, m.aux, 64, cudaMemcpyDeviceToDevice, s), "hash commit");
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, full, 8, cudaMemcpyDeviceToHost, s), "hash full");
    CK(cudaStreamSynchronize(s), "sync");
    cudaFree(full);
    if (h) return set_err(rt, -E2BIG, "merged hash union exceeds max_entries (%llu refused)", h);
    return 0;
}

}  // extern "C"

/* ------------------------------------------------------------------ gx_comm_init / gx_merge (S3) */

namespace {


struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};
NcclApi &nccl() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        /* the NCCL already in the process (torch.distributed's) first, then GX_NCCL_LIB, then the
         * loader path */
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h && getenv("GX_NCCL_LIB")) h = dlopen(getenv("GX_NCCL_LIB"), RTLD_NOW);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) {
            a.err = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
#define GX_NCCL_SYM(f, n) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, n))
        GX_NCCL_SYM(getUniqueId, "ncclGetUniqueId");
        GX_NCCL_SYM(commInitRank, "ncclCommInitRank");
        GX_NCCL_SYM(commDestroy, "ncclCommDestroy");
        GX_NCCL_SYM(allReduce, "ncclAllReduce");
        GX_NCCL_SYM(allGather, "ncclAllGather");
        GX_NCCL_SYM(send, "ncclSend");
        GX_NCCL_SYM(recv, "ncclRecv");
        GX_NCCL_SYM(groupStart, "ncclGroupStart");
        GX_NCCL_SYM(groupEnd, "ncclGroupEnd");
        GX_NCCL_SYM(getErrorString, "ncclGetErrorString");
#undef GX_NCCL_SYM
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.allReduce && a.allGather && a.send && a.recv &&
               a.groupStart && a.groupEnd;
        if (!a.ok) a.err = "libnccl.so.2 lacks a needed symbol";
    });
    return a;
}

/* NCCL: the collectives are stream-ordered on the merge stream; point-to-point exchanges are one
 * grouped send/recv set (the all-to-all of the key-sharded hash merge) */
struct NcclComm : GxComm {
    ncclComm_t comm = nullptr;
    std::string last;
    bool device_buffers() const override { return true; }
    int fail(ncclResult_t r, const char *what) {
        last = std::string(what) + ": " + (nccl().getErrorString ? nccl().getErrorString(r) : "nccl error");
        return -EIO;
    }
    int allreduce_sum_u64(uint64_t *buf, uint64_t n, cudaStream_t s) override {
        if (!n) return 0;
        ncclResult_t r = nccl().allReduce(buf, buf, n, ncclUint64, ncclSum, comm, s);
        return r == ncclSuccess ? 0 : fail(r, "ncclAllReduce");
    }
    int alltoallv(const uint8_t *send, const uint64_t *sb, const uint64_t *so, uint8_t *recv, const uint64_t *rb,
                  const uint64_t *ro, cudaStream_t s) override {
        ncclResult_t r = nccl().groupStart();
        for (int g = 0; g < nranks && r == ncclSuccess; g++) {
            if (sb[g]) r = nccl().send(send + so[g], sb[g], ncclUint8, g, comm, s);
            if (r == ncclSuccess && rb[g]) r = nccl().recv(recv + ro[g], rb[g], ncclUint8, g, comm, s);
        }
        ncclResult_t r2 = nccl().groupEnd();
        if (r != ncclSuccess) return fail(r, "ncclSend/ncclRecv");
        return r2 == ncclSuccess ? 0 : fail(r2, "ncclGroupEnd");
    }
    int allgather(const void *send, void *recv, uint64_t bytes, cudaStream_t s) override {
        ncclResult_t r = nccl().allGather(send, recv, bytes, ncclUint8, comm, s);
        return r == ncclSuccess ? 0 : fail(r, "ncclAllGather");
    }
    const char *error() const override { return last.c_str(); }
    ~NcclComm() override {
        if (comm) nccl().commDestroy(comm);
    }
};

/* host callbacks (gx_comm_host_ops): buffers are staged through host memory */
struct HostComm : GxComm {
    gx_comm_host_ops ops{};
    bool device_buffers() const override { return false; }
    int allreduce_sum_u64(uint64_t *buf, uint64_t n, cudaStream_t) override {
        return n ? ops.allreduce_sum_u64(ops.user, buf, n) : 0;
    }
    int alltoallv(const uint8_t *send, const uint64_t *sb, const uint64_t *so, uint8_t *recv, const uint64_t *rb,
                  const uint64_t *ro, cudaStream_t) override {
        return ops.alltoallv(ops.user, send, sb, so, recv, rb, ro);
    }
    int allgather(const void *send, void *recv, uint64_t bytes, cudaStream_t) override {
        return ops.allgather(ops.user, send, recv, bytes);
    }
};

/* S3 legality of a map (the verifier's usage facts of every loaded program):
 * ARRAY -- changed only by 64-bit ATOMIC ADD (+-FETCH); PERTHREAD -- any per-thread RMW (its
 * canonical value is the SUM fold, S4); HASH -- values changed only by 64-bit ATOMIC ADD and keys
 * inserted only by update_elem(BPF_NOEXIST).  Returns nullptr or the reason. */
const char *merge_illegal(const gx_rt *rt, int fd) {
    const Map &m = rt->maps[fd];
    for (const Prog &p : rt->progs) {
        if (!p.valid || !p.verified) continue;
        const GxMapUse &u = p.vr.use[fd];
        if (!u.used || !u.writes) continue;
        if (m.spec.type == GX_MAP_ARRAY) {
            if (u.store) return "written by a plain store or a non-ADD atomic";
            if (u.update_call) return "written by bpf_map_update_elem";
            if (u.non_dw_atomic) return "written by a 32-bit atomic";
        } else if (m.spec.type == GX_MAP_HASH) {
            if (u.store) return "values written by a plain store or a non-ADD atomic";
            if (u.upd_overwrite) return "updated with flags other than the constant BPF_NOEXIST";
            if (u.non_dw_atomic) return "values changed by a 32-bit atomic";
        }
    }
    return nullptr;
}

int ms_reserve(gx_rt *rt, uint64_t words) {
    if (rt->ms.words >= words) return 0;
    cudaFree(rt->ms.d);
    rt->ms.d = nullptr;
    rt->ms.words = 0;
    CK(cudaMalloc(&rt->ms.d, words * 8), "cudaMalloc merge scratch");
    rt->ms.words = words;
    if (!rt->comm->device_buffers()) rt->ms.h.resize(words);
    return 0;
}

int comm_err(gx_rt *rt, int rc, const char *what) {
    return set_err(rt, rc ? rc : -EIO, "%s: %s", what, rt->comm ? rt->comm->error() : "");
}

/* the S3 merge of one HASH map: owner-bucketed deltas -> all-to-all -> owners accumulate onto the
 * base -> owners' merged deltas -> all-gather -> every rank rebuilds base + merged deltas */
int merge_hash(gx_rt *rt, Map &m, cudaStream_t s) {
    GxComm &C = *rt->comm;
    const uint32_t G = (uint32_t)C.nranks;
    const uint64_t cap = (uint64_t)m.cap + 2; /* entries a map can export (slots + side slots) */
    /* scratch: [counts 2G | offsets G] [send keys | send vals] [recv keys | recv vals] (cap each) */
    const uint64_t nrecv = cap * G;
    int rc = ms_reserve(rt, 3ull * G + 2 * cap + 2 * nrecv);
    if (rc) return rc;
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(rt->ms.d), *off = cnt + G;
    uint64_t *sk = rt->ms.d + 3ull * G, *sv = sk + cap, *rk = sv + cap, *rv = rk + nrecv;
    GxMapDesc d = make_desc(m), b = make_base_desc(m);
    auto export_pass = [&](int32_t owner, std::vector<uint64_t> &counts) -> int {
        CK(cudaMemsetAsync(cnt, 0, 16ull * G, s), "memset");
        int e = gx_k_hash_export(&d, &b, G, owner, 0, cnt, off, sk, sv, cap, s);
        if (e) return cuda_err(rt, (cudaError_t)e, "hash export");
        counts.assign(G, 0);
        CK(cudaMemcpyAsync(counts.data(), cnt, 8ull * G, cudaMemcpyDeviceToHost, s), "export counts");
        CK(cudaStreamSynchronize(s), "export counts");
        std::vector<uint64_t> o(G);
        uint64_t t = 0;
        for (uint32_t g = 0; g < G; g++) o[g] = t, t += counts[g];
        if (t) {
            CK(cudaMemcpyAsync(off, o.data(), 8ull * G, cudaMemcpyHostToDevice, s), "export offsets");
            e = gx_k_hash_export(&d, &b, G, owner, 1, cnt, off, sk, sv, cap, s);
            if (e) return cuda_err(rt, (cudaError_t)e, "hash export");
        }
        return 0;
    };
    /* device or host views of the exchange buffers */
    const bool dev = C.device_buffers();
    auto stage_out = [&](uint64_t *dptr, uint64_t n) -> uint8_t * {
        if (dev) return reinterpret_cast<uint8_t *>(dptr);
        uint64_t *h = rt->ms.h.data() + (dptr - rt->ms.d);
        if (n) cudaMemcpyAsync(h, dptr, 8 * n, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        return reinterpret_cast<uint8_t *>(h);
    };
    auto host_of = [&](uint64_t *dptr) -> uint8_t * {
        return dev ? reinterpret_cast<uint8_t *>(dptr) : reinterpret_cast<uint8_t *>(rt->ms.h.data() + (dptr - rt->ms.d));
    };
    auto stage_in = [&](uint64_t *dptr, uint64_t n) -> int {
        if (!dev && n) CK(cudaMemcpyAsync(dptr, rt->ms.h.data() + (dptr - rt->ms.d), 8 * n, cudaMemcpyHostToDevice, s), "stage in");
        return 0;
    };
    /* 1. deltas grouped by owner; the G x G count matrix by all-gather */
    std::vector<uint64_t> mine;
    if ((rc = export_pass(-1, mine))) return rc;
    std::vector<uint64_t> mat(G * (uint64_t)G);
    {
        /* counts travel through the recv-key region (device) or host staging */
        uint64_t *tmp = rk;
        CK(cudaMemcpyAsync(tmp, mine.data(), 8ull * G, cudaMemcpyHostToDevice, s), "counts");
        uint8_t *src = stage_out(tmp, G);
        uint8_t *dst = host_of(rv);
        if ((rc = C.allgather(src, dst, 8ull * G, s))) return comm_err(rt, rc, "hash merge counts");
        if (dev) {
            CK(cudaMemcpyAsync(mat.data(), rv, 8ull * G * G, cudaMemcpyDeviceToHost, s), "counts");
            CK(cudaStreamSynchronize(s), "counts");
        } else {
            memcpy(mat.data(), dst, 8ull * G * G);
        }
    }
    /* 2. all-to-all of (key, delta) pairs: keys, then deltas */
    std::vector<uint64_t> sb(G), so(G), rb(G), ro(G);
    uint64_t nin = 0;
    for (uint32_t g = 0, t = 0; g < G; g++) {
        sb[g] = 8 * mine[g];
        so[g] = 8ull * t;
        t += (uint32_t)mine[g];
        rb[g] = 8 * mat[(uint64_t)g * G + C.rank];
        ro[g] = 8 * nin;
        nin += mat[(uint64_t)g * G + C.rank];
    }
    uint64_t nout = 0;
    for (uint32_t g = 0; g < G; g++) nout += mine[g];
    for (int pass = 0; pass < 2; pass++) {
        uint64_t *sp = pass ? sv : sk, *rp = pass ? rv : rk;
        uint8_t *src = stage_out(sp, nout);
        if ((rc = C.alltoallv(src, sb.data(), so.data(), host_of(rp), rb.data(), ro.data(), s)))
            return comm_err(rt, rc, "hash merge all-to-all");
        if ((rc = stage_in(rp, nin))) return rc;
    }
    /* 3. owner: base + every rank's deltas of its keys */
    unsigned long long *full = cnt + 2 * G; /* one spare word after the offsets */
    CK(cudaMemsetAsync(full, 0, 8, s), "memset");
    CK(cudaMemcpyAsync(m.data, m.base, m.data_bytes, cudaMemcpyDeviceToDevice, s), "hash restore");
    CK(cudaMemcpyAsync(m.aux, m.base_aux, 64, cudaMemcpyDeviceToDevice, s), "hash restore");
    if (nin) {
        int e = gx_k_hash_accumulate(&d, rk, rv, nin, full, s);
        if (e) return cuda_err(rt, (cudaError_t)e, "hash accumulate");
    }
    /* 4. the owners' merged deltas to everybody */
    std::vector<uint64_t> own;
    if ((rc = export_pass((int32_t)C.rank, own))) return rc;
    const uint64_t n_own = own[C.rank];
    std::vector<uint64_t> all_n(G);
    {
        CK(cudaMemcpyAsync(rk, &n_own, 8, cudaMemcpyHostToDevice, s), "owner count");
        uint8_t *src = stage_out(rk, 1);
        uint8_t *dst = host_of(rv);
        if ((rc = C.allgather(src, dst, 8, s))) return comm_err(rt, rc, "hash merge owner counts");
        if (dev) {
            CK(cudaMemcpyAsync(all_n.data(), rv, 8ull * G, cudaMemcpyDeviceToHost, s), "owner counts");
            CK(cudaStreamSynchronize(s), "owner counts");
        } else {
            memcpy(all_n.data(), dst, 8ull * G);
        }
    }
    /* the owner's entries start at its own offset in the export (owner >= 0 keeps only its keys) */
    uint64_t own_off = 0;
    for (int g = 0; g < C.rank; g++) own_off += own[g];
    uint64_t ntot = 0;
    for (uint32_t g = 0; g < G; g++) {
        sb[g] = 8 * n_own;
        so[g] = 8 * own_off;
        rb[g] = 8 * all_n[g];
        ro[g] = 8 * ntot;
        ntot += all_n[g];
    }
    for (int pass = 0; pass < 2; pass++) {
        uint64_t *sp = pass ? sv : sk, *rp = pass ? rv : rk;
        uint8_t *src = stage_out(sp, own_off + n_own);
        if ((rc = C.alltoallv(src, sb.data(), so.data(), host_of(rp), rb.data(), ro.data(), s)))
            return comm_err(rt, rc, "hash merge all-gather");
        if ((rc = stage_in(rp, ntot))) return rc;
    }
    /* 5. every rank: base + all merged deltas; commit as the new base */
    CK(cudaMemcpyAsync(m.data, m.base, m.data_bytes, cudaMemcpyDeviceToDevice, s), "hash restore");
    CK(cudaMemcpyAsync(m.aux, m.base_aux, 64, cudaMemcpyDeviceToDevice, s), "hash restore");
    CK(cudaMemsetAsync(full, 0, 8, s), "memset");
    if (ntot) {
        int e = gx_k_hash_accumulate(&d, rk, rv, ntot, full, s);
        if (e) return cuda_err(rt, (cudaError_t)e, "hash accumulate");
    }
    CK(cudaMemcpyAsync(m.base, m.data, m.data_bytes, cudaMemcpyDeviceToDevice, s), "hash commit");
    CK(cudaMemcpyAsync(m.base_aux, m.aux, 64, cudaMemcpyDeviceToDevice, s), "hash commit");
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, full, 8, cudaMemcpyDeviceToHost, s), "hash full");
    CK(cudaStreamSynchronize(s), "hash merge");
    if (h) return set_err(rt, -E2BIG, "merged HASH union exceeds max_entries (%llu keys refused)", h);
    return 0;
}

int comm_attach(gx_rt *rt, std::unique_ptr<GxComm> c) {
    rt->comm = std::move(c);
    rt->merges = 0;
    /* the agreed initial state: every mergeable map's base snapshot, now */
    for (int fd = 0; fd < GX_MAX_MAPS; fd++) {
        Map &m = rt->maps[fd];
        if (!m.valid || m.spec.type == GX_MAP_RINGBUF || m.spec.type == GX_MAP_PREFETCH_QUEUE || m.spec.type == GX_MAP_REGION)
            continue;
        int rc = ensure_base(rt, m, true);
        if (rc) return rc;
    }
    return 0;
}

}  // namespace

extern "C" {

int gx_comm_unique_id(void *id_out) {
    if (!id_out) return -EINVAL;
    NcclApi &a = nccl();
    if (!a.ok) return -ENOSYS;
    ncclUniqueId id;
    if (a.getUniqueId(&id) != ncclSuccess) return -EIO;
    memcpy(id_out, &id, sizeof id);
    return 0;
}

int gx_comm_init(gx_rt *rt, const void *nccl_unique_id, int nranks, int rank) {
    if (!rt || !nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks) return -EINVAL;
    NcclApi &a = nccl();
    if (!a.ok) return set_err(rt, -ENOSYS, "NCCL unavailable: %s", a.err.c_str());
    CK(cudaSetDevice(rt->dev), "cudaSetDevice");
    auto c = std::make_unique<NcclComm>();
    c->nranks = nranks;
    c->rank = rank;
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof id);
    ncclResult_t r = a.commInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess)
        return set_err(rt, -EIO, "ncclCommInitRank: %s", a.getErrorString ? a.getErrorString(r) : "error");
    return comm_attach(rt, std::move(c));
}

int gx_comm_init_host(gx_rt *rt, const gx_comm_host_ops *ops, int nranks, int rank) {
    if (!rt || !ops || !ops->allreduce_sum_u64 || !ops->alltoallv || !ops->allgather || nranks < 1 || rank < 0 ||
        rank >= nranks)
        return -EINVAL;
    auto c = std::make_unique<HostComm>();
    c->nranks = nranks;
    c->rank = rank;
    c->ops = *ops;
    return comm_attach(rt, std::move(c));
}

int gx_merge(gx_rt *rt, void *cuda_stream) {
    NvtxScope nv("gx_merge");
    if (!rt) return -EINVAL;
    gx_log(2, "merge %llu", (unsigned long long)rt->merges);
    if (!rt->comm) return set_err(rt, -EINVAL, "gx_merge before gx_comm_init");
    CK(cudaSetDevice(rt->dev), "cudaSetDevice");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    /* legality first, on every map (a refusal leaves every map untouched) */
    for (int fd = 0; fd < GX_MAX_MAPS; fd++) {
        const Map &m = rt->maps[fd];
        if (!m.valid || m.spec.type == GX_MAP_RINGBUF || m.spec.type == GX_MAP_PREFETCH_QUEUE || m.spec.type == GX_MAP_REGION)
            continue;
        if (const char *why = merge_illegal(rt, fd))
            return set_err(rt, -EINVAL, "map %d cannot be merged (S3): %s", fd, why);
    }
    /* 1. additive maps (ARRAY, PERTHREAD folded): one packed u64 all-reduce of local - base */
    uint64_t total = 0;
    for (int fd = 0; fd < GX_MAX_MAPS; fd++) {
        const Map &m = rt->maps[fd];
        if (m.valid && (m.spec.type == GX_MAP_ARRAY || m.spec.type == GX_MAP_PERTHREAD_ARRAY))
            total += (uint64_t)m.spec.max_entries * m.spec.value_size / 8;
    }
    if (total) {
        int rc = ms_reserve(rt, total);
        if (rc) return rc;
        uint64_t off = 0;
        for (int fd = 0; fd < GX_MAX_MAPS; fd++) {
            const Map &m = rt->maps[fd];
            if (!m.valid || (m.spec.type != GX_MAP_ARRAY && m.spec.type != GX_MAP_PERTHREAD_ARRAY)) continue;
            rc = gx_merge_export(rt, fd, rt->ms.d + off, s);
            if (rc) return rc;
            off += (uint64_t)m.spec.max_entries * m.spec.value_size / 8;
        }
        uint64_t *buf = rt->ms.d;
        if (!rt->comm->device_buffers()) {
            CK(cudaMemcpyAsync(rt->ms.h.data(), rt->ms.d, 8 * total, cudaMemcpyDeviceToHost, s), "merge stage");
            CK(cudaStreamSynchronize(s), "merge stage");
            buf = rt->ms.h.data();
        }
        rc = rt->comm->allreduce_sum_u64(buf, total, s);
        if (rc) return comm_err(rt, rc, "merge all-reduce");
        if (!rt->comm->device_buffers())
            CK(cudaMemcpyAsync(rt->ms.d, rt->ms.h.data(), 8 * total, cudaMemcpyHostToDevice, s), "merge stage");
        off = 0;
        for (int fd = 0; fd < GX_MAX_MAPS; fd++) {
            const Map &m = rt->maps[fd];
            if (!m.valid || (m.spec.type != GX_MAP_ARRAY && m.spec.type != GX_MAP_PERTHREAD_ARRAY)) continue;
            rc = gx_merge_apply(rt, fd, rt->ms.d + off, s);
            if (rc) return rc;
            off += (uint64_t)m.spec.max_entries * m.spec.value_size / 8;
        }
    }
    /* 2. HASH maps: key-sharded exchange */
    for (int fd = 0; fd < GX_MAX_MAPS; fd++) {
        Map &m = rt->maps[fd];
        if (!m.valid || m.spec.type != GX_MAP_HASH) continue;
        int rc = ensure_base(rt, m);
        if (rc) return rc;
        rc = merge_hash(rt, m, s);
        if (rc) return rc;
    }
    CK(cudaStreamSynchronize(s), "merge");
    rt->merges++;
    return 0;
}

int gx_comm_free(gx_rt *rt) {
    if (!rt) return -EINVAL;
    rt->comm.reset();
    return 0;
}

}  // extern "C"
