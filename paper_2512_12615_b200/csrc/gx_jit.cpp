/*
 * gx_jit.cpp -- per-launch JIT of verified programs to sm_100a machine code.
 *
 * "Verified programs are JIT-compiled into native host code or GPU-compatible instructions (e.g.,
 * PTX)" (§4.2); "an LLVM-based backend translates the restricted gpu_ext eBPF
 * instruction subset into GPU device code (PTX)" (§5.1); helpers and map accesses are
 * inlined.  Here the verifier's pre-decoded image (every memory access already
 * resolved to ctx / stack / map / per-thread kind, every helper to its map and argument slots) is
 * translated to straight-line CUDA C++ and compiled by NVRTC for sm_100a; the cubin is loaded with
 * cudaLibraryLoadData.  One kernel per launch configuration (programs + attach table + map
 * descriptors, which are baked in as constants); cached by the runtime.
 *
 * NVRTC is loaded with dlopen so libgx.so has no link-time dependency on it.
 */
#include "gx_jit.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <cstdlib>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "gx_jit_headers.inc"  /* kJitHeaders[]: {name, text} of the device headers */

namespace {

struct Nvrtc {
    bool ok = false;
    std::string err;
    decltype(&nvrtcCreateProgram) create;
    decltype(&nvrtcCompileProgram) compile;
    decltype(&nvrtcGetCUBINSize) cubin_size;
    decltype(&nvrtcGetCUBIN) cubin;
    decltype(&nvrtcGetProgramLogSize) log_size;
    decltype(&nvrtcGetProgramLog) log;
    decltype(&nvrtcDestroyProgram) destroy;
    decltype(&nvrtcGetErrorString) errstr;
};

Nvrtc &nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *cands[] = {getenv("GX_NVRTC"), "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                               "/usr/local/cuda/lib64/libnvrtc.so", "libnvrtc.so"};
        void *h = nullptr;
        for (const char *c : cands)
            if (c && (h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) {
            n.err = "cannot dlopen libnvrtc.so.12";
            return;
        }
#define LOAD(f, name)                                              \
    n.f = (decltype(n.f))dlsym(h, name);                           \
    if (!n.f) {                                                    \
        n.err = std::string("libnvrtc lacks ") + name;             \
        return;                                                    \
    }
        LOAD(create, "nvrtcCreateProgram");
        LOAD(compile, "nvrtcCompileProgram");
        LOAD(cubin_size, "nvrtcGetCUBINSize");
        LOAD(cubin, "nvrtcGetCUBIN");
        LOAD(log_size, "nvrtcGetProgramLogSize");
        LOAD(log, "nvrtcGetProgramLog");
        LOAD(destroy, "nvrtcDestroyProgram");
        LOAD(errstr, "nvrtcGetErrorString");
#undef LOAD
        n.ok = true;
    });
    return n;
}

std::string hex(uint64_t v) {
    char b[32];
    snprintf(b, sizeof b, "0x%llxull", (unsigned long long)v);
    return b;
}

struct Gen {
    std::ostringstream o;
    const GxLaunch &L;
    explicit Gen(const GxLaunch &l) : L(l) {}

    std::string md(int fd) {
        const GxMapDesc &d = L.maps[fd];
        std::ostringstream s;
        s << "GxMapDesc{" << hex(d.data) << ", " << hex(d.aux) << ", " << d.type << "u, " << d.key_size << "u, "
          << d.value_size << "u, " << d.max_entries << "u, " << d.nshards << "u, " << d.cap_mask << "u, "
          << d.priv_off << "u, " << d.coherent << "u}";
        return s.str();
    }

    static std::string R(int r) { return "r" + std::to_string(r); }
    /* physical address of a per-thread word: the constant-geometry form when the map's logical
     * span fits 32-bit index arithmetic */
    std::string ptp(int fd, const std::string &logical) {
        const GxMapDesc &d = L.maps[fd];
        std::string e;
        if ((uint64_t)d.max_entries * d.value_size < (1ull << 31))
            e = "pt_phys_c<" + std::to_string(d.max_entries) + "u, " + std::to_string(d.value_size / 8) + "u>(" +
                hex(d.data) + ", " + logical + ", shard)";
        else
            e = "gxd::pt_phys(" + md(fd) + ", " + logical + ", shard)";
        if (bounds_) e = "(uint8_t *)" + ck("(uint64_t)" + e, 1, fd); /* the physical word within the shards */
        return e;
    }
    static std::string slot(int addr) { return "s" + std::to_string(addr >> 3); }

    /* Load hoisting inside basic blocks: a map / per-thread load moves above earlier instructions
     * that neither touch its registers nor may write the bytes it reads (stores through the same
     * base register to disjoint offsets, stores to another memory kind), so the dependent L2 round
     * trips of read-modify-write sequences overlap (P2 issues both per-thread loads back to back).
     * Never crosses a jump target, branch, helper call, atomic or exit. */
    static bool barrier(const GxInsn &h) {
        return h.op == GX_JA || h.op == GX_EXIT || h.op == GX_OP_NOP || (h.op >= GX_JEQ && h.op <= GX_JSET32) ||
               h.op >= GX_CALL_LOOKUP_ARRAY || h.op == GX_ATOM_STACK || h.op == GX_ATOM_MAP || h.op == GX_ATOM_PT;
    }
    static uint16_t reads(const GxInsn &h) {
        auto R = [](int r) { return (uint16_t)(1u << r); };
        const bool x = h.flags & GXF_X;
        switch (h.op) {
        case GX_MOV64: case GX_MOV32: return x ? R(h.src) : 0;
        case GX_MOVSX64: case GX_MOVSX32: return R(h.src);
        case GX_LDIMM: case GX_LDX_CTX: case GX_LDX_STACK: return 0;
        case GX_LDX_MAP: case GX_LDX_PT: return R(h.src);
        case GX_ST_STACK: return x ? R(h.src) : 0;
        case GX_ST_MAP: case GX_ST_PT: return R(h.dst) | (x ? R(h.src) : 0);
        default: return R(h.dst) | (x ? R(h.src) : 0);
        }
    }
    static uint16_t writes(const GxInsn &h) {
        switch (h.op) {
        case GX_ST_STACK: case GX_ST_MAP: case GX_ST_PT: return 0;
        default: return (uint16_t)(1u << h.dst);
        }
    }
    static std::vector<GxInsn> hoist_loads(const GxInsn *im, uint32_t n, const std::set<uint32_t> &targets) {
        std::vector<GxInsn> v(im, im + n);
        for (uint32_t j = 0; j < n; j++) {
            const GxInsn g = v[j];
            if ((g.op != GX_LDX_MAP && g.op != GX_LDX_PT) || targets.count(j)) continue;
            const uint16_t gd = (uint16_t)(1u << g.dst), gs = (uint16_t)(1u << g.src);
            const uint32_t gsz = 1u << (g.aux & 15);
            uint32_t p = j;
            while (p > 0) {
                const uint32_t i = p - 1;
                const GxInsn &h = v[i];
                if (barrier(h) || targets.count(i)) break;
                if ((reads(h) | writes(h)) & gd) break;
                if (writes(h) & gs) break;
                if (h.op == GX_ST_MAP || h.op == GX_ST_PT) {
                    const bool other_kind = (h.op == GX_ST_MAP) != (g.op == GX_LDX_MAP);
                    const uint32_t hsz = 1u << (h.aux & 15);
                    const bool disjoint = h.dst == g.src && (h.off + (int)hsz <= g.off || g.off + (int)gsz <= h.off);
                    if (!other_kind && !disjoint) break;
                }
                p = i;
            }
            if (p < j) {
                for (uint32_t k = j; k > p; k--) v[k] = v[k - 1];
                v[p] = g;
            }
        }
        return v;
    }

    static bool is_jcc(uint8_t op) { return op >= GX_JEQ && op <= GX_JSET32; }
    static bool is_lookup(uint8_t op) {
        return op == GX_CALL_LOOKUP_ARRAY || op == GX_CALL_LOOKUP_PT || op == GX_CALL_LOOKUP_HASH;
    }
    static bool ends_block(const GxInsn &g) {
        return g.op == GX_JA || g.op == GX_EXIT || g.op == GX_OP_NOP || is_jcc(g.op) ||
               (is_lookup(g.op) && (g.flags & (GXF_FETCH | GXF_W32)));
    }

    /* If-conversion: a conditional jump whose one or two arms are short runs of collective-free
     * instructions that meet again (`jcc L; B...; ja J; L: ...; J:` or `jcc J; B...; J:`) is
     * compiled as per-lane predicated code -- no ballot, no divergence, no min-PC round trip.
     * Each lane still executes exactly its own path, so the result is the scalar one.  (C4's
     * binary search: `jgt r2, r7, left; mov r8, r1; ja next; left: mov r9, r1; next:`.) */
    struct IfConv {
        uint32_t b0, b1, l0, l1, join;
    };
    std::map<uint32_t, IfConv> ifconv_;
    const GxInsn *im_ = nullptr;
    static bool simple(const GxInsn &g) {
        if (g.op == GX_JA || g.op == GX_EXIT || g.op == GX_OP_NOP || is_jcc(g.op)) return false;
        if (g.op >= GX_CALL_LOOKUP_ARRAY) return false; /* helpers (incl. GX_CALL_MEM_PREFETCH) */
        if (g.op == GX_ATOM_STACK || g.op == GX_ATOM_MAP || g.op == GX_ATOM_PT) return false;
        return true;
    }
    void find_ifconv(const GxInsn *im, uint32_t n, const std::map<uint32_t, int> &tcount) {
        ifconv_.clear();
        auto is_target = [&](uint32_t k) { return tcount.count(k) != 0; };
        for (uint32_t i = 0; i < n; i++) {
            if (!is_jcc(im[i].op)) continue;
            const uint32_t t = im[i].aux;
            if (t <= i + 1 || t > n || is_target(i + 1)) continue;
            uint32_t e = i + 1;
            while (e < n && e < t && simple(im[e]) && (e == i + 1 || !is_target(e)) && e - i <= 16) e++;
            if (e == t) { /* triangle: B = [i+1, t), join t */
                ifconv_[i] = {i + 1, t, t, t, t};
                continue;
            }
            if (e < n && im[e].op == GX_JA && e + 1 == t && tcount.at(t) == 1) {
                const uint32_t J = im[e].aux;
                if (J <= t || J > n) continue;
                uint32_t f = t;
                while (f < J && simple(im[f]) && (f == t || !is_target(f)) && f - t <= 16) f++;
                if (f == J) ifconv_[i] = {i + 1, e, t, J, J};
            }
        }
    }

    std::ostringstream *out_ = nullptr;
    bool dmode_ = false; /* emitting the min-PC (diverged) copy of a block */
    bool ifconv_on_ = true; /* GX_JIT_IFCONV=0: off */
    int hc_map_ = -1;    /* HASH map with the shared-memory key -> slot cache (GX_JIT_HASH_CACHE entries) */
    uint32_t hc_n_ = 0;
    bool ptc_ = false;   /* per-thread words through the register write-back cache (GX_JIT_PTCACHE=1; measured slower on C2) */
    int pkc_fd_ = -1;    /* the per-thread map held in the register key cache (GX_JIT_PTKC), or -1 */
    int stages_ = 4;     /* event-ring depth of this module (gx_jit_stages_for) */
    std::vector<const uint16_t *> nin_; /* per program: registers narrow on entry to each slot (verifier) */
    const uint16_t *cur_nin_ = nullptr;
    /* at a block start: re-state the registers the verifier proved below 2^32 there, so that the
     * compiler knows their upper halves are zero across loop back-edges and joins */
    void narrow_entry(uint32_t b) {
        if (!cur_nin_ || (getenv("GX_JIT_NARROW") && atoi(getenv("GX_JIT_NARROW")) == 0)) return;
        const uint16_t m = cur_nin_[b];
        for (int k = 0; k < 10; k++)
            if ((m >> k) & 1) (*out_) << "  " << R(k) << " = (uint64_t)(uint32_t)" << R(k) << ";\n";
    }
    bool bounds_ = false; /* GX_JIT_BOUNDS=1: every map access checked against its map (debug mode) */
    /* [lo, hi) of a map's device allocation (per-thread maps: the physical shard array) */
    void map_range(int fd, uint64_t &lo, uint64_t &hi) const {
        const GxMapDesc &d = L.maps[fd];
        lo = d.data;
        uint64_t bytes = 0;
        switch (d.type) {
        case 2: bytes = (uint64_t)d.max_entries * d.value_size; break;                  /* ARRAY */
        case 6: bytes = (uint64_t)d.max_entries * d.value_size * d.nshards; break;      /* PERTHREAD */
        case 1: bytes = ((uint64_t)d.cap_mask + 1 + 2) * 16; break;                      /* HASH keys + values */
        default: bytes = 0;
        }
        /* GX_JIT_BOUNDS=2: the checked ranges halved -- the checker's own self-test (accesses to the
         * upper halves of the maps must then be counted) */
        if (getenv("GX_JIT_BOUNDS") && atoi(getenv("GX_JIT_BOUNDS")) == 2) bytes /= 2;
        hi = lo + bytes;
    }
    /* a checked address expression (unchanged when the mode is off) */
    std::string ck(const std::string &addr, unsigned size, int fd) const {
        if (!bounds_) return addr;
        uint64_t lo = 0, hi = 0;
        if (fd >= 0) map_range(fd, lo, hi);
        if (fd < 0 || hi == lo)
            return "gx_chk_any((uint64_t)(" + addr + "), " + std::to_string(size) + "u)";
        return "gx_chk((uint64_t)(" + addr + "), " + std::to_string(size) + "u, " + hex(lo) + ", " + hex(hi) + ", " +
               "(unsigned long long *)" + hex(L.stats) + ")";
    }
    /* gx_chk_any: inside some map of the launch (helper arguments through map-value pointers) */
    void emit_chk_any() {
        o << "__device__ __forceinline__ uint64_t gx_chk_any(uint64_t a, uint32_t size) {\n";
        for (int m = 0; m < GX_MAX_MAPS; m++) {
            uint64_t lo, hi;
            if (!L.maps[m].data) continue;
            map_range(m, lo, hi);
            if (hi > lo) o << "  if (a >= " << hex(lo) << " && a < " << hex(hi) << ") return gx_chk(a, size, " << hex(lo) << ", "
                           << hex(hi) << ", (unsigned long long *)" << hex(L.stats) << ");\n";
        }
        o << "  return gx_chk(a, size, 0, 0, (unsigned long long *)" << hex(L.stats) << ");\n}\n";
    }
    /* the per-thread key cache's access forms: key from the value-start pointer, constant word */
    std::string pkc_key(const std::string &ptr) const {
        const GxMapDesc &d = L.maps[pkc_fd_];
        uint32_t lvs = 0;
        while ((1u << lvs) < d.value_size) lvs++;
        return "{ const uint32_t k_ = (uint32_t)(" + ptr + " - " + hex(d.data) + ") >> " + std::to_string(lvs) +
               "; if (k_ != pkc.key) ptkc_switch<" + std::to_string(d.max_entries) + "u, " + std::to_string(d.value_size / 8) +
               "u>(pkc, " + hex(d.data) + ", k_, shard); }";
    }
    /* picks the per-thread map for the key cache: every access to it is through a value-start pointer,
     * at most 4 words per value, no helper writes it (map update) or reads through a map-value
     * pointer (conservatively: no helper takes map-value pointers at all), the most accesses wins */
    void pick_pkc(const std::vector<const GxInsn *> &images, const std::vector<uint32_t> &sizes) {
        pkc_fd_ = -1;
        if (getenv("GX_JIT_PTKC") && atoi(getenv("GX_JIT_PTKC")) == 0) return;
        /* single-program launches only: in an attach-table launch the cached words stay live across
         * every program's code (C5: 4 % slower with the cache, C2: 14 % faster; profiles/r2_ptkc.md) */
        if (images.size() != 1 && !(getenv("GX_JIT_PTKC") && atoi(getenv("GX_JIT_PTKC")) == 2)) return;
        std::map<int, int> hits;
        std::set<int> bad;
        bool mapv_helper = false;
        for (size_t q = 0; q < images.size(); q++)
            for (uint32_t i = 0; i < sizes[q]; i++) {
                const GxInsn &g = images[q][i];
                int fd = -1;
                if (g.op == GX_LDX_PT) fd = (int)g.imm;
                else if (g.op == GX_ST_PT || g.op == GX_ATOM_PT) fd = g.aux >> 4;
                else if (g.op == GX_CALL_UPDATE_PT) bad.insert(g.aux);
                if (g.op >= GX_CALL_LOOKUP_ARRAY && g.op <= GX_CALL_RINGBUF_OUTPUT && (g.flags & (GXF_KEY_MAPV | GXF_VAL_MAPV)))
                    mapv_helper = true;
                if (fd < 0) continue;
                if (!(g.flags & GXF_PT_VSTART)) bad.insert(fd);
                hits[fd]++;
            }
        if (mapv_helper) return;
        int best = 0;
        for (auto &kv : hits) {
            const GxMapDesc &d = L.maps[kv.first];
            if (bad.count(kv.first) || d.value_size > 32 || (d.value_size & (d.value_size - 1)) ||
                (uint64_t)d.max_entries * d.value_size >= (1ull << 31))
                continue;
            if (kv.second > best) best = kv.second, pkc_fd_ = kv.first;
        }
    }
    void st(const std::string &x) { (*out_) << "  " << x << "\n"; }
    void me(const std::string &x) { (*out_) << "  { " << x << " }\n"; }
    std::string M() const { return dmode_ ? "exec" : "active"; }

    /* SIMT-convergent code.  prog<q>(ctx, active, ...) is called by all 32 lanes; `active` is the
     * group of lanes whose event runs program q, and the other lanes return at once.  Uniform copy
     * (labels U<pc>): the group runs every basic block together and branches with one ballot --
     * all taken / none taken jump straight on.  When the group splits, every lane records its next
     * block in `mypc` and enters the min-PC loop (DIV): the lanes at the lowest block id (`exec`)
     * run that block's diverged copy, and once the live lanes all wait at one block again they
     * re-enter the uniform copy there.  This is the interpreter's a3 scheme at basic-block
     * granularity, and it makes the lane group known at every helper call: the helpers' warp
     * collectives take `active` (uniform copy) or `exec` (diverged copy) as their mask.
     * prog<q><FULL = true> is the instance for a whole-warp group (the common case): `active` is
     * the constant full mask throughout its uniform copy -- it re-enters the uniform copy only when
     * all 32 lanes are live again -- so every uniform-copy collective compiles without the
     * runtime-mask convergence checks (REDUX.OR + BRA.DIV per collective, profiles/r1_ncu_c2_jit.md). */
    void program(int q, const GxInsn *im0, uint32_t n) {
        cur_nin_ = (size_t)q < nin_.size() ? nin_[q] : nullptr;
        std::set<uint32_t> targets, leaders{0};
        std::map<uint32_t, int> tcount;
        for (uint32_t i = 0; i < n; i++) {
            const GxInsn &g = im0[i];
            if (g.op == GX_JA || is_jcc(g.op)) targets.insert(g.aux), tcount[g.aux]++;
            if (is_lookup(g.op) && (g.flags & (GXF_FETCH | GXF_W32))) targets.insert((uint32_t)g.imm), tcount[(uint32_t)g.imm]++;
        }
        std::vector<GxInsn> sched = hoist_loads(im0, n, targets);
        const GxInsn *im = sched.data();
        im_ = im;
        if (ifconv_on_) find_ifconv(im, n, tcount);
        else ifconv_.clear();
        for (uint32_t t : targets) leaders.insert(t);
        for (uint32_t i = 0; i < n; i++)
            if (ends_block(im[i]) && i + 1 < n) leaders.insert(i + 1);
        std::set<int> slots;
        for (uint32_t i = 0; i < n; i++) {
            const GxInsn &g = im[i];
            switch (g.op) {
            case GX_LDX_STACK: case GX_ST_STACK: case GX_ATOM_STACK: slots.insert(g.off >> 3); break;
            case GX_CALL_LOOKUP_ARRAY: case GX_CALL_LOOKUP_PT: case GX_CALL_LOOKUP_HASH:
                if (!(g.flags & GXF_KEY_MAPV)) slots.insert(g.off >> 3);
                break;
            case GX_CALL_UPDATE_ARRAY: case GX_CALL_UPDATE_PT: case GX_CALL_UPDATE_HASH: {
                if (!(g.flags & GXF_KEY_MAPV)) slots.insert(g.off >> 3);
                if (!(g.flags & GXF_VAL_MAPV)) {
                    const uint32_t vs = L.maps[g.aux].value_size;
                    for (uint32_t w = 0; w < vs / 8; w++) slots.insert((int)((uint32_t)g.imm / 8 + w));
                }
                break;
            }
            case GX_CALL_RINGBUF_OUTPUT:
                if (!(g.flags & GXF_VAL_MAPV)) {
                    const uint32_t size = (uint32_t)g.imm;
                    for (uint32_t w = 0; w < (size + 7) / 8; w++) slots.insert((int)((uint16_t)g.off / 8 + w));
                }
                break;
            default: break;
            }
        }
        std::vector<std::pair<uint32_t, uint32_t>> blocks; /* [start, end) */
        for (auto it = leaders.begin(); it != leaders.end(); ++it) {
            auto nx = std::next(it);
            blocks.push_back({*it, nx == leaders.end() ? n : *nx});
        }
        o << "template <bool FULL>\n__device__ __forceinline__ void prog" << q
          << "(const Ctx &c, unsigned active, uint64_t &retv, const uint32_t shard, uint32_t *spriv, "
             "unsigned &c_herr, unsigned &c_drop, unsigned long long &c_rbb, unsigned &c_hfull, PtCache &ptc, GxPkc &pkc) {\n"
             "  const unsigned lane = threadIdx.x & 31;\n"
             "  if (FULL) active = GX_ALL;\n"
             "  if (!((active >> lane) & 1)) return;\n"
             "  uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0, r4 = 0, r5 = 0, r6 = 0, r7 = 0, r8 = 0, r9 = 0;\n"
             "  const uint64_t r10 = 512;\n  (void)r10; (void)spriv; (void)shard;\n";
        for (int s : slots) o << "  uint64_t s" << s << " = 0;\n";
        o << "  uint32_t mypc = 0;\n  (void)mypc;\n";
        std::ostringstream body, dbody;
        reent_.clear();
        out_ = &body;
        /* uniform copy */
        dmode_ = false;
        for (auto [b, e] : blocks) {
            body << " U" << b << ":\n";
            if (b) narrow_entry(b);
            for (uint32_t i = b; i < e; i++) insn(im[i], i);
            if (e > b && !ends_block(im[e - 1])) goto_next(e);
        }
        /* min-PC copy (emitted first: it records which pcs a lane's mypc can hold) */
        out_ = &dbody;
        dmode_ = true;
        for (auto [b, e] : blocks) {
            cur_block_ = b;
            dbody << "  case " << b << ": D" << b << ": {\n";
            if (b) narrow_entry(b);
            for (uint32_t i = b; i < e; i++) insn(im[i], i);
            if (e > b && !ends_block(im[e - 1])) goto_next(e);
            dbody << "  }\n";
        }
        dmode_ = false;
        out_ = &body;
        /* the re-entry / dispatch switches list only the pcs mypc can hold: the targets and
         * fall-throughs of conditional branches and backward jumps; forward unconditional
         * transitions in the min-PC copy go straight to the next block (same lanes, same exec), so
         * blocks reached only that way stay single-predecessor code the compiler can merge */
        reent_.insert(0);
        body << " DIV:\n  for (;;) {\n"
                "  const uint32_t pc_ = __reduce_min_sync(active, mypc);\n"
                "  if (pc_ == 0xFFFFFFFFu) return;\n"
                "  const unsigned exec = __ballot_sync(active, mypc == pc_);\n"
                "  const unsigned live = __ballot_sync(active, mypc != 0xFFFFFFFFu);\n"
                "  if (exec == live && (!FULL || live == GX_ALL)) {\n    if (mypc == 0xFFFFFFFFu) return;\n    active = FULL ? GX_ALL : live;\n    switch (pc_) {\n";
        for (auto [b, e] : blocks)
            if (reent_.count(b)) body << "    case " << b << ": goto U" << b << ";\n";
        body << "    default: return;\n    }\n  }\n  if (mypc != pc_) continue;\n  switch (pc_) {\n";
        std::string ds = dbody.str();
        /* drop the case labels no mypc value can select (their D<b> labels stay as goto targets) */
        for (auto [b, e] : blocks)
            if (!reent_.count(b)) {
                const std::string cl = "  case " + std::to_string(b) + ": D" + std::to_string(b) + ":";
                const size_t at = ds.find(cl);
                if (at != std::string::npos) ds.replace(at, cl.size(), "  D" + std::to_string(b) + ":");
            }
        body << ds;
        body << "  default: mypc = 0xFFFFFFFFu; continue;\n  }\n  }\n";
        o << body.str();
        o << "}\n\n";
    }

    std::set<uint32_t> reent_; /* pcs a lane's mypc can hold (min-PC re-entry points) */
    uint32_t cur_block_ = 0;
    void goto_next(uint32_t t) {
        if (dmode_) {
            if (t > cur_block_) {
                st("goto D" + std::to_string(t) + ";");
            } else {
                reent_.insert(t);
                st("mypc = " + std::to_string(t) + "u; continue;");
            }
        } else {
            st("goto U" + std::to_string(t) + ";");
        }
    }
    /* a conditional branch.  `uni`: the verifier's divergence analysis proved the condition warp-
     * uniform (GXF_UNIFORM: every lane that reaches the branch together takes it the same way), so
     * the uniform copy branches without a ballot.  GX_JIT_UNIFORM_CHECK=1 keeps the ballot and
     * counts any split of such a branch in the divergent_steps stat (tests: it must stay 0). */
    void branch(const std::string &cond, uint32_t t, uint32_t nx, bool uni = false) {
        if (dmode_) {
            reent_.insert(t);
            reent_.insert(nx);
            st("mypc = (" + cond + ") ? " + std::to_string(t) + "u : " + std::to_string(nx) + "u; continue;");
            return;
        }
        const bool check = getenv("GX_JIT_UNIFORM_CHECK") && atoi(getenv("GX_JIT_UNIFORM_CHECK")) != 0;
        if (uni && !check) {
            st("if (" + cond + ") goto U" + std::to_string(t) + "; goto U" + std::to_string(nx) + ";");
            return;
        }
        st("{ const bool t_ = " + cond + "; const unsigned tb_ = __ballot_sync(active, t_);");
        if (uni)
            st("  if (tb_ != active && tb_ != 0 && (threadIdx.x & 31) == (unsigned)(__ffs(active) - 1)) "
               "atomicAdd((unsigned long long *)" + hex(L.stats) + " + " + std::to_string(GXS_DIVERGENT) + ", 1ull);");
        st("  if (tb_ == active) goto U" + std::to_string(t) + "; if (tb_ == 0) goto U" + std::to_string(nx) + ";");
        reent_.insert(t);
        reent_.insert(nx);
        st("  mypc = t_ ? " + std::to_string(t) + "u : " + std::to_string(nx) + "u; goto DIV; }");
    }
    void exit_lanes(const std::string &val) {
        if (dmode_) st("retv = " + val + "; mypc = 0xFFFFFFFFu; continue;");
        else st("retv = " + val + "; return;");
    }

    std::string src_operand(const GxInsn &g, bool is64) {
        if (g.flags & GXF_X) return is64 ? R(g.src) : "(uint32_t)" + R(g.src);
        return is64 ? hex(g.imm) : hex((uint32_t)g.imm);
    }

    void insn(const GxInsn &g, uint32_t i) {
        const std::string d = R(g.dst), s = R(g.src);
        const std::string S64 = src_operand(g, true), S32 = src_operand(g, false);
        const bool sxf = g.flags & GXF_SX;
        const unsigned lg = g.aux & 15;
        auto ld_fix = [&](const std::string &v) {
            return sxf ? "sx(" + v + ", " + std::to_string(8u << lg) + ")" : v;
        };
        if (g.flags & GXF_NARROW) {
            /* the verifier proved operands and result below 2^32 on every path: the 32-bit operation,
             * zero-extended, is the 64-bit one (and the compiler keeps the upper halves known-zero) */
            const std::string a = "(uint32_t)" + d, b = (g.flags & GXF_X) ? "(uint32_t)" + s : std::to_string((uint32_t)g.imm) + "u";
            const char *opc = nullptr;
            switch (g.op) {
            case GX_ADD64: opc = "+"; break;
            case GX_SUB64: opc = "-"; break;
            case GX_MUL64: opc = "*"; break;
            case GX_OR64: opc = "|"; break;
            case GX_AND64: opc = "&"; break;
            case GX_XOR64: opc = "^"; break;
            case GX_RSH64: opc = ">>"; break;
            default: break;
            }
            if (g.op == GX_RSH64) {
                /* a 32-bit shift the compiler cannot re-widen (it otherwise folds a preceding narrow
                 * add into a 64-bit add + funnel shift to keep the carry bit it then masks off) */
                me("{ uint32_t t_; asm(\"shr.b32 %0, %1, %2;\" : \"=r\"(t_) : \"r\"(" + a + "), \"r\"((uint32_t)(" + b +
                   "))); " + d + " = (uint64_t)t_; }");
                return;
            }
            if (opc) {
                me(d + " = (uint64_t)(uint32_t)(" + a + " " + opc + " " + b + ");");
                return;
            }
            if (g.op == GX_MOV64) {
                me(d + " = (uint64_t)" + b + ";");
                return;
            }
            if (g.op == GX_DIV64 || g.op == GX_MOD64) {
                const bool dv = g.op == GX_DIV64;
                me("const uint32_t t = " + b + ", a_ = " + a + "; " + d + " = (uint64_t)(t ? a_ " + (dv ? "/" : "%") + " t : " +
                   (dv ? "0u" : "a_") + ");");
                return;
            }
        }
        switch (g.op) {
        case GX_ADD64: me(d + " += " + S64 + ";"); break;
        case GX_SUB64: me(d + " -= " + S64 + ";"); break;
        case GX_MUL64: me(d + " *= " + S64 + ";"); break;
        case GX_DIV64: me("const uint64_t t = " + S64 + "; " + d + " = t ? " + d + " / t : 0;"); break;
        case GX_MOD64: me("const uint64_t t = " + S64 + "; " + d + " = t ? " + d + " % t : " + d + ";"); break;
        case GX_SDIV64:
            me("const int64_t a = (int64_t)" + d + ", t = (int64_t)" + S64 + "; " + d +
               " = t == 0 ? 0 : (a == (int64_t)0x8000000000000000ll && t == -1) ? (uint64_t)a : (uint64_t)(a / t);");
            break;
        case GX_SMOD64:
            me("const int64_t a = (int64_t)" + d + ", t = (int64_t)" + S64 + "; " + d +
               " = t == 0 ? (uint64_t)a : t == -1 ? 0 : (uint64_t)(a % t);");
            break;
        case GX_OR64: me(d + " |= " + S64 + ";"); break;
        case GX_AND64: me(d + " &= " + S64 + ";"); break;
        case GX_XOR64: me(d + " ^= " + S64 + ";"); break;
        case GX_LSH64: me(d + " <<= (" + S64 + " & 63);"); break;
        case GX_RSH64: me(d + " >>= (" + S64 + " & 63);"); break;
        case GX_ARSH64: me(d + " = (uint64_t)((int64_t)" + d + " >> (" + S64 + " & 63));"); break;
        case GX_NEG64: me(d + " = 0 - " + d + ";"); break;
        case GX_MOV64: me(d + " = " + S64 + ";"); break;
        case GX_MOVSX64: me(d + " = sx(" + s + ", " + std::to_string(g.aux) + ");"); break;
        case GX_ADD32: me(d + " = (uint32_t)((uint32_t)" + d + " + " + S32 + ");"); break;
        case GX_SUB32: me(d + " = (uint32_t)((uint32_t)" + d + " - " + S32 + ");"); break;
        case GX_MUL32: me(d + " = (uint32_t)((uint32_t)" + d + " * " + S32 + ");"); break;
        case GX_DIV32: me("const uint32_t t = " + S32 + "; " + d + " = t ? (uint32_t)" + d + " / t : 0;"); break;
        case GX_MOD32: me("const uint32_t t = " + S32 + "; " + d + " = t ? (uint32_t)" + d + " % t : (uint32_t)" + d + ";"); break;
        case GX_SDIV32:
            me("const int32_t a = (int32_t)" + d + ", t = (int32_t)" + S32 + "; " + d +
               " = (uint32_t)(t == 0 ? 0 : (a == (int32_t)0x80000000 && t == -1) ? a : a / t);");
            break;
        case GX_SMOD32:
            me("const int32_t a = (int32_t)" + d + ", t = (int32_t)" + S32 + "; " + d +
               " = (uint32_t)(t == 0 ? a : t == -1 ? 0 : a % t);");
            break;
        case GX_OR32: me(d + " = (uint32_t)" + d + " | " + S32 + ";"); break;
        case GX_AND32: me(d + " = (uint32_t)" + d + " & " + S32 + ";"); break;
        case GX_XOR32: me(d + " = (uint32_t)" + d + " ^ " + S32 + ";"); break;
        case GX_LSH32: me(d + " = (uint32_t)((uint32_t)" + d + " << (" + S32 + " & 31));"); break;
        case GX_RSH32: me(d + " = (uint32_t)" + d + " >> (" + S32 + " & 31);"); break;
        case GX_ARSH32: me(d + " = (uint32_t)((int32_t)" + d + " >> (" + S32 + " & 31));"); break;
        case GX_NEG32: me(d + " = (uint32_t)(0u - (uint32_t)" + d + ");"); break;
        case GX_MOV32: me(d + " = (uint32_t)(" + S32 + ");"); break;
        case GX_MOVSX32: me(d + " = (uint32_t)sx(" + s + ", " + std::to_string(g.aux) + ");"); break;
        case GX_LE:
            if (g.aux < 64) me(d + " &= " + hex((1ull << g.aux) - 1) + ";");
            break;
        case GX_BE: me(d + " = bswap_w(" + d + ", " + std::to_string(g.aux) + ");"); break;
        case GX_LDIMM:
            if (g.flags & GXF_VAL_MAPV) me(d + " = " + hex(L.maps[g.aux].data + g.imm) + ";");
            else me(d + " = " + hex(g.imm) + ";");
            break;
        case GX_JA:
            goto_next(g.aux);
            break;
        case GX_EXIT: exit_lanes((g.flags & GXF_SX) ? hex(g.imm) : "r0"); break;
        case GX_OP_NOP:
            st("c_herr++;");
            exit_lanes("0");
            break;
        case GX_LDX_CTX: me(d + " = " + ld_fix("ctx_ld(c, " + std::to_string(g.off) + ", " + std::to_string(lg) + ")") + ";"); break;
        case GX_LDX_STACK:
            me(d + " = " + ld_fix("zx(" + slot(g.off) + " >> " + std::to_string(8 * (g.off & 7)) + ", " + std::to_string(lg) + ")") + ";");
            break;
        case GX_LDX_MAP: {
            const bool coh = L.maps[g.imm].coherent;
            me(d + " = " + ld_fix(std::string("gload<") + (coh ? "true" : "false") + ">(" +
                                  ck(s + " + (int64_t)" + std::to_string(g.off), 1u << lg, (int)g.imm) + ", " + std::to_string(lg) + ")") + ";");
            break;
        }
        case GX_LDX_PT:
            if ((int)g.imm == pkc_fd_)
                me(pkc_key(s) + " " + d + " = " + ld_fix("zx(pkc.v[" + std::to_string(g.off >> 3) + "] >> " +
                                                          std::to_string(8 * (g.off & 7)) + ", " + std::to_string(lg) + ")") + ";");
            else if (ptc_)
                me("const uint64_t la_ = " + s + " + (int64_t)" + std::to_string(g.off) + "; " + d + " = " +
                   ld_fix("ptc_ld(ptc, la_, " + ptp((int)g.imm, "la_") + ", " + std::to_string(lg) + ")") + ";");
            else
                me(d + " = " + ld_fix("ptload((uint64_t)" + ptp((int)g.imm, s + " + (int64_t)" + std::to_string(g.off)) + ", " +
                                      std::to_string(lg) + ")") + ";");
            break;
        case GX_ST_STACK: {
            const std::string v = (g.flags & GXF_X) ? s : hex(g.imm);
            me(slot(g.off) + " = word_set(" + slot(g.off) + ", " + std::to_string(g.off & 7) + ", " + std::to_string(lg) + ", " + v + ");");
            break;
        }
        case GX_ST_MAP: {
            const std::string v = (g.flags & GXF_X) ? s : hex(g.imm);
            me("gstore(" + ck(d + " + (int64_t)" + std::to_string(g.off), 1u << lg, -1) + ", " + std::to_string(lg) + ", " + v + ");");
            break;
        }
        case GX_ST_PT: {
            const std::string v = (g.flags & GXF_X) ? s : hex(g.imm);
            if ((g.aux >> 4) == pkc_fd_) {
                const std::string w = "pkc.v[" + std::to_string(g.off >> 3) + "]";
                me(pkc_key(d) + " " + w + " = word_set(" + w + ", " + std::to_string(g.off & 7) + ", " + std::to_string(lg) + ", " + v + ");");
            } else if (ptc_)
                me("const uint64_t la_ = " + d + " + (int64_t)" + std::to_string(g.off) + "; ptc_st(ptc, la_, " + ptp(g.aux >> 4, "la_") + ", " + std::to_string(lg) + ", " + v + ");");
            else
                me("ptstore((uint64_t)" + ptp(g.aux >> 4, d + " + (int64_t)" + std::to_string(g.off)) + ", " + std::to_string(lg) +
                   ", " + v + ");");
            break;
        }
        case GX_ATOM_STACK: case GX_ATOM_PT: case GX_ATOM_MAP: atomic(g); break;
        case GX_CALL_LOOKUP_ARRAY: case GX_CALL_LOOKUP_PT: case GX_CALL_LOOKUP_HASH: {
            const GxMapDesc &m = L.maps[g.aux];
            if (g.op == GX_CALL_LOOKUP_HASH) {
                std::string key = (g.flags & GXF_KEY_MAPV)
                                      ? (m.key_size == 4 ? "(uint64_t)*(const uint32_t *)" + ck("r2", 4, -1) : "*(const uint64_t *)" + ck("r2", 8, -1))
                                      : "(" + slot(g.off) + " >> " + std::to_string(8 * (g.off & 7)) + ")";
                if (m.key_size == 4) key = "(" + key + " & 0xFFFFFFFFull)";
                if ((int)g.aux == hc_map_)
                    st("{ const uint64_t k_ = " + key + "; r0 = (uint64_t)hash_lookup_cached<" + std::to_string(hc_n_) + "u>(" +
                       md(g.aux) + ", k_, " + M() + ", gx_hc); }");
                else
                    st("{ const uint64_t k_ = " + key + "; r0 = (uint64_t)gxd::hash_lookup_coop(" + md(g.aux) + ", k_, true, " +
                       M() + "); }");
            } else {
                const std::string key = (g.flags & GXF_KEY_MAPV)
                                            ? "*(const uint32_t *)" + ck("r2", 4, -1)
                                            : "(uint32_t)(" + slot(g.off) + " >> " + std::to_string(8 * (g.off & 7)) + ")";
                if (g.flags & GXF_SX) /* key below max_entries on every path (verifier): never NULL */
                    me("const uint32_t k = " + key + "; r0 = " + hex(m.data) + " + (uint64_t)k * " + std::to_string(m.value_size) + "u;");
                else
                    me("const uint32_t k = " + key + "; r0 = k < " + std::to_string(m.max_entries) + "u ? " + hex(m.data) +
                       " + (uint64_t)k * " + std::to_string(m.value_size) + "u : 0;");
            }
            if (g.flags & GXF_FETCH) branch("r0 == 0", (uint32_t)g.imm, i + 1, (g.flags & GXF_UNIFORM) != 0);
            if (g.flags & GXF_W32) branch("r0 != 0", (uint32_t)g.imm, i + 1, (g.flags & GXF_UNIFORM) != 0);
            break;
        }
        case GX_CALL_UPDATE_ARRAY: case GX_CALL_UPDATE_PT: {
            const GxMapDesc &m = L.maps[g.aux];
            const std::string key = (g.flags & GXF_KEY_MAPV)
                                        ? "*(const uint32_t *)" + ck("r2", 4, -1)
                                        : "(uint32_t)(" + slot(g.off) + " >> " + std::to_string(8 * (g.off & 7)) + ")";
            std::ostringstream b;
            /* ARRAY: lanes writing the same key keep the sequential result -- the group's last lane's
             * value (one copy per key); the return code depends on the key and flags only */
            b << "const uint32_t k = " << key << "; int64_t rc = 0;";
            if (g.op == GX_CALL_UPDATE_ARRAY)
                b << " const unsigned kg_ = __match_any_sync(" << M() << ", k) & __ballot_sync(" << M() << ", r4 == 0 || r4 == 2);";
            b << " if (r4 > 2) rc = -22; else if (k >= " << m.max_entries << "u) rc = -7; else if (r4 == 1) rc = -17; else";
            b << (g.op == GX_CALL_UPDATE_ARRAY ? " if ((int)lane == 31 - __clz(kg_)) {" : " {");
            for (uint32_t w = 0; w < m.value_size / 8; w++) {
                const std::string v = (g.flags & GXF_VAL_MAPV) ? "((const uint64_t *)" + ck("r3", 8, -1) + ")[" + std::to_string(w) + "]"
                                                               : "s" + std::to_string((uint32_t)g.imm / 8 + w);
                const std::string logical = hex(m.data) + " + (uint64_t)k * " + std::to_string(m.value_size) + "u + " +
                                            std::to_string(8 * w);
                if (g.op == GX_CALL_UPDATE_ARRAY) b << " *(uint64_t *)(" << logical << ") = " << v << ";";
                else if (ptc_)
                    b << " { const uint64_t la_ = " << logical << "; ptc_st(ptc, la_, " << ptp(g.aux, "la_") << ", 3, " << v << "); }";
                else b << " *(uint64_t *)" << ptp(g.aux, logical) << " = " << v << ";";
            }
            b << " } if (rc) c_herr++; r0 = (uint64_t)rc;";
            me(b.str());
            break;
        }
        case GX_CALL_UPDATE_HASH: {
            const GxMapDesc &m = L.maps[g.aux];
            std::string key = (g.flags & GXF_KEY_MAPV)
                                  ? (m.key_size == 4 ? "(uint64_t)*(const uint32_t *)" + ck("r2", 4, -1) : "*(const uint64_t *)" + ck("r2", 8, -1))
                                  : "(" + slot(g.off) + " >> " + std::to_string(8 * (g.off & 7)) + ")";
            if (m.key_size == 4) key = "(" + key + " & 0xFFFFFFFFull)";
            const std::string v = (g.flags & GXF_VAL_MAPV) ? "*(const uint64_t *)" + ck("r3", 8, -1) : "s" + std::to_string((uint32_t)g.imm / 8);
            st("{ const uint64_t k_ = " + key + ", v_ = " + v + ";");
            st("  const int64_t rc = gxd::hash_update_coop(" + md(g.aux) + ", k_, v_, r4, true, " + M() + ");");
            st("  if (rc) c_herr++; if (rc == -7) c_hfull++; r0 = (uint64_t)rc; }");
            break;
        }
        case GX_CALL_PREFETCH_L2:
            st("{ const int64_t rc_ = gxd::l2_prefetch(" + md(g.aux) + ", r2, r3); r0 = (uint64_t)rc_; if (rc_) c_herr++; }");
            break;
        case GX_CALL_MEM_PREFETCH:
            st("{ const int64_t rc_ = gxd::pfq_request_coop(" + md(g.aux) + ", r2, r3, true, " + M() +
               ", c_drop); r0 = (uint64_t)rc_; if (rc_) c_herr++; }");
            break;
        case GX_CALL_RINGBUF_OUTPUT: {
            const uint32_t size = (uint32_t)g.imm, flags = (uint32_t)(g.imm >> 32);
            if (flags > 2) {
                me("r0 = (uint64_t)(int64_t)-22; c_herr++;");
                break;
            }
            std::ostringstream b;
            b << "{ ";
            if (g.flags & GXF_VAL_MAPV) b << "const uint64_t *w = (const uint64_t *)" << ck("r2", 8, -1) << ";";
            else {
                b << "const uint64_t w[" << (size + 7) / 8 << "] = {";
                for (uint32_t k = 0; k < (size + 7) / 8; k++) b << (k ? ", " : "") << "s" << ((uint16_t)g.off / 8 + k);
                b << "};";
            }
            b << " const int64_t rc = group_ringbuf(" << M() << ", " << md(g.aux) << ", w, " << size << "u, c_drop, c_rbb);"
              << " r0 = (uint64_t)rc; if (rc) c_herr++; }";
            st(b.str());
            break;
        }
        default:
            if (is_jcc(g.op)) {
                const bool is32 = g.op >= GX_JEQ32;
                const int cop = is32 ? g.op - (GX_JEQ32 - GX_JEQ) : g.op;
                std::string a = is32 ? "(uint32_t)" + d : d;
                std::string b = is32 ? S32 : S64;
                std::string sa = is32 ? "(int32_t)" + d : "(int64_t)" + d;
                std::string sb = is32 ? "(int32_t)(" + S32 + ")" : "(int64_t)(" + S64 + ")";
                std::string c;
                switch (cop) {
                case GX_JEQ: c = a + " == " + b; break;
                case GX_JNE: c = a + " != " + b; break;
                case GX_JGT: c = a + " > " + b; break;
                case GX_JGE: c = a + " >= " + b; break;
                case GX_JLT: c = a + " < " + b; break;
                case GX_JLE: c = a + " <= " + b; break;
                case GX_JSGT: c = sa + " > " + sb; break;
                case GX_JSGE: c = sa + " >= " + sb; break;
                case GX_JSLT: c = sa + " < " + sb; break;
                case GX_JSLE: c = sa + " <= " + sb; break;
                default: c = "(" + a + " & " + b + ") != 0"; break;
                }
                auto ic = ifconv_.find(i);
                if (ic != ifconv_.end()) {
                    const IfConv &v = ic->second;
                    st("{ const bool t_ = " + c + ";");
                    if (v.b1 > v.b0) {
                        st("if (!t_) {");
                        for (uint32_t k = v.b0; k < v.b1; k++) insn(im_[k], k);
                        st("}");
                    }
                    if (v.l1 > v.l0) {
                        st("if (t_) {");
                        for (uint32_t k = v.l0; k < v.l1; k++) insn(im_[k], k);
                        st("}");
                    }
                    goto_next(v.join);
                    st("}");
                } else {
                    branch(c, g.aux, i + 1, (g.flags & GXF_UNIFORM) != 0);
                }
            } else {
                st("c_herr++;");
                exit_lanes("0");
            }
        }
    }

    void atomic(const GxInsn &g) {
        const uint32_t op = (uint32_t)(g.imm & 0xFF);
        const bool w32 = (g.aux & 15) == 2, fetch = op & 1, kop = g.flags & GXF_PRIV;
        const std::string v = kop ? hex((uint64_t)(int64_t)(int32_t)(g.imm >> 32)) : R(g.src);
        const std::string ret = op == 0xF1 ? "r0" : R(g.src);
        if (g.op == GX_ATOM_STACK) {
            std::string e = "rmw_word(" + slot(g.off) + ", " + std::to_string(g.off & 7) + ", " + (w32 ? "true" : "false") +
                            ", " + std::to_string(op) + "u, " + v + ", r0)";
            me(fetch ? "const uint64_t old = " + e + "; " + ret + " = old;" : "(void)" + e + ";");
            return;
        }
        const int fd = g.aux >> 4;
        const std::string addr = g.op == GX_ATOM_MAP ? ck(R(g.dst) + " + (int64_t)" + std::to_string(g.off), w32 ? 4u : 8u, fd)
                                                     : R(g.dst) + " + (int64_t)" + std::to_string(g.off);
        if (g.op == GX_ATOM_PT && fd == pkc_fd_) {
            std::string e = "rmw_word(pkc.v[" + std::to_string(g.off >> 3) + "], " + std::to_string(g.off & 7) + ", " +
                            (w32 ? "true" : "false") + ", " + std::to_string(op) + "u, " + v + ", r0)";
            me(pkc_key(R(g.dst)) + " " + (fetch ? "const uint64_t old = " + e + "; " + ret + " = old;" : "(void)" + e + ";"));
            return;
        }
        if (g.op == GX_ATOM_PT) {
            std::string e = ptc_ ? "ptc_rmw(ptc, " + addr + ", " + ptp(fd, addr) + ", " +
                                       (w32 ? "true" : "false") + ", " + std::to_string(op) + "u, " + v + ", r0)"
                                 : "rmw_global_private((uint64_t)" + ptp(fd, addr) + ", " +
                                       (w32 ? "true" : "false") + ", " + std::to_string(op) + "u, " + v + ", r0)";
            me(fetch ? "const uint64_t old = " + e + "; " + ret + " = old;" : "(void)" + e + ";");
            return;
        }
        /* XCHG / CMPXCHG on shared map values: lanes grouped by address, the group's sequential
         * result in lane order (gx_jit_rt.cuh group_xchg / group_cmpxchg) */
        if (op == 0xE1) {
            st("{ const uint64_t res_ = group_xchg<" + std::string(w32 ? "true" : "false") + ">(" + M() + ", " + addr + ", " + v +
               "); " + R(g.src) + " = res_; }");
            return;
        }
        if (op == 0xF1) {
            st("{ const uint64_t res_ = group_cmpxchg<" + std::string(w32 ? "true" : "false") + ">(" + M() + ", " + addr +
               ", r0, " + v + "); r0 = res_; }");
            return;
        }
        const GxMapDesc &m = L.maps[fd];
        if (m.priv_off != 0xFFFFFFFFu && !fetch && (op & 0xF0) == 0 && !w32) {
            const uint32_t nw = m.max_entries * m.value_size / 8;
            st("group_priv_add(" + M() + ", spriv + " + std::to_string(m.priv_off / 4) + ", spriv + " + std::to_string(m.priv_off / 4 + nw) +
               ", (uint32_t)((" + addr + " - " + hex(m.data) + ") >> 3), " + v + ");");
            return;
        }
        if (kop && (op & 0xF0) == 0) {
            const std::string e = std::string("group_add_const<") + (w32 ? "true" : "false") + ", " + (fetch ? "true" : "false") +
                                  ">(" + M() + ", " + addr + ", " + (w32 ? hex((uint32_t)(g.imm >> 32)) : v) + ")";
            if (fetch) st("{ const uint64_t res_ = " + e + "; " + R(g.src) + " = res_; }");
            else st("(void)" + e + ";");
            return;
        }
        std::string e = "group_atomic<" + std::to_string(op & 0xF0) + "u, " + (w32 ? "true" : "false") + ", " +
                        (fetch ? "true" : "false") + ">(" + M() + ", " + addr + ", " + v + ")";
        if (fetch) st("{ const uint64_t res_ = " + e + "; " + R(g.src) + " = res_; }");
        else st("(void)" + e + ";");
    }

    void kernel(const std::vector<const GxInsn *> &images, const std::vector<uint32_t> &sizes, int B, unsigned vmask) {
        int U = 2;
        if (const char *e = getenv("GX_JIT_UNROLL")) U = std::max(1, std::min(8, atoi(e)));
        /* GX_JIT_MINB: min resident blocks per SM in __launch_bounds__ (default 1: up to 64 registers
         * at 1024 threads -- without it NVRTC caps at 32 and spills; measured faster on every config);
         * GX_JIT_PUNROLL=0: one inlined copy of the programs (records rotate through the load buffer) */
        const int minb = getenv("GX_JIT_MINB") ? atoi(getenv("GX_JIT_MINB")) : 1;
        const bool punroll = !getenv("GX_JIT_PUNROLL") || atoi(getenv("GX_JIT_PUNROLL")) != 0;
        ptc_ = getenv("GX_JIT_PTCACHE") && atoi(getenv("GX_JIT_PTCACHE")) != 0;
        bounds_ = getenv("GX_JIT_BOUNDS") && atoi(getenv("GX_JIT_BOUNDS")) != 0;
        ifconv_on_ = !getenv("GX_JIT_IFCONV") || atoi(getenv("GX_JIT_IFCONV")) != 0;
        if (const char *e = getenv("GX_JIT_WAIT_HINT")) o << "#define GX_WAIT_HINT " << atoi(e) << "\n";
        if (const char *e = getenv("GX_JIT_HASH_L1PROBE")) o << "#define GX_HASH_L1PROBE " << atoi(e) << "\n";
        if (const char *e = getenv("GX_JIT_PIN")) o << "#define GX_PIN " << atoi(e) << "\n";
        if (const char *e = getenv("GX_JIT_ATOM_MIXED")) o << "#define GX_ATOM_MIXED " << atoi(e) << "\n";
        if (getenv("GX_JIT_COLD_INLINE")) o << "#define GX_COLD_INLINE 1\n";
        if (const char *e = getenv("GX_JIT_LOCKSTEP")) o << "#define GX_HASH_LOCKSTEP " << atoi(e) << "\n";
        if (const char *e = getenv("GX_JIT_PROBE_W")) o << "#define GX_HASH_PROBE_W " << atoi(e) << "\n";
        if (const char *e = getenv("GX_JIT_PT_HINT")) o << "#define GX_PT_HINT " << atoi(e) << "\n";
        o << "#include \"gx_jit_rt.cuh\"\nusing namespace gxj;\n\n";
        pick_pkc(images, sizes);
        if (bounds_) {
            pkc_fd_ = -1;  /* every per-thread access through the checked physical address */
            emit_chk_any();
        }
        if (pkc_fd_ >= 0)
            o << "typedef PtKc<" << L.maps[pkc_fd_].max_entries << "u, " << L.maps[pkc_fd_].value_size / 8 << "u> GxPkc;\n";
        else
            o << "typedef PtKc<1u, 1u> GxPkc;\n";
        /* the first HASH map with 8-byte values that a program looks up gets the per-block key -> slot
         * cache (GX_JIT_HASH_CACHE entries, a power of two; 0 = off) */
        {
            uint32_t ncache = 2048;
            if (const char *e = getenv("GX_JIT_HASH_CACHE")) ncache = (uint32_t)atoi(e);
            if (ncache & (ncache - 1)) ncache = 0;
            hc_map_ = -1;
            /* static shared memory stays under the 48-KiB static limit: the privatised accumulators
             * (spriv), the stats, the ring barriers and the key cache (16 B per entry) share it */
            const uint32_t fixed = 4u * ((L.priv_bytes + 3) / 4) + 1024u;
            const uint32_t room = fixed < 48u * 1024u ? (48u * 1024u - fixed) / 16u : 0u;
            hc_n_ = std::min<uint32_t>(ncache, 2048);
            while (hc_n_ && hc_n_ > room) hc_n_ >>= 1;
            if (hc_n_ < 64) hc_n_ = 0; /* too small to pay for itself */
            for (size_t q = 0; q < images.size() && hc_n_ && hc_map_ < 0; q++)
                for (uint32_t i = 0; i < sizes[q]; i++)
                    if (images[q][i].op == GX_CALL_LOOKUP_HASH && L.maps[images[q][i].aux].value_size == 8) {
                        hc_map_ = images[q][i].aux;
                        break;
                    }
            if (hc_map_ >= 0) o << "__shared__ __align__(16) unsigned long long gx_hc[" << 2 * hc_n_ << "];\n\n";
        }
        for (size_t q = 0; q < images.size(); q++) program((int)q, images[q], sizes[q]);
        /* two launch bodies: event ingest through the block-wide TMA ring (large batches of light
         * programs) and through per-lane register loads (small batches, ALU-heavy programs) --
         * the runtime picks per launch (gx_runtime.cpp launch_cfg) */
        /* only the instances `vmask` asks for (GX_JIT_V_*): a module per launch variant keeps NVRTC
         * time proportional to what runs -- each instance inlines every program U times */
        const int S = gx_jit_stages_for(images, sizes);
        stages_ = S >= 2 ? S : 3;
        if (vmask & (GX_JIT_V_RING | GX_JIT_V_RING_R)) body("gx_body_ring", stages_, B, U, punroll, images);
        if (vmask & (GX_JIT_V_REG | GX_JIT_V_REG_R)) body("gx_body_reg", 0, B, U, punroll, images);
        const std::string lb = "__launch_bounds__(" + std::to_string(B) + (minb > 0 ? ", " + std::to_string(minb) : std::string()) + ")";
        const char *args = "(const uint4 *__restrict__ ev, uint64_t n, uint64_t *__restrict__ ret, unsigned long long *__restrict__ gstats)";
        for (int k = 0; k < 4; k++)
            if (vmask & (1u << k))
                o << "extern \"C\" __global__ void " << lb << " " << gx_jit_kernel_name(k) << args << " {\n  "
                  << (k < 2 ? "gx_body_ring" : "gx_body_reg") << (k & 1 ? "<true>" : "<false>") << "(ev, n, ret, gstats);\n}\n";
    }

    /* f4: the program as __device__ hooks a user kernel calls inline -- the paper's
     * "trampolines ... at GPU kernel entry, selected memory instructions" made at
     * compile time.  The hooking lanes pass their group explicitly (a ballot taken where the warp
     * is converged): the helpers' warp collectives need the exact set of lanes that reach them.
     * The ctx is built in registers from the call site; per-thread shards are keyed by the
     * hardware slot (SM, warp slot, lane), unique among resident threads. */
    uint32_t pt_shards_min() const {
        uint32_t v = ~0u;
        for (int m = 0; m < GX_MAX_MAPS; m++)
            if (L.maps[m].type == 6 /* PERTHREAD_ARRAY */ && L.maps[m].nshards) v = std::min(v, L.maps[m].nshards);
        return v == ~0u ? 1u << 30 : v;
    }
    void instrument(const GxInsn *image, uint32_t n, const std::string &user) {
        ptc_ = false;
        ifconv_on_ = !getenv("GX_JIT_IFCONV") || atoi(getenv("GX_JIT_IFCONV")) != 0;
        o << "#include \"gx_jit_rt.cuh\"\nusing namespace gxj;\ntypedef PtKc<1u, 1u> GxPkc;\n\n";
        pkc_fd_ = -1; /* no flush point in a user kernel */
        program(0, image, n);
        o << "/* rec (optional): receives the 32-B event record the program ran on (hook logs) */\n"
             "__device__ __forceinline__ uint64_t gx_hook_event(unsigned group, uint64_t addr, uint32_t hook, uint32_t size,\n"
             "                                                  uint32_t *rec = nullptr) {\n"
             "  uint32_t smid, wslot;\n"
             "  asm volatile(\"mov.u32 %0, %%smid;\" : \"=r\"(smid));\n"
             "  asm volatile(\"mov.u32 %0, %%warpid;\" : \"=r\"(wslot));\n"
             "  uint64_t ts;\n"
             "  asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(ts));\n"
             "  const uint32_t lane = threadIdx.x & 31;\n"
             "  const uint32_t blk = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);\n"
             "  Ctx c;\n"
             "  c.w[0] = (uint32_t)addr; c.w[1] = (uint32_t)(addr >> 32); c.w[2] = (uint32_t)ts; c.w[3] = (uint32_t)(ts >> 32);\n"
             "  c.w[4] = hook; c.w[5] = blk; c.w[6] = (smid & 0xFFFF) | ((wslot & 63) << 16) | (lane << 24); c.w[7] = size;\n"
             "  if (rec) { for (int k = 0; k < 8; k++) rec[k] = c.w[k]; }\n"
             "  /* unique among resident threads; the shards are sized from %nsmid (gx_open), the modulo\n"
             "   * only keeps a device that reports more SM ids than that inside the map */\n"
             "  const uint32_t shard = ((smid * 64 + (wslot & 63)) * 32 + lane) % " << pt_shards_min() << "u;\n"
             "  uint64_t retv = 0;\n"
             "  unsigned herr = 0, drop = 0, hfull = 0;\n"
             "  unsigned long long rbb = 0;\n"
             "  PtCache ptc;\n  GxPkc pkc;\n"
             "  if (group == GX_ALL) prog0<true>(c, GX_ALL, retv, shard, nullptr, herr, drop, rbb, hfull, ptc, pkc);\n"
             "  else prog0<false>(c, group, retv, shard, nullptr, herr, drop, rbb, hfull, ptc, pkc);\n"
             "  unsigned long long *st = (unsigned long long *)" << hex(L.stats) << ";\n"
             "  if (herr) atomicAdd(&st[" << GXS_HERR << "], herr);\n"
             "  if (drop) atomicAdd(&st[" << GXS_RB_DROPS << "], drop);\n"
             "  if (rbb) atomicAdd(&st[" << GXS_RB_BYTES << "], rbb);\n"
             "  if (hfull) atomicAdd(&st[" << GXS_HFULL << "], hfull);\n"
             "  return retv;\n"
             "}\n"
             "/* memory-access hook (gdev_mem_ops.access, PAPER.md:225-230): returns the program's R0 */\n"
             "__device__ __forceinline__ uint64_t gx_hook_access(unsigned group, const void *addr, uint32_t size, bool is_write) {\n"
             "  return gx_hook_event(group, (uint64_t)addr, " << 0 << "u | (is_write ? 0x10000u : 0u), size);\n"
             "}\n"
             "/* block-entry hook (gdev_sched_ops.enter, PAPER.md:260-262) */\n"
             "__device__ __forceinline__ uint64_t gx_hook_block_enter(unsigned group, uint64_t unit, uint32_t cost) {\n"
             "  return gx_hook_event(group, unit, 1u, cost);\n"
             "}\n"
             "/* memory-fence hook (gdev_mem_ops.fence, PAPER.md:225-230): addr = the caller's scope id */\n"
             "__device__ __forceinline__ uint64_t gx_hook_fence(unsigned group, uint64_t scope) {\n"
             "  return gx_hook_event(group, scope, 3u, 0u);\n"
             "}\n"
             "/* device-function entry / return hooks (gdev_sched_ops.probe / .retprobe, PAPER.md:265-267):\n"
             " * addr = the caller's function id, size = the low 32 bits of the return value (retprobe) */\n"
             "__device__ __forceinline__ uint64_t gx_hook_probe(unsigned group, uint64_t fn) {\n"
             "  return gx_hook_event(group, fn, 6u, 0u);\n"
             "}\n"
             "__device__ __forceinline__ uint64_t gx_hook_retprobe(unsigned group, uint64_t fn, uint32_t retval) {\n"
             "  return gx_hook_event(group, fn, 7u, retval);\n"
             "}\n\n#line 1 \"user.cu\"\n"
          << user << "\n";
    }

    /* one launch body (template on WANT_RET: write per-event R0) with S-stage ring ingest (S >= 2)
     * or register ingest (S == 0) */
    void body(const std::string &fname, int S, int B, int U, bool punroll, const std::vector<const GxInsn *> &images) {
        const uint32_t priv_words = (L.priv_bytes + 3) / 4;
        bool two_level = S < 2; /* record loop nested in a batch loop (register ingest, ring claims) */
        o << "template <bool WANT_RET>\n__device__ __forceinline__ void " << fname << "(const uint4 *__restrict__ ev, "
             "uint64_t n, uint64_t *__restrict__ ret, unsigned long long *__restrict__ gstats) {\n";
        o << "  __shared__ uint32_t spriv[" << (priv_words ? priv_words : 1) << "];\n"
             "  __shared__ unsigned long long sstats[8];\n"
             "  for (uint32_t k = threadIdx.x; k < " << priv_words << "u; k += " << B << ") spriv[k] = 0;\n"
          << (hc_map_ >= 0 ? "  for (uint32_t k = threadIdx.x; k < " + std::to_string(hc_n_) + "u; k += " + std::to_string(B) +
                                 ") gx_hc[2 * k] = GX_HASH_EMPTY;\n" : std::string()) <<
             "  if (threadIdx.x < 8) sstats[threadIdx.x] = 0;\n"
             "  __syncthreads();\n"
             "  const uint32_t lane = threadIdx.x & 31;\n"
             "  const uint32_t shard = blockIdx.x * " << B << " + threadIdx.x;\n"
             "  /* per-thread event counts in 32 bits (register pressure), widened for the warp reduction */\n"
             "  unsigned c_run = 0, c_skip = 0, c_herr = 0, c_drop = 0, c_hfull = 0;\n"
             "  unsigned long long c_rbb = 0;\n"
             "  PtCache ptc;\n  GxPkc pkc;\n"
             "  const uint64_t nrec = (n + 31) >> 5, nfull = n >> 5; /* records, whole records */\n"
             "  const uint64_t nwarps = (uint64_t)gridDim.x * " << B / 32 << ";\n"
             "  const uint64_t pol = evict_first_policy();\n"
             "  /* PDL (gx_run_batch_ex GX_RUN_OVERLAP): let the next batch's grid be scheduled; no-ops\n"
             "   * for a plain launch */\n"
             "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n";
        const char *pdl_wait = "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\"); /* maps after the previous grid */\n";
        if (S >= 2 && gx_jit_stage_mode() == 3) {
            /* a1 through a block-wide ring of S stages, each one contiguous chunk of W = B/32 warp
             * records (W KiB) brought in by ONE 1-D TMA bulk copy and signalled on the stage's
             * mbarrier.  The block's chunk c covers records (c * gridDim + blockIdx) * W + w.  Warps
             * claim records in order from a shared counter (dynamic, so uneven per-record cost does
             * not stall the ring); the warp that reads a stage's last record (shared counter)
             * refills it with chunk c + S -- no producer warp, no empty-barrier waits. */
            const int W = B / 32;
            /* ONE record per claim.  Stage phases are told apart by parity only, so a warp must never
             * claim a record S or more chunks past a stage that has not been refilled: with one record
             * per claim the W warps can at most cover one whole unloaded chunk (and then all wait on
             * it); claiming 2 records let half the warps block a chunk while the rest ran two chunks
             * ahead onto a stale phase (measured: corrupted ring, launch failure at 2^24 events). */
            two_level = true;
            /* stage release: atom (default: a shared counter, the last reader refills the stage) or
             * GX_JIT_RING_RELEASE=mbar (every warp arrives on the stage's "empty" mbarrier -- no
             * returning atomic; the first claimant of chunk c waits for chunk c-1 to be read and
             * issues chunk c+S-1).  Measured equal on C2/C3/C5/C6 (profiles/r1_jit_variants.md). */
            const bool mbar_rel = getenv("GX_JIT_RING_RELEASE") && strcmp(getenv("GX_JIT_RING_RELEASE"), "mbar") == 0;
            /* record assignment: static (default: warp w runs record w of every chunk; no claim atomic,
             * stage/phase advanced incrementally) or GX_JIT_RING_CLAIM=dynamic (claimed from a shared
             * counter, so one slow warp does not hold back the refills).  Static measured faster on
             * C2/C3/C5/C6 (profiles/r1_jit_variants.md §7); ALU-heavy loop programs take the
             * register-ingest body anyway. */
            const bool stat = !getenv("GX_JIT_RING_CLAIM") || strcmp(getenv("GX_JIT_RING_CLAIM"), "dynamic") != 0;
            /* static assignment may give each warp P consecutive records of a (W x P)-record stage
             * (GX_JIT_RING_RPW): bigger bulk copies, the same number of streams per SM */
            const int P = stat ? gx_jit_ring_rpw(stages_) : 1;
            const int CW = W * P; /* records per chunk (one stage) */
            o << "  extern __shared__ __align__(128) uint4 gx_ring[];\n"
                 "  __shared__ __align__(8) uint64_t gx_full[" << S << "];\n"
                 "  __shared__ uint32_t gx_used[" << S << "];\n"
                 "  __shared__ uint32_t gx_next;\n"
                 "  __shared__ __align__(8) uint64_t gx_empty[" << S << "];\n"
                 "  const uint32_t empty_s = pin32((uint32_t)__cvta_generic_to_shared(gx_empty));\n"
                 "  const uint32_t ring_s = pin32((uint32_t)__cvta_generic_to_shared(gx_ring));\n"
                 "  const uint32_t full_s = pin32((uint32_t)__cvta_generic_to_shared(gx_full));\n"
                 "  const uint32_t wid = threadIdx.x >> 5;\n"
                 "  const uint64_t gstride = (uint64_t)gridDim.x * " << CW << ";\n"
                 "  auto stage_issue = [&](uint32_t st, uint64_t r0_) {\n"
                 "    if (r0_ >= nrec) return;\n"
                 "    const uint64_t left_ = n - r0_ * 32;\n"
                 "    const uint32_t bytes_ = left_ >= " << 32 * CW << "ull ? " << 1024 * CW << "u : (uint32_t)left_ * 32u;\n"
                 "    bulk_load(ring_s + st * " << 1024 * CW << "u, ev + r0_ * 64, bytes_, full_s + st * 8u, pol);\n"
                 "  };\n"
                 "  if (threadIdx.x == 0) {\n"
                 "    for (int k = 0; k < " << S << "; k++) { mbar_init(full_s + k * 8u, 1); mbar_init(empty_s + k * 8u, " << W << "); gx_used[k] = 0; }\n"
                 "    gx_next = 0;\n"
                 "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
                 "    for (int k = 0; k < " << S << "; k++) stage_issue(k, k * gstride + (uint64_t)blockIdx.x * " << CW << ");\n"
                 "  }\n"
                 "  __syncthreads();\n"
              << pdl_wait <<
                 "  const uint32_t my_ring = pin32(ring_s + lane * 32u);\n"
                 "  const uint32_t used_s = pin32((uint32_t)__cvta_generic_to_shared(gx_used));\n"
                 "  const uint32_t next_s = (uint32_t)__cvta_generic_to_shared(&gx_next);\n"
                 "  uint32_t st_s = 0, ph_s = 0;\n  (void)st_s; (void)ph_s;\n"
                 "  uint64_t rbase_s = (uint64_t)blockIdx.x * " << CW << ";\n  (void)rbase_s;\n"
                 "  #pragma unroll 1\n"
              << (stat ?
                 "  for (uint32_t c_ = 0;; c_++) {\n"
                 "    const uint32_t w_ = wid;\n"
                 "    const uint64_t rbase = rbase_s;\n"
                 "    rbase_s += gstride;\n"
                 "    if (rbase >= nrec) break;\n"
                 "    const uint32_t st = st_s, ph_c = ph_s;\n"
                 "    if (++st_s == " + std::to_string(S) + "u) { st_s = 0; ph_s ^= 1u; }\n" :
                 "  for (;;) {\n"
                 "    /* claim the block's next record: warps are not tied to a slot, so a slow record\n"
                 "     * (a long program, a diverged warp) does not hold back the stage refills */\n"
                 "    uint32_t r_ = 0;\n"
                 "    if (lane == 0) r_ = atoms_add(next_s, " + std::to_string(P) + "u);\n"
                 "    r_ = __shfl_sync(GX_ALL, r_, 0);\n"
                 "    const uint32_t c_ = r_ / " + std::to_string(W) + "u, w_ = r_ % " + std::to_string(W) + "u;\n"
                 "    const uint64_t rbase = (uint64_t)c_ * gstride + (uint64_t)blockIdx.x * " + std::to_string(W) + ";\n"
                 "    if (rbase >= nrec) break;\n"
                 "    const uint32_t st = c_ % " + std::to_string(S) + "u, ph_c = (c_ / " + std::to_string(S) + "u) & 1u;\n")
              << (mbar_rel ?
                 "    if (w_ == 0 && c_ >= 1) {                /* first claimant of chunk c: issue chunk c+S-1 */\n"
                 "      const uint32_t c2 = c_ + " + std::to_string(S - 1) + "u, st2 = c2 % " + std::to_string(S) + "u;\n"
                 "      if (lane == 0) {\n"
                 "        mbar_wait(empty_s + st2 * 8u, ((c2 / " + std::to_string(S) + "u) - 1u) & 1u);   /* chunk c-1 read */\n"
                 "        asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
                 "        stage_issue(st2, (uint64_t)c2 * gstride + (uint64_t)blockIdx.x * " + std::to_string(CW) + ");\n"
                 "      }\n"
                 "    }\n" : "") <<
                 "    mbar_wait(full_s + st * 8u, ph_c);\n"
                 "    const uint32_t ra_ = my_ring + st * " << 1024 * CW << "u + w_ * " << 1024 * P << "u;\n"
                 "    uint4 ea_[" << P << "], eb_[" << P << "];\n"
                 "    #pragma unroll\n"
                 "    for (int u = 0; u < " << P << "; u++) { ea_[u] = lds128(ra_ + u * 1024u); eb_[u] = lds128(ra_ + u * 1024u + 16u); }\n"
                 "    __syncwarp();\n"
              << (mbar_rel ?
                 "    if (lane == 0) asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(empty_s + st * 8u) : \"memory\");\n" :
                 "    if (lane == 0 && atoms_add(used_s + st * 4u, 1u) == " + std::to_string(W - 1) + "u) {\n"
                 "      gx_used[st] = 0;\n"
                 "      asm volatile(\"fence.proxy.async.shared::cta;\" ::: \"memory\");\n"
                 "      stage_issue(st, rbase + " + std::to_string(S) + " * gstride);\n"
                 "    }\n") <<
                 "    /* " << P << " records per claim: one claim and one release atomic per " << P << " */\n"
                 "    #pragma unroll\n"
                 "    for (int u = 0; u < " << P << "; u++) {\n"
                 "    const uint64_t rec = rbase + w_ * " << P << " + u;\n"
                 "    if (rec >= nrec) break;\n"
                 "    const uint4 a = ea_[u], b = eb_[u];\n";
        } else if (S >= 2) {
            /* a1 through a per-warp ring of S one-record (1 KiB) slots in dynamic shared memory:
             * record k+S-1 is in flight while record k runs.  Modes (GX_JIT_STAGE_MODE):
             *   0 lane: lane l cp.asyncs its own event's two 16-B halves to slot words l, 32+l
             *           (no cross-lane hazard; stride-32 B global reads),
             *   1 coal: lane l cp.asyncs record bytes 16l and 512+16l (coalesced), the record keeps
             *           its AoS layout and a __syncwarp orders the lanes,
             *   2 bulk: one 1-D TMA bulk copy per record (cp.async.bulk + per-slot mbarrier). */
            const int mode = gx_jit_stage_mode();
            auto issue = [&](const std::string &ls, const std::string &rec) {
                std::ostringstream t;
                if (mode == 0) {
                    t << "{ const uint64_t i_ = (" << rec << ") * 32 + lane; if (i_ < n) { cp_async16(ring_s + (" << ls
                      << ") * 1024u + lane * 16u, ev + 2 * i_, pol); cp_async16(ring_s + (" << ls
                      << ") * 1024u + 512u + lane * 16u, ev + 2 * i_ + 1, pol); } cp_async_commit(); }";
                } else if (mode == 1) {
                    t << "{ const uint64_t r_ = " << rec << "; const uint64_t i_ = r_ * 32 + (lane >> 1);"
                      << " if (i_ < n) cp_async16(ring_s + (" << ls << ") * 1024u + lane * 16u, ev + r_ * 64 + lane, pol);"
                      << " if (i_ + 16 < n) cp_async16(ring_s + (" << ls << ") * 1024u + 512u + lane * 16u, ev + r_ * 64 + 32 + lane, pol);"
                      << " cp_async_commit(); }";
                } else {
                    t << "{ const uint64_t r_ = " << rec << "; if (lane == 0 && r_ < nrec) { const uint64_t left_ = n - r_ * 32;"
                      << " bulk_load(ring_s + (" << ls << ") * 1024u, ev + r_ * 64, left_ >= 32 ? 1024u : (uint32_t)left_ * 32u, bar_s + ("
                      << ls << ") * 8u, pol); } }";
                }
                return t.str();
            };
            o << "  extern __shared__ __align__(128) uint4 gx_ring[];\n"
                 "  const uint4 *ring = gx_ring + (threadIdx.x >> 5) * " << 64 * S << ";\n"
                 "  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);\n"
                 "  const uint64_t rec0 = (uint64_t)blockIdx.x * " << B / 32 << " + (threadIdx.x >> 5);\n";
            if (mode == 2) {
                o << "  __shared__ __align__(8) uint64_t gx_bar[" << (B / 32) * S << "];\n"
                     "  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(gx_bar + (threadIdx.x >> 5) * " << S << ");\n"
                     "  if (lane == 0) {\n"
                     "    for (int k = 0; k < " << S << "; k++) mbar_init(bar_s + k * 8u, 1);\n"
                     "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n"
                     "  }\n"
                     "  __syncwarp();\n"
                     "  uint32_t phases = 0;\n";
            }
            o << "  #pragma unroll\n"
                 "  for (int k = 0; k < " << S - 1 << "; k++) " << issue("k", "rec0 + k * nwarps") << "\n"
              << pdl_wait <<
                 "  uint32_t slot = 0;\n"
                 "  #pragma unroll 1\n"
                 "  for (uint64_t rec = rec0; rec < nrec; rec += nwarps) {\n"
                 "    {\n"
                 "      const uint32_t ls = slot == 0 ? " << S - 1 << "u : slot - 1;\n"
              << (mode == 0 ? "" : "      __syncwarp();\n")
              << "      " << issue("ls", "rec + " + std::to_string(S - 1) + " * nwarps") << "\n"
                 "    }\n";
            if (mode == 2)
                o << "    mbar_wait(bar_s + slot * 8u, (phases >> slot) & 1u);\n"
                     "    phases ^= 1u << slot;\n";
            else
                o << "    cp_async_wait<" << S - 1 << ">();\n";
            if (mode == 1) o << "    __syncwarp();\n";
            if (mode == 0)
                o << "    const uint4 a = ring[slot * 64 + lane], b = ring[slot * 64 + 32 + lane];\n";
            else
                o << "    const uint4 a = ring[slot * 64 + 2 * lane], b = ring[slot * 64 + 2 * lane + 1];\n";
            o << "    slot = slot == " << S - 1 << "u ? 0u : slot + 1;\n";
        } else {
            o << pdl_wait;
            o << "  /* one warp = one 32-event record at a time (event lane == executor lane); U records per\n"
                 "   * iteration, their loads issued back to back */\n"
                 "  for (uint64_t rb = (uint64_t)blockIdx.x * " << B / 32 << " + (threadIdx.x >> 5); rb < nrec; rb += nwarps * " << U << ") {\n"
                 "    uint4 ea[" << U << "], eb[" << U << "];\n"
                 "    #pragma unroll\n"
                 "    for (int u = 0; u < " << U << "; u++) {\n"
                 "      const uint64_t i = (rb + u * nwarps) * 32 + lane;\n"
                 "      if (i < n) { ea[u] = ldg_stream_ef(ev + 2 * i, pol); eb[u] = ldg_stream_ef(ev + 2 * i + 1, pol); }\n"
                 "    }\n"
                 "    #pragma unroll" << (punroll ? "" : " 1") << "\n"
                 "    for (int u = 0; u < " << U << "; u++) {\n"
                 "    const uint64_t rec = rb + u * nwarps;\n"
                 "    if (rec >= nrec) break;\n"
              << (punroll ? "    const uint4 a = ea[u], b = eb[u];\n"
                          : "    const uint4 a = ea[0], b = eb[0];\n"
                            "    #pragma unroll\n    for (int k = 0; k + 1 < " + std::to_string(U) +
                                "; k++) { ea[k] = ea[k + 1]; eb[k] = eb[k + 1]; }\n");
        }
        o << "    Ctx c; c.w[0] = a.x; c.w[1] = a.y; c.w[2] = a.z; c.w[3] = a.w; c.w[4] = b.x; c.w[5] = b.y; c.w[6] = b.z; c.w[7] = b.w;\n"
             "    const uint64_t i = rec * 32 + lane;\n"
             "    uint64_t retv = 0;\n";
        if (L.single >= 0) {
            /* one program for every event.  A whole record (the warp-uniform test rec*32+32 <= n) runs
             * the whole-warp instance; a ragged tail record runs the masked one.  The run count (= n)
             * is added once at the end instead of per event. */
            o << "    if (rec < nfull) {\n"
                 "      prog0<true>(c, GX_ALL, retv, shard, spriv, c_herr, c_drop, c_rbb, c_hfull, ptc, pkc);\n"
                 "      if (WANT_RET) ret[i] = retv;\n"
                 "    } else {\n"
                 "      const bool valid = i < n;\n"
                 "      const unsigned m = __ballot_sync(GX_ALL, valid);\n"
                 "      prog0<false>(c, m, retv, shard, spriv, c_herr, c_drop, c_rbb, c_hfull, ptc, pkc);\n"
                 "      if (WANT_RET && valid) ret[i] = retv;\n"
                 "    }\n";
        } else {
            o << "    const bool valid = i < n;\n    int p = -1;\n"
                 "    if (valid) { const uint32_t kind = b.x & 0xFF, tenant = (b.x >> 8) & 0xFF;\n      switch (kind * 256 + tenant) {\n";
            for (int k = 0; k < GX_MAX_KINDS; k++)
                for (int t = 0; t < 256; t++)
                    if (L.attach[k][t] >= 0) o << "      case " << k * 256 + t << ": p = " << (int)L.attach[k][t] << "; break;\n";
            o << "      default: break;\n      }\n    }\n";
            o << "    if (valid) { if (p >= 0) c_run++; else c_skip++; }\n"
                 "    unsigned todo = __ballot_sync(GX_ALL, p >= 0);\n"
                 "    while (todo) {\n"
                 "      const int pq = __shfl_sync(GX_ALL, p, __ffs(todo) - 1);\n"
                 "      const unsigned m = __ballot_sync(GX_ALL, p == pq) & todo;\n"
                 "      todo &= ~m;\n"
                 "      switch (pq) {\n";
            for (size_t q = 0; q < images.size(); q++)
                o << "      case " << q << ":\n        if (m == GX_ALL) prog" << q << "<true>(c, m, retv, shard, spriv, c_herr, c_drop, c_rbb, c_hfull, ptc, pkc);\n"
                  << "        else prog" << q << "<false>(c, m, retv, shard, spriv, c_herr, c_drop, c_rbb, c_hfull, ptc, pkc);\n        break;\n";
            o << "      default: break;\n      }\n    }\n"
                 "    if (WANT_RET && valid) ret[i] = retv;\n";
        }
        o << (two_level ? "    }\n  }\n" : "  }\n");
        o << "  ptc_flush(ptc);\n";
        if (pkc_fd_ >= 0)
            o << "  ptkc_flush(pkc, " << hex(L.maps[pkc_fd_].data) << ", shard);\n";
        o << ""
             "  {\n"
             "  unsigned long long w_run = c_run, w_skip = c_skip, w_herr = c_herr, w_drop = c_drop, w_hfull = c_hfull;\n"
             "  for (int s = 16; s; s >>= 1) {\n"
             "    w_run += __shfl_xor_sync(GX_ALL, w_run, s); w_skip += __shfl_xor_sync(GX_ALL, w_skip, s);\n"
             "    w_herr += __shfl_xor_sync(GX_ALL, w_herr, s); w_drop += __shfl_xor_sync(GX_ALL, w_drop, s);\n"
             "    c_rbb += __shfl_xor_sync(GX_ALL, c_rbb, s); w_hfull += __shfl_xor_sync(GX_ALL, w_hfull, s);\n"
             "  }\n"
             "  if (lane == 0) {\n"
             "    if (w_run) atomicAdd(&sstats[" << GXS_RUN << "], w_run);\n"
             "    if (w_skip) atomicAdd(&sstats[" << GXS_SKIP << "], w_skip);\n"
             "    if (w_herr) atomicAdd(&sstats[" << GXS_HERR << "], w_herr);\n"
             "    if (w_drop) atomicAdd(&sstats[" << GXS_RB_DROPS << "], w_drop);\n"
             "    if (c_rbb) atomicAdd(&sstats[" << GXS_RB_BYTES << "], c_rbb);\n"
             "    if (w_hfull) atomicAdd(&sstats[" << GXS_HFULL << "], w_hfull);\n"
             "  }\n"
             "  }\n"
             "  __syncthreads();\n";
        for (uint32_t k = 0; k < L.n_priv; k++) {
            const GxMapDesc &m = L.maps[L.priv_maps[k]];
            const uint32_t nw = m.max_entries * m.value_size / 8;
            o << "  for (uint32_t w = threadIdx.x; w < " << nw << "u; w += " << B << ") {\n";
            o << "    const uint64_t v = (uint64_t)spriv[" << m.priv_off / 4 << " + w] | ((uint64_t)spriv["
              << m.priv_off / 4 + nw << " + w] << 32);\n"
              << "    if (v) atomicAdd((unsigned long long *)" << hex(m.data) << " + w, (unsigned long long)v);\n  }\n";
        }
        if (L.single >= 0) o << "  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&gstats[" << GXS_RUN << "], (unsigned long long)n);\n";
        o << "  if (threadIdx.x < 8 && sstats[threadIdx.x]) atomicAdd(&gstats[threadIdx.x], sstats[threadIdx.x]);\n}\n\n";
    }
};

}  // namespace

/* read at every compile (a compiled configuration keeps its shared-memory size in LaunchCfg) */
int gx_jit_stages() {
    /* 4 stages of 32 KiB (round 2, profiles/r2_stages.md): once the per-thread key cache took the
     * per-thread RMWs off C2, the deeper ring wins (C2 5.27 -> 4.90 ms, C5 3.79 -> 3.49, C1 2^26
     * 0.313 -> 0.303; C3 6.16 -> 6.28).  Round 1 measured 2 best (profiles/r1_jit_variants.md §9). */
    int v = 4;
    if (const char *e = getenv("GX_JIT_STAGES")) v = atoi(e);
    return std::max(0, std::min(8, v));
}

/* The ring depth of one launch configuration: the default (4) unless the launch is ONE program that
 * probes a hash map -- its probe chain walks through L1, which a deeper ring's shared memory takes
 * away (C3: 6.16 ms at 2 stages, 6.28-6.48 at 4; profiles/r2_stages.md).  GX_JIT_STAGES overrides. */
int gx_jit_stages_for(const std::vector<const GxInsn *> &images, const std::vector<uint32_t> &sizes) {
    if (getenv("GX_JIT_STAGES")) return gx_jit_stages();
    if (images.size() == 1)
        for (uint32_t i = 0; i < sizes[0]; i++)
            if (images[0][i].op == GX_CALL_LOOKUP_HASH) return 2;
    return gx_jit_stages();
}

int gx_jit_ring_rpw(int stages) {
    int v = 1;
    if (const char *e = getenv("GX_JIT_RING_RPW")) v = atoi(e);
    if (getenv("GX_JIT_RING_CLAIM") && strcmp(getenv("GX_JIT_RING_CLAIM"), "dynamic") == 0) v = 1;
    v = std::max(1, std::min(4, v));
    const int st = stages >= 2 ? stages : 3;
    while (v > 1 && st * v * (gx_jit_block() / 32) > 200) v--; /* the ring stays within 200 KiB of SMEM */
    return v;
}

int gx_jit_stage_mode() {
    int v = 3;
    if (const char *e = getenv("GX_JIT_STAGE_MODE")) v = atoi(e);
    return (v >= 0 && v <= 3) ? v : 3;
}

int gx_jit_block() {
    static int b = [] {
        int v = 1024;
        if (const char *e = getenv("GX_JIT_BLOCK")) v = atoi(e);
        return (v >= 64 && v <= 1024 && v % 32 == 0) ? v : 1024;
    }();
    return b;
}

const char *gx_jit_kernel_name(int variant) {
    static const char *names[4] = {"gx_jit_kernel", "gx_jit_kernel_r", "gx_jit_kernel_g", "gx_jit_kernel_gr"};
    return names[variant & 3];
}

std::string gx_jit_source(const GxLaunch &L, const std::vector<const GxInsn *> &images, const std::vector<uint32_t> &sizes,
                          int block, unsigned vmask, const std::vector<const uint16_t *> *narrow_in) {
    Gen g(L);
    if (narrow_in && narrow_in->size() == images.size()) g.nin_ = *narrow_in;
    g.kernel(images, sizes, block, vmask);
    return g.o.str();
}

std::string gx_jit_instrument_source(const GxLaunch &L, const GxInsn *image, uint32_t n, const std::string &user) {
    Gen g(L);
    g.instrument(image, n, user);
    return g.o.str();
}

int gx_jit_compile(const std::string &src, std::vector<char> &cubin, std::string &log) {
    Nvrtc &nv = nvrtc();
    if (!nv.ok) {
        log = nv.err;
        return -1;
    }
    std::vector<const char *> names, texts;
    for (int k = 0; kJitHeaders[k].name; k++) {
        names.push_back(kJitHeaders[k].name);
        texts.push_back(kJitHeaders[k].text);
    }
    nvrtcProgram prog;
    nvrtcResult r = nv.create(&prog, src.c_str(), "gx_jit.cu", (int)names.size(), texts.data(), names.data());
    if (r != NVRTC_SUCCESS) {
        log = nv.errstr(r);
        return -1;
    }
    const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-DGX_JIT=1", "-w"};
    r = nv.compile(prog, (int)(sizeof opts / sizeof *opts), opts);
    size_t ls = 0;
    nv.log_size(prog, &ls);
    log.assign(ls, 0);
    if (ls) nv.log(prog, &log[0]);
    if (r != NVRTC_SUCCESS) {
        nv.destroy(&prog);
        return -1;
    }
    size_t cs = 0;
    nv.cubin_size(prog, &cs);
    cubin.resize(cs);
    nv.cubin(prog, cubin.data());
    nv.destroy(&prog);
    if (const char *dump = getenv("GX_JIT_DUMP_CUBIN")) {
        if (FILE *f = fopen(dump, "wb")) {
            fwrite(cubin.data(), 1, cubin.size(), f);
            fclose(f);
        }
    }
    return 0;
}
