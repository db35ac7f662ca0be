/*
 * gx.h -- C ABI of the gx device-side eBPF runtime for B200 (sm_100a).
 *
 * The boundary of the data-parallel hot path of gpu_ext (arXiv 2512.12615): "a loader library
 * that installs policies and configures eBPF maps" (§4.2 User-space Control
 * Plane); device programs are "verified ... JIT-compiled ... [and run] at warp granularity"
 * (§4.2), with a SIMT-aware verifier (§4.4.1; 310, §5.3) and
 * maps "accessible from host-side driver hooks, GPU-side device policies, and user-space
 * control planes" (§4.4.3).  The calls follow SURVEY.md §8(b).
 *
 * Conventions (all calls):
 *   - Return 0 (or a non-negative handle) on success, a NEGATIVE errno on failure:
 *       -EINVAL  malformed argument, bytecode or map spec
 *       -EACCES  the verifier rejected the program (details in the report / log)
 *       -E2BIG   program too large, complexity limit or budget exceeded, or a full map
 *       -ENOMEM  device or host allocation failed
 *       -EFAULT  a CUDA error; gx_last_error() has the text
 *       -EPERM   running a program that has not passed gx_verify
 *       -ENOENT  unknown handle
 *     No C++ exception crosses this ABI.  gx_verify never raises: a rejection is a value.
 *   - Handles (map fds, program fds) are small non-negative ints, as BPF_PSEUDO_MAP_FD expects
 *     (bpf.h:1247-1266).  A program references a map by putting its fd in an ldimm64.
 *   - Device buffers passed in (events, R0) are caller-owned CUDA device memory (e.g. torch
 *     tensors) and must stay alive until the stream work completes (stream-ordered).
 *   - Maps are runtime-owned device memory, freed by gx_close.  Host map reads/writes are
 *     synchronous and ordered after all prior gx_run_batch calls on any stream of the runtime.
 *   - Batches of one gx_rt run one after another in submission order, even when they are given
 *     different streams (every batch records an event on its stream; a batch on another stream
 *     waits on it).  Under CUDA graph capture, give the runtime's batches the capturing stream.
 *   - One gx_rt per CUDA device.  A gx_rt is not thread-safe.
 *
 * Event record (the ctx every program sees in r1; read-only; 32 B, 32-B aligned):
 *     0 u64 addr | 8 u64 ts | 16 u32 hook (bits 0-7 kind, 8-15 tenant, 16 is_write)
 *     20 u32 block_id | 24 u16 sm_id | 26 u8 warp_id | 27 u8 lane_id | 28 u32 size
 *   Uniformity tags ("compact warp-uniform context"; 310 BTF annotations):
 *   addr and lane_id are LANE_VARYING, every other field is UNIFORM across the 32 events of
 *   an aligned warp record.  Uniformity is a performance contract, never a correctness one.
 */
#ifndef GX_H
#define GX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gx_rt gx_rt;

/* map types: bpf.h:925-965 numbering; PERTHREAD_ARRAY takes PERCPU_ARRAY's slot */
enum { GX_MAP_HASH = 1, GX_MAP_ARRAY = 2, GX_MAP_PERTHREAD_ARRAY = 6, GX_MAP_RINGBUF = 27,
       /* device->host prefetch request queue (F-2): key_size = value_size
        * = 0, max_entries = capacity in requests (a power of two in [64, 2^24]) */
       GX_MAP_PREFETCH_QUEUE = 64,
       /* device region (F-7): caller-owned device memory [base, base + len) that
        * gdev_prefetch_l2 may prefetch; made by gx_region_map, never by gx_create_map */
       GX_MAP_REGION = 65 };
/* Device helper ids beyond Linux's: gdev_mem_prefetch (§4.3.1 listing
 * "Request prefetch, triggers handler in host driver"), called as
 *     r0 = gdev_mem_prefetch(r1 = prefetch-queue map, r2 = addr, r3 = len)
 * The region is the run of 4-KiB pages [addr >> 12, (addr + len - 1) >> 12]; it queues the
 * request {first_page, npages} and returns 0, -EAGAIN (-11) if the queue is full (dropped,
 * counted in ringbuf_drops) or -EINVAL (-22) if len == 0, len > 2 MiB or addr + len wraps.
 * Prefetching is idempotent: the queue's content is a SET, and the device merges identical
 * requests of one warp group (PAPER.md:286 warp-level aggregation). */
enum { GX_FN_MEM_PREFETCH = 1000 };
/* gdev_prefetch_l2 ("Device-side L2 prefetch instructions (prefetch.global.L2)",
 * Table 1 "GPU L2 Stride Prefetch ... Device"), called as
 *     r0 = gdev_prefetch_l2(r1 = region map, r2 = addr, r3 = len)
 * issues one prefetch.global.L2 per 128-B line of [addr, addr + len) and returns 0, or -EINVAL
 * (-22) if len == 0 or len > 64 KiB, or -EFAULT (-14) if the range is not inside the region (no
 * prefetch is issued then).  A hint: no map or event state changes. */
enum { GX_FN_PREFETCH_L2 = 1001 };
/* hook kinds (event hook word bits 0-7): PAPER.md:225-230 (gdev_mem_ops.access), 260-262
 * (gdev_sched_ops.enter), 303 (fault-style records) */
enum { GX_HOOK_MEM_ACCESS = 0, GX_HOOK_BLOCK_ENTER = 1, GX_HOOK_FAULT = 2,
       GX_HOOK_FENCE = 3 /* gdev_mem_ops.fence: f4 gx_hook_fence */ };
/* update flags, bpf.h:1300-1302 */
enum { GX_ANY = 0, GX_NOEXIST = 1, GX_EXIST = 2 };

typedef struct {
    uint32_t type;         /* GX_MAP_* */
    uint32_t key_size;     /* ARRAY/PERTHREAD: 4.  HASH: 4 or 8.  RINGBUF: 0 */
    uint32_t value_size;   /* multiple of 8.  ARRAY <= 65536, PERTHREAD <= 256, HASH == 8. RINGBUF: 0 */
    uint32_t max_entries;  /* > 0.  RINGBUF: byte capacity, a power of two >= 4096 */
    uint32_t flags;        /* must be 0 */
} gx_map_spec;

typedef struct {
    uint32_t simt_strict;      /* 1: enforce PAPER.md:282's SIMT rules (uniform branches, loop
                                  bounds, map-update keys, atomics); 0 (default): relaxed, the
                                  executor handles divergence at run time */
    uint32_t max_insns;        /* worst-case executed instructions per event (0 -> 4096) */
    uint32_t max_helpers;      /* worst-case weighted helper calls (lookup 1, update 2, other 1; 0 -> 64) */
    uint32_t max_memops;       /* worst-case memory operations (0 -> 1024) */
    uint32_t complexity_limit; /* verifier processed-instruction limit (0 -> 1000000) */
} gx_verify_opts;

/* verifier rule ids */
enum {
    GX_OK = 0, GX_BAD_INSN, GX_BAD_REG, GX_BAD_JUMP, GX_FALLTHROUGH, GX_UNREACHABLE, GX_UNINIT_READ,
    GX_OOB_ACCESS, GX_NULL_DEREF, GX_MISALIGNED, GX_PTR_LEAK, GX_SHIFT_RANGE, GX_BAD_HELPER,
    GX_FORBIDDEN_SYNC, GX_UNBOUNDED_LOOP, GX_COMPLEXITY, GX_BUDGET, GX_UNIFORM_BRANCH,
    GX_UNIFORM_LOOP_BOUND, GX_UNIFORM_MAP_KEY, GX_NON_UNIFORM_ATOMIC, GX_MIXED_PTR, GX_NUM_RULES
};

typedef struct {
    int32_t verdict;           /* 0 accepted, else -EACCES / -E2BIG / -EINVAL */
    uint32_t n_violations;
    uint32_t first_insn;       /* slot index of the first violation */
    uint32_t first_rule;       /* GX_* rule id of the first violation */
    uint64_t worst_insns;      /* worst case over explored paths */
    uint64_t worst_helpers;
    uint64_t worst_memops;
    uint64_t processed_insns;  /* verifier work */
    uint32_t stack_depth;      /* bytes, rounded up to 8 */
    uint32_t all_uniform;      /* 1 if no conditional branch depends on a LANE_VARYING value */
    uint32_t commutative;      /* 1 if shared maps change only through commutative updates */
    uint32_t n_insns;          /* input slots */
    uint32_t image_insns;      /* executor instructions after pre-decoding (dead helper-argument
                                  set-up removed, superinstructions fused, ldimm64 pairs merged) */
    uint32_t reserved;
} gx_verify_report;

typedef struct {
    uint64_t events_run;       /* events a program ran on */
    uint64_t events_skipped;   /* no program attached for the event's (kind, tenant) */
    uint64_t divergent_steps;  /* warp-steps executed on the min-PC divergent path */
    uint64_t helper_errors;    /* helpers that returned a negative errno */
    uint64_t ringbuf_bytes;    /* bytes committed to ring buffers */
    uint64_t ringbuf_drops;    /* ringbuf_output calls dropped (-EAGAIN) */
    uint64_t hash_full;        /* hash inserts refused because max_entries was reached */
    uint64_t warp_steps;       /* interpreted warp-instructions (all paths; 0 for the JIT engine) */
    uint64_t bounds_violations; /* GX_JIT_BOUNDS=1 (debug mode of the JIT engine): map accesses whose
                                   address fell outside their map -- redirected to a scratch word and
                                   counted instead of executed (0 in the default mode) */
} gx_batch_stats;

/* ---------------------------------------------------------------- runtime */
int  gx_open(int cuda_device, gx_rt **out);              /* -EFAULT if the device is not sm_100 */
void gx_close(gx_rt *rt);
const char *gx_last_error(gx_rt *rt);                   /* text of the last failure ("" if none) */

/* ---------------------------------------------------------------- maps */
/* Creates a zero-initialised map in device memory; *map_fd = its handle. */
int  gx_create_map(gx_rt *rt, const gx_map_spec *spec, int *map_fd);
/* Registers caller-owned device memory [dev_ptr, dev_ptr + len) (len > 0; it must outlive the map
 * and every launch that uses it) as a GX_MAP_REGION map for gdev_prefetch_l2.  A region has no
 * content: gx_update_map / gx_read_map return -EINVAL and merges skip it.  -EINVAL if dev_ptr is
 * NULL, len is 0 or dev_ptr + len wraps. */
int  gx_region_map(gx_rt *rt, const void *dev_ptr, uint64_t len, int *map_fd);
/* Host control-plane write of n (key, value) pairs, packed back to back (key_size / value_size
 * bytes each, host memory), with bpf_map_update_elem semantics (bpf.h:1762-1776).  PERTHREAD:
 * writes shard 0 and zeroes the other shards.  Synchronous.  Returns 0 or the first -errno. */
int  gx_update_map(gx_rt *rt, int map_fd, const void *keys, const void *vals, uint64_t n, uint64_t flags);
/* Canonical view into host buffers.  ARRAY / PERTHREAD (summed over shards):
 * all max_entries values in key order (keys gets the u32 indices when non-NULL).  HASH: live
 * entries sorted by key as an unsigned little-endian integer.  cap = capacity in entries;
 * *n_out = entries written.  -E2BIG if cap is too small.  Synchronous. */
int  gx_read_map(gx_rt *rt, int map_fd, void *keys, void *vals, uint64_t cap, uint64_t *n_out);
/* Copies the committed ring-buffer bytes ([u32 len | u32 pg_off | payload padded to 8]*,
 * bpf.h:6064-6066 layout) into buf and resets the buffer.  *n_bytes = bytes copied.  -E2BIG
 * (nothing copied) if cap < committed bytes.  Synchronous. */
int  gx_ringbuf_drain(gx_rt *rt, int map_fd, void *buf, uint64_t cap, uint64_t *n_bytes);
/* Copies the queued prefetch requests as u64 pairs {first_page, npages} (queue order, identical
 * requests of one warp group merged) into reqs and empties the queue.  cap = capacity in
 * requests; *n_req = requests copied; -E2BIG (nothing copied) if cap is too small.  Synchronous.
 * (With a daemon running, the daemon drains the queues instead.) */
int  gx_prefetch_drain(gx_rt *rt, int map_fd, uint64_t *reqs, uint64_t cap, uint64_t *n_req);

/* ---------------------------------------------------------------- inline instrumentation (§8f f4)
 * "Trampolines, placed at GPU kernel entry, selected memory instructions (such as global loads and
 * atomic operations) ... verified eBPF code executes after kernel launch" (§5.3);
 * the vector-add hook-overhead microbenchmark.  Here the trampoline is made
 * at compile time: gx_instrument JIT-compiles the verified program prog_fd as inline __device__ hooks
 * together with user_src (CUDA C++ with extern "C" __global__ kernels) in one NVRTC sm_100a module:
 *     uint64_t gx_hook_access(unsigned group, const void *addr, uint32_t size, bool is_write);
 *     uint64_t gx_hook_block_enter(unsigned group, uint64_t unit, uint32_t cost);
 *     uint64_t gx_hook_fence(unsigned group, uint64_t scope);                  (kind GX_HOOK_FENCE)
 *     uint64_t gx_hook_probe(unsigned group, uint64_t fn);                     (kind GX_HOOK_PROBE)
 *     uint64_t gx_hook_retprobe(unsigned group, uint64_t fn, uint32_t retval);  (kind GX_HOOK_RETPROBE)
 *     uint64_t gx_hook_event(unsigned group, uint64_t addr, uint32_t hook, uint32_t size,
 *                            uint32_t *rec = nullptr);  (any kind; rec receives the 8-word record)
 * Each call runs the program once per lane of `group` on an event record built in registers
 * (addr, globaltimer ts, hook word, linear block id, %smid, hardware warp slot, lane, size) and
 * returns that lane's R0 (the policy decision).  `group` must be exactly the set of lanes making the
 * call together -- e.g. __ballot_sync(~0u, pred) taken where the warp is converged, then the call
 * under `if (pred)` -- because the helpers' warp collectives name it.  Per-thread maps are sharded by
 * (SM, warp slot, lane); maps are never privatised in shared memory; map addresses are baked into
 * the module (the maps must outlive the handle).  Errors: -ENOENT (no program), -EPERM (not
 * verified), -EINVAL (module does not compile; log holds the NVRTC log). */
typedef struct gx_kernel gx_kernel;
int  gx_instrument(gx_rt *rt, int prog_fd, const char *user_src, gx_kernel **out, char *log, uint64_t log_len);
/* Launches kernel `name` of the module (cuLaunchKernel argument conventions; async on the stream). */
int  gx_kernel_launch(gx_rt *rt, gx_kernel *k, const char *name, const uint32_t grid[3], const uint32_t block[3],
                      uint32_t smem, void **args, void *cuda_stream);
void gx_kernel_free(gx_rt *rt, gx_kernel *k);

/* ---------------------------------------------------------------- block scheduling (§8f f3)
 * The work-stealing thread-block scheduler of PAPER.md §4.3.2 ("Return whether to steal work (TB
 * scheduler)") and §6.2.1 (persistent worker blocks pull work units; FixedWork / Greedy /
 * LatencyBudget): n_workers persistent worker blocks, unit u initially in the deque of home[u]
 * (unit order).  A worker pops its own deque's head: ENTER hook, cost_us[u] microseconds of work
 * (a globaltimer spin standing for the unit's kernel body), EXIT hook; with an empty deque it runs
 * the STEAL hook -- R0 == 0 retires the worker, otherwise it takes the tail unit of the largest
 * deque (lowest id on ties; a CAS per attempt), spins steal_cost_us, and runs it with the stolen bit.
 * Hook records (F-5): addr = unit (STEAL: 0), ts = %globaltimer, hook = kind
 * (GX_HOOK_BLOCK_ENTER 1, GX_HOOK_BLOCK_EXIT 4, GX_HOOK_STEAL 5) | stolen << 16, block_id =
 * worker, size = cost_us.  prog_fd (verified) is compiled into the worker kernel (gx_instrument).
 * Outputs (host arrays): executed_by[n_units] (worker), stolen[n_units], busy_ns / end_ns (from
 * the first worker's start) / steals [n_workers], *makespan_ns (device globaltimer).  Synchronous. */
enum { GX_HOOK_BLOCK_EXIT = 4, GX_HOOK_STEAL = 5, GX_HOOK_PROBE = 6, GX_HOOK_RETPROBE = 7 };
int  gx_sched_run(gx_rt *rt, int prog_fd, uint32_t n_units, const uint32_t *cost_us, const uint32_t *home,
                  uint32_t n_workers, uint32_t steal_cost_us, uint32_t *executed_by, uint8_t *stolen,
                  uint64_t *busy_ns, uint64_t *end_ns, uint32_t *steals, uint64_t *makespan_ns);
/* gx_sched_run with modes and a hook log (F-6).
 * flags: GX_SCHED_CLC -- no deques: the grid has one block per unit (unit u = block u; home must be
 *   NULL, n_workers is ignored and every per-worker array has n_units entries).  After its unit a
 *   block runs the STEAL hook; R0 != 0 cancels a not-yet-launched block with Blackwell cluster launch
 *   control (clusterlaunchcontrol.try_cancel) and runs that block's unit with the stolen bit (the
 *   paper's "MaxSteals (CLC)" row); R0 == 0 or a failed cancel ends the block.  A
 *   cancelled block never starts (its end_ns is 0).
 *   GX_SCHED_PROBES -- the unit body is bracketed by PROBE (addr = 1, size = 0) and RETPROBE (addr = 1,
 *   size = unit) hooks: device function 1 starts / returns (gdev_sched_ops.probe/.retprobe,
 *   PAPER.md:265-267).
 * smem_per_block: dynamic shared memory per block (bytes; limits residency so that blocks stay
 *   pending for CLC to cancel).
 * log (host, log_cap entries, may be NULL with log_cap 0): every hook call in completion order --
 *   the 32-B record the program ran on, its R0, the worker (block) and the worker's hook sequence
 *   number 0, 1, ...; *log_n = hooks that ran.  -ENOSPC (after all outputs are written) when
 *   *log_n > log_cap (the first log_cap completed calls are kept). */
enum { GX_SCHED_CLC = 1, GX_SCHED_PROBES = 2 };
typedef struct { uint8_t rec[32]; uint64_t r0; uint32_t worker, seq; } gx_hook_log;
int  gx_sched_run_ex(gx_rt *rt, int prog_fd, uint32_t flags, uint32_t n_units, const uint32_t *cost_us,
                     const uint32_t *home, uint32_t n_workers, uint32_t steal_cost_us, uint32_t smem_per_block,
                     uint32_t *executed_by, uint8_t *stolen, uint64_t *busy_ns, uint64_t *end_ns, uint32_t *steals,
                     uint64_t *makespan_ns, gx_hook_log *log, uint64_t log_cap, uint64_t *log_n);

/* ---------------------------------------------------------------- runtime daemon (§8f f2)
 * "A runtime daemon asynchronously flushes GPU-local shards to host-visible canonical map
 * instances, providing coherent snapshots to host-side policies without synchronization
 * overhead" (§5.3); "snapshot-based aggregation at GPU kernel completion
 * boundaries"; device prefetch requests "trigger host-side prefetch
 * handlers".
 * While a daemon runs, every gx_run_batch / gx_run_batch_ex appends to ITS OWN stream, right
 * after the batch's kernel (= at that kernel-completion boundary): a publish kernel that writes
 * each prefetch queue's requests and each watched map's canonical snapshot into pinned host
 * memory and empties the queues, then an event.  The daemon thread waits for the event and
 * hands the requests to the handler and the snapshots to gx_snapshot_read -- the caller's
 * stream never synchronises with the host.  Four publish slots: a batch that finds none free
 * waits for the daemon (backpressure, counted).  Handlers run on the daemon thread. */
typedef void (*gx_prefetch_handler)(void *user, int map_fd, const uint64_t *reqs, uint64_t n_req);
typedef struct {
    uint64_t batches;          /* publish points processed */
    uint64_t requests;         /* prefetch requests handed to the handler */
    uint64_t snapshots;        /* map snapshots published */
    uint64_t backpressure;     /* batches that waited for a free publish slot */
    uint64_t managed_prefetches; /* default handler: cudaMemPrefetchAsync calls issued */
} gx_daemon_stats;
/* Starts the daemon.  handler == NULL installs the default handler: requests whose pages lie in
 * CUDA managed memory are prefetched to the device with cudaMemPrefetchAsync, others are only
 * counted.  -EBUSY if one runs. */
int  gx_daemon_start(gx_rt *rt, gx_prefetch_handler handler, void *user);
/* Drains what is published, then stops.  Safe when none runs. */
int  gx_daemon_stop(gx_rt *rt);
/* Adds an ARRAY or PERTHREAD_ARRAY map to the snapshot set (-EINVAL for other types). */
int  gx_daemon_watch(gx_rt *rt, int map_fd);
/* Latest published canonical snapshot of a watched map (max_entries * value_size bytes;
 * per-thread maps folded) and its version (= publish points so far; 0: none yet).  Never
 * touches the device.  -ENOENT if not watched, -E2BIG if cap is too small. */
int  gx_snapshot_read(gx_rt *rt, int map_fd, void *buf, uint64_t cap, uint64_t *version);
int  gx_daemon_get_stats(gx_rt *rt, gx_daemon_stats *out);
/* Registers the CUDA managed range the default handler prefetches into (requests outside it are
 * only counted); ptr == NULL clears it. */
int  gx_daemon_prefetch_range(gx_rt *rt, void *managed_ptr, uint64_t bytes);

/* ---------------------------------------------------------------- programs */
/* Copies n_slots 8-byte struct bpf_insn slots (bpf.h:72-77); structural decode and map-fd
 * relocation happen in gx_verify.  hook = the GX_HOOK_* kind the program is written for. */
int  gx_load_prog(gx_rt *rt, uint32_t hook, const void *insn_slots, uint32_t n_slots, int *prog_fd);
/* Runs the verifier and, on acceptance, pre-decodes the program for the
 * executor.  opts may be NULL (defaults).  report and log may be NULL.  The log receives one
 * line per violation "insn <i>: <RULE>: <message>".  Returns report->verdict. */
int  gx_verify(gx_rt *rt, int prog_fd, const gx_verify_opts *opts, gx_verify_report *report,
               char *log, uint64_t log_len);
/* The same verifier without a runtime or device: maps[i] describes the map whose fd is i
 * (type 0 = no such map; n_maps <= 64).  For tooling and CPU-side tests.  Returns
 * report->verdict. */
int  gx_verify_offline(const void *insn_slots, uint32_t n_slots, const gx_map_spec *maps, uint32_t n_maps,
                       const gx_verify_opts *opts, gx_verify_report *report, char *log, uint64_t log_len);
/* Generates and compiles (NVRTC, sm_100a) the JIT kernel of one program against map specs, with
 * placeholder map addresses, without a runtime or device -- for tooling and CPU-side tests.
 * src (nullable) receives the generated CUDA C++; log the compiler log.  Returns 0, the
 * verifier's -errno, or -ENOSYS if NVRTC is unavailable / compilation failed. */
int  gx_jit_offline(const void *insn_slots, uint32_t n_slots, const gx_map_spec *maps, uint32_t n_maps,
                    char *src, uint64_t src_len, char *log, uint64_t log_len);
/* Attach table entry (hook kind, tenant) -> program.  prog_fd = -1 detaches. */
int  gx_attach(gx_rt *rt, int prog_fd, uint32_t hook_kind, uint32_t tenant);

/* ---------------------------------------------------------------- execution (hot path) */
/* Runs one batch: every event runs its program (prog_fd >= 0: that program for all events;
 * -1: the attach table on the event's hook word) against the persistent maps (§8c c.1, S1, S2).
 * d_events: n_events * 32 B of device memory, 32-B aligned.  d_ret: NULL or n_events u64 of
 * device memory receiving R0 (0 for skipped events).  cuda_stream: a cudaStream_t (NULL = the
 * legacy default stream).  Asynchronous (stream-ordered).  -EPERM if the program is unverified. */
int  gx_run_batch(gx_rt *rt, const void *d_events, uint64_t n_events, int prog_fd, uint64_t *d_ret,
                  void *cuda_stream);
/* gx_run_batch with launch flags (0 = gx_run_batch):
 *   GX_RUN_OVERLAP  programmatic dependent launch (JIT engine; ignored by the interpreter): the
 *                   batch's grid may be scheduled while the preceding kernel on the stream is still
 *                   draining and may start READING d_events before that kernel completes; every
 *                   map access, stat update and d_ret write still waits for its completion and
 *                   memory flush (griddepcontrol.wait), so back-to-back batches keep the sequential
 *                   semantics (S1).  The caller promises that d_events is not written by the work
 *                   immediately preceding on the stream (e.g. events generated or copied earlier
 *                   and already complete, as in a steady-state stream of resident batches).
 * Errors as gx_run_batch; -EINVAL for unknown flags. */
enum { GX_RUN_OVERLAP = 1 };
int  gx_run_batch_ex(gx_rt *rt, const void *d_events, uint64_t n_events, int prog_fd, uint64_t *d_ret,
                     void *cuda_stream, uint32_t flags);
/* Same, from HOST memory (pinned or pageable): the events are copied to the device in chunks
 * on the runtime's own streams, overlapping copies with execution; h_ret (nullable) receives R0.
 * Synchronous.  This is the end-to-end path bench.py times as "e2e". */
int  gx_run_batch_host(gx_rt *rt, const void *h_events, uint64_t n_events, int prog_fd, uint64_t *h_ret);
/* Execution engine for subsequent batches (default GX_ENGINE_JIT):
 *   GX_ENGINE_INTERP  the warp-cooperative interpreter (uniform-PC fast path, min-PC divergent
 *                     path);
 *   GX_ENGINE_JIT     the verified, pre-decoded programs of a launch configuration compiled to
 *                     sm_100a code by NVRTC, cached
 *                     per configuration; -ENOSYS if libnvrtc cannot be loaded.
 * Both engines compute the same results (parity-tested against the oracle). */
enum { GX_ENGINE_INTERP = 0, GX_ENGINE_JIT = 1 };
int  gx_set_engine(gx_rt *rt, int engine);
int  gx_get_engine(gx_rt *rt);
/* Cumulative stats since the last call (then reset).  Synchronous. */
int  gx_get_stats(gx_rt *rt, gx_batch_stats *out);
/* Launch geometry of the executor: grid blocks, threads per block, dynamic shared bytes of the
 * last launch, and the number of kernel launches issued since gx_open. */
int  gx_exec_info(gx_rt *rt, uint32_t *grid, uint32_t *block, uint32_t *smem, uint64_t *launches);

/* ---------------------------------------------------------------- multi-GPU merge (§8e, S3)
 * Snapshot-and-merge across G replicas ("snapshot ... at GPU kernel
 * completion boundaries").  Every rank created the same maps from the same initial state.
 *   gx_merge_export: additive maps (ARRAY / PERTHREAD folded) -> d_delta[u64 words] =
 *     local - base (mod 2^64), for the map's max_entries*value_size/8 words.
 *   gx_merge_apply:  local = base + d_sum; base = local (d_sum = the allreduced deltas).
 *   gx_hash_export:  entries whose value differs from the base (or that are new), as
 *     (key, value - base value) pairs, grouped by owner rank g = mix64(key) mod nranks into
 *     d_keys / d_vals (device, cap entries); h_counts[g] (host, nranks entries) = pairs of owner g,
 *     stored in owner order.  owner >= 0 keeps only the keys that rank owns.  Synchronous.
 *   gx_hash_apply:   GX_MERGE_RESTORE: local := base first; then, for every (key, delta):
 *     value += delta (absent keys are inserted at 0 first; duplicate keys accumulate);
 *     GX_MERGE_COMMIT: afterwards base := local.  -E2BIG if the union exceeds max_entries.
 *   gx_merge_words:  number of u64 words gx_merge_export writes for this map.
 * The key-sharded hash merge is: export grouped by owner -> all-to-all ->
 * apply(RESTORE) on the owner -> export(owner = self) -> all-gather -> apply(RESTORE|COMMIT).
 * All device pointers are caller-owned; merge_export / merge_apply / hash_apply are stream-ordered
 * on cuda_stream (hash_apply synchronises before returning). */
enum { GX_MERGE_RESTORE = 1, GX_MERGE_COMMIT = 2 };
/* (Re)takes the base snapshot of a map = the state every rank agrees on.  Call it on every rank
 * after identical initialisation and before the first batch; each merge then advances it. */
int  gx_merge_snapshot(gx_rt *rt, int map_fd);
int  gx_merge_words(gx_rt *rt, int map_fd, uint64_t *words);
int  gx_merge_export(gx_rt *rt, int map_fd, uint64_t *d_delta, void *cuda_stream);
int  gx_merge_apply(gx_rt *rt, int map_fd, const uint64_t *d_sum, void *cuda_stream);
int  gx_hash_export(gx_rt *rt, int map_fd, uint32_t nranks, int32_t owner, uint64_t *d_keys, uint64_t *d_vals,
                    uint64_t cap, uint64_t *h_counts);
int  gx_hash_apply(gx_rt *rt, int map_fd, const uint64_t *d_keys, const uint64_t *d_vals, uint64_t n,
                   uint32_t flags, void *cuda_stream);

/* ---- Multi-GPU merge (§4.4.3 "merges these shards into canonical
 * snapshots at synchronization points", §5.3 "snapshot-based aggregation at GPU kernel
 * completion boundaries").  One gx_rt per GPU, one process per GPU; every rank creates the same maps,
 * applies the same host writes and loads the same programs, then runs its own event shard.
 *   gx_comm_unique_id: a fresh NCCL unique id (128 bytes into id_out) -- rank 0 makes it, the caller
 *     ships it to the other ranks (process bootstrap, e.g. torch.distributed).  -ENOSYS without NCCL.
 *   gx_comm_init:   joins the NCCL communicator (ncclCommInitRank on this gx_rt's device; collective
 *     over the nranks processes) and takes every map's base snapshot: the state all ranks agree on.
 *     Host writes (gx_update_map) after it must be identical on every rank and followed by
 *     gx_merge_snapshot of that map on every rank.
 *   gx_comm_init_host: the same merge over caller callbacks on HOST buffers (several ranks sharing one
 *     device, where NCCL refuses two ranks on one GPU; tests): allreduce_sum_u64 sums n u64 words in
 *     place over the ranks (wraparound); alltoallv sends send_bytes[g] bytes at send + send_off[g] to
 *     rank g and receives recv_bytes[g] bytes from rank g into recv + recv_off[g]; allgather puts rank
 *     g's `bytes` bytes at recv + g * bytes.  Callbacks return 0 or a negative errno.
 *   gx_merge:       collective over all ranks (call it on every rank at the same point, between
 *     batches): every map reaches S3's canonical state:
 *       ARRAY / PERTHREAD: canon = base + sum over ranks of (local - base), per u64 word (PERTHREAD
 *         folded first) -- one packed u64 SUM all-reduce over all such maps;
 *       HASH: key union, value = base (or 0 if new) + sum of deltas -- owner-sharded (owner =
 *         mix64(key) mod nranks): counts all-gather, (key, delta) all-to-all, owners accumulate onto
 *         the base, owners' merged deltas all-gathered, every rank rebuilds;
 *       RINGBUF / PREFETCH QUEUE: rank-local (their union is the multiset / set union; drain each).
 *     Afterwards base = canon on every rank.  Stream-ordered on cuda_stream; returns after it.
 *     -EINVAL (nothing changed) if a map is not mergeable by S3: an ARRAY written by anything but
 *     64-bit ATOMIC ADD (+-FETCH), a HASH whose values change by anything but 64-bit ATOMIC ADD or
 *     whose keys are inserted by update_elem with flags other than the constant BPF_NOEXIST (the
 *     verifier's usage facts of every loaded program); -E2BIG if a merged HASH union exceeds
 *     max_entries; -EIO on a transport error (gx_last_error).
 *   gx_comm_free:   leaves the communicator (gx_close does too). */
typedef struct {
    void *user;
    int (*allreduce_sum_u64)(void *user, uint64_t *buf, uint64_t n);
    int (*alltoallv)(void *user, const void *send, const uint64_t *send_bytes, const uint64_t *send_off, void *recv,
                     const uint64_t *recv_bytes, const uint64_t *recv_off);
    int (*allgather)(void *user, const void *send, void *recv, uint64_t bytes);
} gx_comm_host_ops;
int  gx_comm_unique_id(void *id_out);
int  gx_comm_init(gx_rt *rt, const void *nccl_unique_id, int nranks, int rank);
int  gx_comm_init_host(gx_rt *rt, const gx_comm_host_ops *ops, int nranks, int rank);
int  gx_merge(gx_rt *rt, void *cuda_stream);
int  gx_comm_free(gx_rt *rt);

#ifdef __cplusplus
}
#endif
#endif /* GX_H */
