/* gx_jit.h -- internal interface of the per-launch JIT (gx_jit.cpp). */
#pragma once
#include <string>
#include <vector>

#include "gx_internal.h"

/* launch variants of a configuration: event ingest (block-wide TMA ring / per-lane register loads)
 * x per-event R0 (off / on); bit k of a variant mask = variant k, kernel gx_jit_kernel_name(k) */
enum { GX_JIT_V_RING = 1, GX_JIT_V_RING_R = 2, GX_JIT_V_REG = 4, GX_JIT_V_REG_R = 8, GX_JIT_V_ALL = 15 };
const char *gx_jit_kernel_name(int variant);
/* CUDA C++ source of one launch configuration (programs in launch-slot order), the kernels of
 * the variants in `vmask` only. */
std::string gx_jit_source(const GxLaunch &L, const std::vector<const GxInsn *> &images,
                          const std::vector<uint32_t> &sizes, int block, unsigned vmask = GX_JIT_V_ALL,
                          const std::vector<const uint16_t *> *narrow_in = nullptr);
/* f4: CUDA C++ of the program as inline __device__ hooks (gx_hook_access / gx_hook_block_enter)
 * followed by the user's kernels; no privatised maps (L must have none). */
std::string gx_jit_instrument_source(const GxLaunch &L, const GxInsn *image, uint32_t n, const std::string &user);
/* NVRTC -> sm_100a cubin.  Returns 0, or -1 with the compiler log. */
int gx_jit_compile(const std::string &src, std::vector<char> &cubin, std::string &log);
/* preferred threads per block of the generated kernel (1024; GX_JIT_BLOCK = 256 / 512 for experiments);
 * the runtime falls back to 256 only when a 1024-thread block cannot be resident */
int gx_jit_block();
/* depth of the shared-memory event ring (cp.async / TMA staging, a1): 4 by default
 * (GX_JIT_STAGES; < 2 = register loads, GX_JIT_UNROLL records per iteration).  Dynamic shared memory per block =
 * gx_jit_smem(block) bytes. */
int gx_jit_stages();
/* staging mode: 0 per-lane cp.async, 1 coalesced cp.async, 2 per-warp TMA bulk, 3 block-wide TMA bulk
 * (default: one 32-KiB cp.async.bulk per block stage) */
int gx_jit_stage_mode();
/* records per warp per ring stage with static record assignment (GX_JIT_RING_RPW, 1 by default; a
 * stage then holds (block/32) x rpw records, brought in by one bulk copy) */
int gx_jit_ring_rpw(int stages);
/* the ring depth of one launch configuration (default 4; 2 for a single program that probes a hash map) */
int gx_jit_stages_for(const std::vector<const GxInsn *> &images, const std::vector<uint32_t> &sizes);
inline unsigned gx_jit_smem(int block, int stages) {
    const int s = stages >= 2 ? stages : 3;
    return (unsigned)(block / 32) * (unsigned)s * (unsigned)gx_jit_ring_rpw(s) * 1024u; /* the ring stages */
}
