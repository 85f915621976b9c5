// api.cu — the C ABI (include/dfk.h): contexts, weight registration +
// prepack, the fused forward path and its unfused cuBLASLt comparators,
// host-buffer forward, and the memory / timing plumbing.
//
// Reference behaviour mirrored here (paths under /root/reference/proj):
//   shape validation & ShapeError       src/fused.cpp:49-68, swiglu.cpp:26-39
//   run_fused = stage 1 then down       src/fused.cpp:209-216
//   two-kernel layout (gate cols first) src/swiglu.cpp:130-166, 194-212
//   four-kernel layout                  src/swiglu.cpp:170-192
//   down_projection                     src/swiglu.cpp:214-226
//   balanced_ranges                     src/tp.cpp:8-29
//   fused traffic model                 src/traffic.cpp:70-76, 82-94
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_profiler_api.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "internal.h"
#include "layout.cuh"
#include "stream_kernels.cuh"

namespace dfk {

namespace {
thread_local std::string g_last_error;
}

void set_error(int status, const std::string& msg) {
  (void)status;
  g_last_error = msg;
}

int fail(int status, const std::string& msg) {
  set_error(status, msg);
  return status;
}

void free_weights(dfk_weights_s* w) {
  if (w->s1_pack) cudaFree(w->s1_pack);
  if (w->dn_pack) cudaFree(w->dn_pack);
  if (w->cat_t) cudaFree(w->cat_t);
  if (w->down_t) cudaFree(w->down_t);
  delete w;
}

int clone_weights(dfk_context_s* ctx, const dfk_weights_s* w, dfk_weights_s** out) {
  auto* c = new dfk_weights_s(*w);
  c->s1_pack = c->dn_pack = nullptr;
  c->cat_t = c->down_t = nullptr;
  const size_t s1 = static_cast<size_t>(w->s1_tiles) * w->s1_kblocks * kBlockBytes;
  const size_t dn = static_cast<size_t>(w->dn_tiles) * w->dn_kblocks * kBlockBytes;
  if ((w->s1_pack && cudaMalloc(&c->s1_pack, s1) != cudaSuccess) ||
      (w->dn_pack && cudaMalloc(&c->dn_pack, dn) != cudaSuccess)) {
    cudaGetLastError();
    free_weights(c);
    return fail(DFK_ERR_NOMEM, "scheduler weight copy");
  }
  if (w->s1_pack) DFK_CUDA(cudaMemcpyAsync(c->s1_pack, w->s1_pack, s1,
                                           cudaMemcpyDeviceToDevice, ctx->stream));
  if (w->dn_pack) DFK_CUDA(cudaMemcpyAsync(c->dn_pack, w->dn_pack, dn,
                                           cudaMemcpyDeviceToDevice, ctx->stream));
  *out = c;
  return DFK_OK;
}

void release_clone(dfk_weights_s* w) {
  if (w) free_weights(w);
}

int tp_degree(const dfk_context_s* ctx, const dfk_weights_s* w) {
  int p = std::max(ctx->nranks, ctx->tp_sym_size);
  if (w && w->d_ff > 0 && w->d_ff < w->d_ff_total)
    p = std::max(p, static_cast<int>(std::lround(static_cast<double>(w->d_ff_total) / w->d_ff)));
  return std::max(p, 1);
}

int ensure_buf(dfk_context_s* ctx, DeviceBuf& b, size_t bytes, bool zero, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return DFK_OK;
  if (b.p) {
    cudaStreamSynchronize(s);
    cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
  }
  // Captured decode graphs bake buffer addresses in: any (re)allocation
  // invalidates them (decode.cpp checks the generation before a replay).
  ++ctx->generation;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    return fail(DFK_ERR_NOMEM, std::string("cudaMalloc(") +
                                   std::to_string(bytes) +
                                   "): " + cudaGetErrorString(e));
  }
  b.bytes = bytes;
  if (zero) DFK_CUDA(cudaMemsetAsync(b.p, 0, bytes, s));
  return DFK_OK;
}

std::string config_label(const dfk_config& c) {
  if (c.label[0]) return c.label;
  std::ostringstream o;
  if (c.variant == DFK_VARIANT_TWO_KERNEL) return "two_kernel_cublaslt";
  if (c.variant == DFK_VARIANT_FOUR_KERNEL) return "four_kernel_cublaslt";
  if (c.block_kernel) {
    if (c.dynamic_sched) o << "dyn" << c.chunk_kb << "_";
    if (c.dynamic_sched && c.s1_chunk_kb) o << "s1k" << c.s1_chunk_kb << "_";
    if (c.dynamic_sched && c.s1_tail > 0) o << "s1t" << c.s1_tail << "_";
    if (c.s1_split_k > 1) o << "sk" << c.s1_split_k << "_";
    o << "block_" << (c.s1_family == DFK_FAMILY_GEMV ? "gemv" : "tc") << "_st"
      << c.s1_stages << "_kbs" << c.kbs << "_c" << c.s1_ctas
      << (c.pdl ? "_pdl" : "");
    return o.str();
  }
  if (c.dynamic_sched) o << "dyn" << c.chunk_kb << "_";
  if (c.dynamic_sched && c.s1_chunk_kb) o << "s1k" << c.s1_chunk_kb << "_";
  if (c.s1_split_k > 1) o << "sk" << c.s1_split_k << "_";
  o << "fused_s1" << (c.s1_family == DFK_FAMILY_GEMV ? "gemv" : "tc") << "_st"
    << c.s1_stages << "_c" << c.s1_ctas << "_dn"
    << (c.down_family == DFK_FAMILY_GEMV ? "gemv" : "tc") << "_st"
    << c.down_stages << "_c" << c.down_ctas << "_kbs" << c.kbs
    << (c.pdl ? "_pdl" : "");
  return o.str();
}

namespace {

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// ---------------------------------------------------------------------------
// TMA descriptors (driver entry point fetched through the runtime so the
// library does not link libcuda directly).
// ---------------------------------------------------------------------------
// Stream memory operations (driver API; the host-buffer forward's side
// stream waits on / writes 32-bit device flags).
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
template <typename Fn>
Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<Fn>(p);
  return nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
  }
  return fn;
}

// 2-D bf16 tensor [rows x inner] with row stride `ld` elements; box
// 64 (inner) x box_rows, 128B swizzle; out-of-bounds reads are zero.
int get_tmap(dfk_context_s* ctx, const void* ptr, int64_t inner, int64_t rows,
             int64_t ld, int box_rows, CUtensorMap* out) {
  auto key = std::make_tuple(reinterpret_cast<uintptr_t>(ptr), inner, rows, ld,
                             box_rows);
  auto it = ctx->tmaps.find(key);
  if (it != ctx->tmaps.end()) {
    *out = it->second;
    return DFK_OK;
  }
  auto enc = tmap_encoder();
  if (!enc) return fail(DFK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner),
                        static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    return fail(DFK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" +
                                  std::to_string(static_cast<int>(r)) + ")");
  }
  if (ctx->tmaps.size() > 4096) ctx->tmaps.clear();
  ctx->tmaps.emplace(key, m);
  *out = m;
  return DFK_OK;
}

// 3-D view of a [rows x inner] bf16 activation for one-TMA-per-stage loads
// (StreamArgs::x3d): dims (64 K, rows, K blocks), the K-block dimension 128 B
// apart; box (64, box_rows, box_kb).  inner must be a multiple of 64.
int get_tmap3(dfk_context_s* ctx, const void* ptr, int64_t inner, int64_t rows,
              int64_t ld, int box_rows, int box_kb, CUtensorMap* out) {
  auto key = std::make_tuple(reinterpret_cast<uintptr_t>(ptr), inner, rows, ld,
                             box_rows | (box_kb << 16) | (1 << 30));
  auto it = ctx->tmaps.find(key);
  if (it != ctx->tmaps.end()) {
    *out = it->second;
    return DFK_OK;
  }
  auto enc = tmap_encoder();
  if (!enc) return fail(DFK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  cuuint64_t dims[3] = {64u, static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(inner / 64)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 2), 128u};
  cuuint32_t box[3] = {64u, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_kb)};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DFK_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed (" +
                                  std::to_string(static_cast<int>(r)) + ")");
  if (ctx->tmaps.size() > 4096) ctx->tmaps.clear();
  ctx->tmaps.emplace(key, m);
  *out = m;
  return DFK_OK;
}

// The stage-1 X map of a launch: 3-D (one TMA per ring stage) when a->x3d.
int get_xmap(dfk_context_s* ctx, const StreamArgs& a, const void* x, int64_t dm, int64_t rows,
             int64_t ld, CUtensorMap* out) {
  if (a.x3d) return get_tmap3(ctx, x, dm, rows, ld, a.xrows, a.kbs, out);
  return get_tmap(ctx, x, dm, rows, ld, a.xrows, out);
}

int max_stages(dfk_context_s* ctx, int n_pad, int kbs, int split_k = 1, int a2_tma = 0) {
  const int avail = ctx->max_smem_optin - 1024 - 1024 - split_red_bytes(n_pad, split_k) -
                    a2_stage_bytes(n_pad, a2_tma);
  int s = std::min(avail / stream_stage_bytes(n_pad, kbs), 32);
  while (s > 2 && stream_smem_bytes(n_pad, s, kbs, split_k, a2_tma) > ctx->max_smem_optin) --s;
  return s;
}

// Bigger ring stages stream faster (tools/stream_probe.cu, profiles/): take
// the largest stage (up to 4 x 16 KiB weight blocks) that still leaves 3
// slots in shared memory.
int pick_kbs(dfk_context_s* ctx, int n_pad, int requested, int split_k = 1,
             int a2_tma = 0) {
  if (requested > 0) return std::min(requested, 4);
  for (int kbs = 4; kbs > 1; --kbs)
    if (max_stages(ctx, n_pad, kbs, split_k, a2_tma) >= 3) return kbs;
  return 1;
}

// Persistent stage-1 grid: as many CTAs as keep every CTA at the same tile
// count (224 tiles on 148 SMs -> 112 CTAs x 2 tiles): per-SM bandwidth
// scales with bytes in flight, so fewer, evenly loaded CTAs beat a ragged
// last wave.
int balanced_grid(int tiles, int sms) {
  const int waves = (tiles + sms - 1) / sms;
  return (tiles + waves - 1) / waves;
}

int gemv_nb(int64_t b) {
  if (b <= 1) return 1;
  if (b <= 2) return 2;
  if (b <= 4) return 4;
  return 8;
}

// Makes an activation operand TMA-legal (16-byte aligned base, row stride a
// multiple of 16 bytes); copies into `pad` when it is not.
int tma_operand(dfk_context_s* ctx, const void* p, int64_t rows, int64_t cols,
                int64_t ld, DeviceBuf& pad, const void** out, int64_t* out_ld) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld % 8) == 0) {
    *out = p;
    *out_ld = ld;
    return DFK_OK;
  }
  const int64_t ld2 = round_up(cols, 8);
  DFK_TRY(ensure_buf(ctx, pad, static_cast<size_t>(rows * ld2 * 2), false,
                     ctx->stream));
  DFK_CUDA(launch_pad_rows(static_cast<const __nv_bfloat16*>(p), rows, cols,
                           ld, static_cast<__nv_bfloat16*>(pad.p), ld2,
                           ctx->stream));
  ctx->launches++;
  *out = pad.p;
  *out_ld = ld2;
  return DFK_OK;
}

int check_batch(int64_t B) {
  if (B < 1) {
    return fail(DFK_ERR_SHAPE, "batch must be >= 1, got " + std::to_string(B));
  }
  return DFK_OK;
}

// ---------------------------------------------------------------------------
// Fused launchers.
// ---------------------------------------------------------------------------
struct Launch {
  bool tc;
  int64_t chunk;  // batch rows per launch
};

Launch launch_shape(int family) {
  const bool tc = family != DFK_FAMILY_GEMV;
  return {tc, tc ? 256 : 8};
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Experiment / tuning overrides, read once per process (DESIGN.md §7b lists
// them); the defaults are the measured optima.
struct Knobs {
  int a2_tma = env_int("DFK_A2_TMA", 1);            // A2 by one TMA store per tile
  int xrows8 = env_int("DFK_XROWS8", 1);            // 8-row activation boxes at B <= 8
  int nacc = env_int("DFK_NACC", 1);                // independent accumulator chains
  int pf_kb = env_int("DFK_PF_KB", -1);             // K blocks prefetched to L2 before PDL wait (-1 = auto)
  int trace_s0 = env_int("DFK_TRACE_S0", 24);       // first ring stage the trace records
  int dn_chunk = env_int("DFK_DN_CHUNK", 0);        // down K chunk (0 = heuristic)
  int grid = env_int("DFK_GRID", 0);                // block-kernel CTAs (0 = heuristic)
  int host_stagek = env_int("DFK_HOST_STAGEK", 0);  // host path: staging kernel
  int red_v4 = env_int("DFK_RED_V4", 1);            // 0 off, 1 small shards, 2 always
  int trace_rel = env_int("DFK_TRACE_REL", 0);      // trace: stage release / MMA issue times
  int lt_tune = env_int("DFK_LT_TUNE", 1);          // autotune the cuBLASLt comparator's algorithm
  int bal = env_int("DFK_BAL", 0);                  // balanced stream-K: 0 off, 1 small shards, 2 always
  int x3d = env_int("DFK_X3D", 1);                  // one 3-D X / A2 TMA per ring stage
  int y_direct = env_int("DFK_Y_DIRECT", 1);        // block kernel red.adds into fp32 Y itself
  int s1_tail = env_int("DFK_S1_TAIL", 0);          // overrides dfk_config.s1_tail (A/B runs)
  int s1_whole = env_int("DFK_S1_WHOLE", 0);        // whole stage-1 tiles first (0 = grid)
};

const Knobs& knobs() {
  static const Knobs k;
  return k;
}

int fill_dynamic(dfk_context_s* ctx, dfk_weights_s* w, const dfk_config& cfg,
                 int grid, StreamArgs* a, bool down_only = false, bool block = false) {
  if (!cfg.dynamic_sched) return DFK_OK;
  DFK_TRY(ensure_buf(ctx, ctx->sched, 64, true, ctx->stream));
  a->dynamic = 1;
  a->sched = static_cast<int*>(ctx->sched.p);
  // 32-K-block (512 KiB) down chunks measured best on full-size weights; a
  // shard with few down tiles gets smaller chunks so that there are at least
  // ~1.5 pieces per CTA -- but never under max(4, N/4) K blocks: every piece
  // ends in 128 x N fp32 red.adds, which at large N cost more than the
  // extra balance buys (tools/tp_shard_sweep.py, profiles/r1b_tp_shards.md).
  // At N <= 16 smaller chunks (~16 K blocks, a divisor of the K-block count
  // when one exists) balance the drain better: -1 to -2 % at B = 1..16; at
  // N >= 32, 24 K blocks (sweep 16..36 on the full grid: -2 to -5 % against
  // 32 once the epilogues became straight-line code, profiles/r1c_epilogue.md).
  // The down kernel on its own (dfk_down, no stage-1 dependency): 32 K
  // blocks at every N (sweep 8..56 on all SMs: -11 to -18 % against 16/24,
  // profiles/r1c_epilogue.md).
  int chunk = std::min(w->dn_kblocks, a->n_pad <= 16 || down_only ? 32 : 24);
  if (a->n_pad <= 16 && w->dn_kblocks > 16 && !down_only) {
    chunk = 16;
    for (int c = 16; c >= 12; --c)
      if (w->dn_kblocks % c == 0) {
        chunk = c;
        break;
      }
  }
  const int64_t pieces = static_cast<int64_t>(w->dn_tiles) *
                         ((w->dn_kblocks + chunk - 1) / chunk);
  if (pieces * 2 < 3LL * grid) {
    // ~one down piece per CTA (every piece ends in 128 x N fp32 red.adds:
    // more, smaller pieces lose at N >= 16; sweep of the TP shards,
    // profiles/r1b_tp_shards.md)
    const int per_tile = std::max(
        1, static_cast<int>(std::lround(static_cast<double>(grid) / w->dn_tiles)));
    chunk = std::max(std::min(4, w->dn_kblocks), (w->dn_kblocks + per_tile - 1) / per_tile);
  }
  // Block kernel at N <= 32: the stage-1 split below (about two stage-1
  // pieces per CTA) goes with 16-K-block down chunks.
  const int s1_per_tile = block && a->n_pad <= 32 && a->split_k <= 1
                              ? std::min(4, std::max(1, static_cast<int>(std::lround(
                                                            2.0 * grid / w->s1_tiles))))
                              : 1;
  if (s1_per_tile > 1) chunk = std::min(16, w->dn_kblocks);
  if (knobs().dn_chunk > 0) chunk = std::min(knobs().dn_chunk, w->dn_kblocks);
  a->chunk_kb = cfg.chunk_kb > 0 ? cfg.chunk_kb : chunk;
  // Vector partial-sum reductions on shards with fewer stage-1 tiles than
  // CTAs (latency-bound epilogue chains); neutral on full shards.
  a->red_v4 = knobs().red_v4 >= 2 || (knobs().red_v4 == 1 && w->s1_tiles < grid);
  // Stage-1 stream-K: a shard with fewer stage-1 tiles than CTAs splits
  // every tile's K range so that ~1.5 x grid stage-1 pieces keep all SMs
  // streaming (s1_chunk_kb > 0 forces a chunk; >= K blocks = whole tiles).
  int s1c = w->s1_kblocks;
  if (cfg.s1_chunk_kb > 0) {
    s1c = std::min(cfg.s1_chunk_kb, w->s1_kblocks);
  } else if (s1_per_tile > 1) {
    // Block kernel at N <= 32 on shards with up to ~1.3 x grid stage-1
    // tiles (TP shards): split each tile's K range into round(2 x grid /
    // tiles) pieces, at most 4, each >= 16 K blocks -- the fit to the sweep
    // over the TP shards of BASELINE configs 2-5 at TP 2/4/8 and B = 1..32
    // (tools/chunk_sweep.py, profiles/r2_chunk_sweep.md): mean gap to the
    // best swept configuration 5.8 % -> 2.3 % at N <= 16, 5.8 % -> 3.7 % at
    // N = 32.
    s1c = std::max(std::min(16, w->s1_kblocks),
                   (w->s1_kblocks + s1_per_tile - 1) / s1_per_tile);
  } else if (w->s1_tiles < grid) {
    // About 0.87 stage-1 pieces per CTA (rounded to whole pieces per tile),
    // each >= 256 KiB (16 K blocks): the best of chunk-size sweeps over the
    // TP shards of SURVEY §8e at B = 1, 16, 64 (profiles/r1b_tp_shards.md).
    const int per_tile =
        std::max(1, static_cast<int>(std::lround(0.87 * grid / w->s1_tiles)));
    const int min_kb = 16;
    s1c = std::max(std::min(min_kb, w->s1_kblocks),
                   (w->s1_kblocks + per_tile - 1) / per_tile);
  }
  a->s1_chunk = s1c;
  a->s1_tail = 0;
  a->s1_whole = 0;
  // (0 = auto: 3 parts at N >= 32 -- B = 32: Llama-8B -3 %, Qwen2.5-32B TP2
  // -8 %, Llama-70B TP2 -3 %; B = 64: -1 / -7 / -2 %, Qwen2.5-7B +1 %;
  // neutral at N <= 16, profiles/r2_tail_split.md; 1 = off)
  const int tail = knobs().s1_tail > 0 ? knobs().s1_tail
                   : cfg.s1_tail > 0  ? cfg.s1_tail
                   : a->n_pad >= 32   ? 3
                                      : 0;
  if (block && s1c >= w->s1_kblocks && tail > 1 && w->s1_tiles > grid && a->split_k <= 1) {
    a->s1_tail = std::min(tail, w->s1_kblocks);
    a->s1_whole = knobs().s1_whole > 0 ? std::min(knobs().s1_whole, w->s1_tiles) : grid;
  }
  if (s1c < w->s1_kblocks || a->s1_tail > 1) {
    DFK_TRY(ensure_buf(ctx, ctx->s1acc,
                       static_cast<size_t>(w->s1_tiles) * a->n_pad * kBlockRows * 4,
                       true, ctx->stream));
    DFK_TRY(ensure_buf(ctx, ctx->s1cnt, static_cast<size_t>(w->s1_tiles) * 4, true,
                       ctx->stream));
    a->s1acc = static_cast<float*>(ctx->s1acc.p);
    a->s1cnt = static_cast<int*>(ctx->s1cnt.p);
  }
  return DFK_OK;
}

// Stage-1 split-K (cluster of `split` CTAs per tile, DSMEM reduction): only
// for the tcgen05 family, the static plan, N <= 64 (reduction buffer) and a
// K-block count divisible by the split.  Returns 1 when not applicable.
int effective_split(const dfk_config& cfg, const dfk_weights_s* w, int64_t nb,
                    int dyn_block_sms = 0) {
  const int sk = cfg.s1_split_k;
  if (sk <= 1 || cfg.s1_family == DFK_FAMILY_GEMV) return 1;
  // Dynamic block kernel: every stage-1 tile's K parts are the first pieces
  // of one cluster, so all t1 x sk of them must fit in one wave.
  if (cfg.dynamic_sched && (dyn_block_sms <= 0 || w->s1_tiles * sk > dyn_block_sms)) return 1;
  if (sk > 8 || w->s1_kblocks % sk != 0) return 1;
  if (split_red_bytes(static_cast<int>(round_up(nb, 16)), sk) > 64 * 1024) return 1;
  return sk;
}

// Clusters of `split` CTAs that can be co-resident for this launch shape.
int cluster_cap(int mode, const StreamArgs& a) {
  if (a.split_k <= 1) return 1 << 30;
  const int smem = stream_smem_bytes(a.n_pad, a.stages, a.kbs, a.split_k, a.a2_tma);
  return stream_max_clusters(mode, a.split_k, smem);
}

// Stage-1 A2 through one TMA store per tile: tcgen05 family, no cluster
// split, and an A2 the tensor map can address (16-byte aligned base/rows).
int want_a2_tma(const dfk_config& cfg, bool tc, int split_k, const void* a2, int64_t a2_ld) {
  return tc && split_k <= 1 && knobs().a2_tma &&
         (reinterpret_cast<uintptr_t>(a2) & 15) == 0 && (a2_ld * 2) % 16 == 0 &&
         cfg.mutant == 0;
}

// Ring geometry for one launch: stage size (kbs) and depth.
void fill_common(dfk_context_s* ctx, dfk_weights_s* w, int64_t nb, bool tc,
                 int stages_req, const dfk_config& cfg, StreamArgs* a) {
  const int n_pad = tc ? static_cast<int>(round_up(nb, 16)) : 8;
  a->w1 = w->s1_pack;
  a->t1 = w->s1_tiles;
  a->kb1 = w->s1_kblocks;
  a->w2 = w->dn_pack;
  a->t2 = w->dn_tiles;
  a->kb2 = w->dn_kblocks;
  a->B = static_cast<int>(nb);
  a->n_pad = n_pad;
  // Activation rows a TMA box brings in: at B <= 8 only the first 8-row
  // swizzle atom of the N=16 operand (rows 8-15 of the smem tile are left
  // as they are: they only feed accumulator columns >= B, never stored).
  a->xrows = (tc && nb <= 8 && knobs().xrows8) ? 8 : n_pad;
  const int sk = a->split_k > 1 ? a->split_k : 1;
  a->kbs = pick_kbs(ctx, n_pad, cfg.kbs, sk, a->a2_tma);
  a->trace = ctx->trace;
  if (a->trace) {
    a->trace_s0 = knobs().trace_s0;
    a->trace_rel = knobs().trace_rel;
  }
  a->tp_error = ctx->err_dev;
  // (the GEMV family's 8-row boxes already pack 8 x 128 B per K block)
  a->x3d = knobs().x3d && w->d_model % 64 == 0 && (tc || a->xrows == n_pad);
  a->a3d = knobs().x3d && w->d_ff % 64 == 0 && (tc || a->xrows == n_pad);
  // Independent accumulator chains (tcgen05): 1, 2 or 4, as TMEM allows.
  a->nacc = 1;
  if (tc && sk == 1) {
    int n = std::max(1, std::min(knobs().nacc, 256 / n_pad));
    a->nacc = n >= 4 ? 4 : n >= 2 ? 2 : 1;
  }
  // 12 K blocks (192 KiB) of L2 prefetch: the measured optimum on full
  // shards (A/B sweep 0..60, profiles/r1b_tuning.md); 8 on shards with fewer
  // stage-1 tiles than SMs (-0.2 to -0.5 us on the TP8 shards once the down
  // tail got shorter, profiles/r2_tail_split.md).
  a->pf_kb = knobs().pf_kb >= 0 ? knobs().pf_kb : (w->s1_tiles < ctx->sm_count ? 8 : 12);
  const int ms = std::max(2, max_stages(ctx, n_pad, a->kbs, sk, a->a2_tma));
  a->stages = stages_req > 0 ? std::max(2, std::min(stages_req, ms)) : ms;
}

int ensure_down_workspace(dfk_context_s* ctx, dfk_weights_s* w, int64_t rows) {
  DFK_TRY(ensure_buf(ctx, ctx->yacc,
                     static_cast<size_t>(rows) * w->dn_tiles * kDownCols *
                         sizeof(float),
                     true, ctx->stream));
  return ensure_buf(ctx, ctx->counters, static_cast<size_t>(w->dn_tiles) * 4, true,
                    ctx->stream);
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const auto pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
  return pa < pb + nb && pb < pa + na;
}

// True for memory of a device (cudaMalloc / pool), false for host-mapped,
// managed or unknown pointers.
bool device_memory(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice;
}

void fill_down(dfk_context_s* ctx, dfk_weights_s* w, void* y, int64_t b0,
               int64_t y_ld, bool y_bf16, StreamArgs* a) {
  a->yacc = static_cast<float*>(ctx->yacc.p);
  a->yacc_ld = w->dn_tiles * kDownCols;
  a->counters = static_cast<int*>(ctx->counters.p);
  a->y = y_bf16 ? static_cast<void*>(static_cast<__nv_bfloat16*>(y) + b0 * y_ld)
                : static_cast<void*>(static_cast<float*>(y) + b0 * y_ld);
  a->y_ld = y_ld;
  a->y_bf16 = y_bf16 ? 1 : 0;
  a->y_vec4 = !y_bf16 && y_ld % 4 == 0 && (reinterpret_cast<uintptr_t>(a->y) & 15) == 0;
  a->out_cols = static_cast<int>(w->d_model);
}

int stage1_fused(dfk_context_s* ctx, dfk_weights_s* w, const void* x,
                 int64_t B, __nv_bfloat16* a2, int64_t a2_ld,
                 const dfk_config& cfg) {
  const Launch L = launch_shape(cfg.s1_family);
  const void* xp;
  int64_t x_ld;
  DFK_TRY(tma_operand(ctx, x, B, w->d_model, w->d_model, ctx->xpad, &xp, &x_ld));
  for (int64_t b0 = 0; b0 < B; b0 += L.chunk) {
    const int64_t nb = std::min(L.chunk, B - b0);
    StreamArgs a = {};
    a.split_k = effective_split(cfg, w, nb);
    a.a2_tma = want_a2_tma(cfg, L.tc, a.split_k, a2 + b0 * a2_ld, a2_ld);
    fill_common(ctx, w, nb, L.tc, cfg.s1_stages, cfg, &a);
    a.a3d = 0;  // stage 1 alone never loads A2
    CUtensorMap tm, am;
    DFK_TRY(get_tmap(ctx, static_cast<const __nv_bfloat16*>(xp) + b0 * x_ld,
                     w->d_model, nb, x_ld, a.xrows, &tm));
    am = tm;
    if (a.x3d)
      DFK_TRY(get_xmap(ctx, a, static_cast<const __nv_bfloat16*>(xp) + b0 * x_ld, w->d_model, nb,
                       x_ld, &tm));
    if (a.a2_tma)
      DFK_TRY(get_tmap(ctx, a2 + b0 * a2_ld, w->d_ff, nb, a2_ld, a.xrows, &am));
    a.a2 = a2 + b0 * a2_ld;
    a.a2_ld = a2_ld;
    a.cols_valid = static_cast<int>(w->d_ff);
    a.mutant = cfg.mutant;
    if (cfg.mutant == 2) {
      DFK_TRY(ensure_buf(ctx, ctx->mat_scratch, static_cast<size_t>(nb * w->d_ff) * 4, false,
                         ctx->stream));
      a.mat_scratch = static_cast<float*>(ctx->mat_scratch.p);
    }
    const int sk = a.split_k;
    // Clusters of sk CTAs; as many clusters as keep every cluster at the
    // same tile count, never more than can be co-resident.
    int grid;
    if (cfg.dynamic_sched && sk == 1) {
      // Dynamic: whole tiles on the balanced grid, or -- a shard with fewer
      // tiles than 7/8 of the SMs -- stream-K pieces over 7/8 of the SMs.
      grid = cfg.s1_ctas > 0 ? cfg.s1_ctas
             : w->s1_tiles < ctx->sm_count * 7 / 8
                 ? ctx->sm_count * 7 / 8
                 : balanced_grid(w->s1_tiles, ctx->sm_count);
      grid = std::max(1, std::min(grid, ctx->sm_count));
      DFK_TRY(fill_dynamic(ctx, w, cfg, grid, &a));
      const int per_tile = (w->s1_kblocks + a.s1_chunk - 1) / a.s1_chunk;
      grid = std::min(grid, w->s1_tiles * per_tile);
    } else {
      int clusters = cfg.s1_ctas > 0 ? cfg.s1_ctas / sk
                                     : balanced_grid(w->s1_tiles, ctx->sm_count / sk);
      clusters =
          std::max(1, std::min({clusters, w->s1_tiles, cluster_cap(kModeStage1, a)}));
      grid = clusters * sk;
    }
    cudaError_t e = launch_stream(kModeStage1, L.tc, gemv_nb(nb), tm, am, a,
                                  grid, cfg.pdl != 0, ctx->stream);
    if (e != cudaSuccess)
      return fail(DFK_ERR_CUDA, std::string("stage-1 launch: ") +
                                    cudaGetErrorString(e));
    ctx->launches++;
  }
  return DFK_OK;
}

int down_fused(dfk_context_s* ctx, dfk_weights_s* w, const void* a2,
               int64_t a2_ld, int64_t B, void* y, int64_t y_ld, bool y_bf16,
               const dfk_config& cfg) {
  const Launch L = launch_shape(cfg.down_family);
  const void* ap;
  int64_t a_ld;
  DFK_TRY(tma_operand(ctx, a2, B, w->d_ff, a2_ld, ctx->a2pad, &ap, &a_ld));
  DFK_TRY(ensure_down_workspace(ctx, w, std::min(L.chunk, B)));
  for (int64_t b0 = 0; b0 < B; b0 += L.chunk) {
    const int64_t nb = std::min(L.chunk, B - b0);
    StreamArgs a = {};
    fill_common(ctx, w, nb, L.tc, cfg.down_stages, cfg, &a);
    CUtensorMap tm;
    DFK_TRY(get_tmap(ctx, static_cast<const __nv_bfloat16*>(ap) + b0 * a_ld,
                     w->d_ff, nb, a_ld, a.xrows, &tm));
    fill_down(ctx, w, y, b0, y_ld, y_bf16, &a);
    CUtensorMap a3m = tm;
    if (a.a3d)
      DFK_TRY(get_tmap3(ctx, static_cast<const __nv_bfloat16*>(ap) + b0 * a_ld, w->d_ff, nb, a_ld,
                        a.xrows, a.kbs, &a3m));
    const int64_t U = static_cast<int64_t>(w->dn_tiles) * w->dn_kblocks;
    // Default: every SM (the dynamic queue balances; 3/4 of the SMs, the
    // first session's optimum for the static plan, is 11-18 % slower now,
    // profiles/r1c_epilogue.md).
    int64_t grid = cfg.down_ctas > 0 ? cfg.down_ctas : ctx->sm_count;
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, U));
    DFK_TRY(fill_dynamic(ctx, w, cfg, static_cast<int>(grid), &a, true));
    // Direct Y as in the block kernel (every CTA zeroes its slice after the
    // PDL wait; the first reduction comes a whole first piece later).
    // (not when Y overlaps the A2 operand: Y is zeroed while A2 is read; and
    // only when every CTA is resident -- a CTA's first reduction waits for
    // all slices, so a caller's down_ctas beyond the SM count would hang)
    if (a.dynamic && knobs().y_direct && !y_bf16 && a.y_vec4 && w->d_model % 4 == 0 &&
        grid <= ctx->sm_count &&
        !overlaps(ap, static_cast<size_t>(B * a_ld) * 2, y,
                  static_cast<size_t>(B * y_ld) * 4) &&
        device_memory(a.y))
      a.y_direct = 1;
    cudaError_t e = launch_stream(kModeDown, L.tc, gemv_nb(nb), tm, tm, a,
                                  static_cast<int>(grid), cfg.pdl != 0,
                                  ctx->stream, &a3m);
    if (e != cudaSuccess)
      return fail(DFK_ERR_CUDA,
                  std::string("down launch: ") + cudaGetErrorString(e));
    ctx->launches++;
  }
  return DFK_OK;
}

// Work plan of the block kernel (see StreamArgs): stage-1 tiles round-robin,
// then down units in two groups so that no CTA waits long on a stage-1 tile
// that is still being computed.  Group A (K blocks whose stage-1 tile lies in
// an early round-robin wave) goes to the CTAs with one tile fewer, group B
// (last wave) is shared by everyone with byte-balanced budgets.
void block_plan(int G, const dfk_weights_s* w, StreamArgs* a) {
  // With split-K, stage-1 tiles go round-robin over Q = G / split clusters
  // and every CTA of a cluster owns kb1 / split K blocks of each tile.
  const int split = a->split_k > 1 ? a->split_k : 1;
  const int Q = G / split;
  const int T1 = w->s1_tiles, kb1c = w->s1_kblocks / split;
  const int t2 = w->dn_tiles, kb2 = w->dn_kblocks;
  const int q = T1 / Q, rt = T1 % Q;
  const int r = rt * split;  // heavy CTAs (in the first rt clusters)
  a->bp_r = r;
  a->bp_L = G - r;
  if (rt > 0) {
    a->bp_nA = q * Q;
    a->bp_nB = rt;
    a->bp_kB0 = q * Q;
  } else {  // every cluster owns q tiles: no early group
    a->bp_nA = 0;
    a->bp_nB = kb2;
    a->bp_kB0 = 0;
  }
  const int64_t L = a->bp_L;
  const int64_t A = static_cast<int64_t>(t2) * a->bp_nA;
  const int64_t Bn = static_cast<int64_t>(t2) * a->bp_nB;
  // Group B: uniform.
  a->bp_bl = Bn / G;
  a->bp_rB = Bn - a->bp_bl * G;
  // Group A: total per CTA balanced, i.e. light ranks take one stage-1 part
  // (kb1c K blocks) more.
  const int64_t WT = static_cast<int64_t>(T1) * kb1c * split +
                     static_cast<int64_t>(t2) * kb2;
  int64_t ah = (WT - static_cast<int64_t>(G) * (q + 1) * kb1c - Bn) / G;
  if (ah < 0 || r == 0) ah = 0;
  if (ah * r > A) ah = r > 0 ? A / r : 0;
  const int64_t al = (A - ah * r) / L;
  a->bp_ah = ah;
  a->bp_al = al;
  a->bp_rA = A - al * L - ah * r;
}

// The whole block in one persistent launch per batch chunk (kModeBlock).
// Every CTA must be co-resident (down pieces spin on stage-1 tile flags), so
// the grid never exceeds the SM count.
int block_fused(dfk_context_s* ctx, dfk_weights_s* w, const void* x, int64_t B,
                __nv_bfloat16* a2, int64_t a2_ld, void* y, int64_t y_ld,
                bool y_bf16, const dfk_config& cfg, const StreamArgs* tp) {
  const Launch L = launch_shape(cfg.s1_family);
  const void* xp;
  int64_t x_ld;
  DFK_TRY(tma_operand(ctx, x, B, w->d_model, w->d_model, ctx->xpad, &xp, &x_ld));
  DFK_TRY(ensure_down_workspace(ctx, w, std::min(L.chunk, B)));
  DFK_TRY(ensure_buf(ctx, ctx->flags, static_cast<size_t>(w->s1_tiles) * 4, true,
                     ctx->stream));
  for (int64_t b0 = 0; b0 < B; b0 += L.chunk) {
    const int64_t nb = std::min(L.chunk, B - b0);
    StreamArgs a = {};
    a.split_k = effective_split(cfg, w, nb, ctx->sm_count);
    a.a2_tma = want_a2_tma(cfg, L.tc, a.split_k, a2 + b0 * a2_ld, a2_ld);
    fill_common(ctx, w, nb, L.tc, cfg.s1_stages, cfg, &a);
    CUtensorMap xm, am;
    DFK_TRY(get_xmap(ctx, a, static_cast<const __nv_bfloat16*>(xp) + b0 * x_ld, w->d_model, nb,
                     x_ld, &xm));
    DFK_TRY(get_tmap(ctx, a2 + b0 * a2_ld, w->d_ff, nb, a2_ld, a.xrows, &am));
    CUtensorMap a3m = am;
    if (a.a3d)
      DFK_TRY(get_tmap3(ctx, a2 + b0 * a2_ld, w->d_ff, nb, a2_ld, a.xrows, a.kbs, &a3m));
    a.a2 = a2 + b0 * a2_ld;
    a.a2_ld = a2_ld;
    a.cols_valid = static_cast<int>(w->d_ff);
    fill_down(ctx, w, y, b0, y_ld, y_bf16, &a);
    if (tp) {  // fused TP all-reduce (tp.cpp): peer workspaces and outputs
      a.tp_rank = tp->tp_rank;
      a.tp_size = tp->tp_size;
      a.tp_total_kb = tp->tp_total_kb;
      for (int r = 0; r < kMaxTp; ++r) {
        a.tp_yacc[r] = tp->tp_yacc[r];
        a.tp_cnt[r] = tp->tp_cnt[r];
        a.tp_done[r] = tp->tp_done[r];
        // the chunk's rows of every rank's Y (GEMV family: 8-row chunks)
        a.tp_y[r] = tp->tp_y[r] ? tp->tp_y[r] + b0 * y_ld : nullptr;
      }
      a.yacc_ld = tp->yacc_ld;
      a.tp_late_trigger = ctx->tp_colocated ? 1 : 0;
    }
    if (ctx->pend_x_ready && b0 == 0 && B <= L.chunk) {  // host-buffer X flags
      a.x_ready = ctx->pend_x_ready;
      a.x_free = ctx->pend_x_free;
      a.y_done = ctx->pend_y_done;
      a.x_seq = ctx->pend_x_seq;
    }
    a.flags = static_cast<unsigned*>(ctx->flags.p);
    if (++ctx->epoch == 0) ++ctx->epoch;
    a.epoch = ctx->epoch;
    a.mutant = cfg.mutant;
    if (cfg.mutant == 2) {
      DFK_TRY(ensure_buf(ctx, ctx->mat_scratch, static_cast<size_t>(nb * w->d_ff) * 4, false,
                         ctx->stream));
      a.mat_scratch = static_cast<float*>(ctx->mat_scratch.p);
    }
    // Dynamic: 7/8 of the SMs at N <= 16 (the idle eighth starts the next
    // PDL launch's weight stream early; measured optimum, profiles/), every
    // SM at N >= 32 on shards with a full stage-1 wave (-2 to -3 % at
    // B = 32/64, profiles/r1c_epilogue.md).  Static: the balanced stage-1
    // grid but at least 3/4 of the SMs (the down work needs the CTAs even
    // when the shard has few stage-1 tiles).  Never more CTAs than SMs or
    // resident clusters: down pieces spin on other CTAs' stage-1 flags.
    const bool full = a.n_pad > 16 && w->s1_tiles >= ctx->sm_count;
    int grid = cfg.s1_ctas > 0 ? cfg.s1_ctas
               : cfg.dynamic_sched
                   ? (full ? ctx->sm_count : ctx->sm_count * 7 / 8)
                   : std::max(balanced_grid(w->s1_tiles, ctx->sm_count),
                              ctx->sm_count * 3 / 4);
    if (knobs().grid > 0 && cfg.s1_ctas <= 0) grid = knobs().grid;
    grid = std::max(1, std::min(grid, ctx->sm_count));
    // Ranks sharing this GPU (emulation): every rank's launch must fit
    // beside the others' (they wait for each other's contributions).
    if (tp && ctx->tp_colocated) grid = std::max(1, std::min(grid, ctx->sm_count / tp->tp_size));
    grid = std::min(grid / a.split_k, cluster_cap(kModeBlock, a)) * a.split_k;
    grid = std::max(grid, a.split_k);
    if (cfg.dynamic_sched && a.split_k > 1 && w->s1_tiles * a.split_k > grid) {
      // (the 7/8 grid rounded to clusters can fall below t1 x sk)
      grid = std::min(ctx->sm_count / a.split_k, cluster_cap(kModeBlock, a)) * a.split_k;
      if (w->s1_tiles * a.split_k > grid)
        return fail(DFK_ERR_INVALID, "dynamic split-K: stage-1 parts exceed one wave");
    }
    block_plan(grid, w, &a);
    if (a.split_k == 1 || cfg.dynamic_sched)
      DFK_TRY(fill_dynamic(ctx, w, cfg, grid, &a, false, true));
    if (a.dynamic && a.split_k > 1) a.s1_chunk = w->s1_kblocks;  // K split by the cluster
    if (a.dynamic && (knobs().bal >= 2 || (knobs().bal == 1 && w->s1_tiles < grid))) {
      // balanced stream-K pieces: partial stage-1 tiles need the workspace
      a.bal = 1;
      a.red_v4 = knobs().red_v4 >= 1;
      DFK_TRY(ensure_buf(ctx, ctx->s1acc,
                         static_cast<size_t>(w->s1_tiles) * a.n_pad * kBlockRows * 4, true,
                         ctx->stream));
      DFK_TRY(ensure_buf(ctx, ctx->s1cnt, static_cast<size_t>(w->s1_tiles) * 4, true,
                         ctx->stream));
      a.s1acc = static_cast<float*>(ctx->s1acc.p);
      a.s1cnt = static_cast<int*>(ctx->s1cnt.p);
    }
    // Direct Y (stream_kernels.cuh): fp32 Y in this GPU's memory with whole
    // 16-byte row groups; not under the fused TP all-reduce (its own tile
    // owners) nor for Y in mapped host memory (no PCIe reductions).
    // Nor when Y overlaps X: Y is zeroed while X is still being loaded.
    if (a.dynamic && !tp && knobs().y_direct && !y_bf16 && a.y_vec4 &&
        w->d_model % 4 == 0 &&
        !overlaps(xp, static_cast<size_t>(B * x_ld) * 2, y,
                  static_cast<size_t>(B * y_ld) * 4) &&
        device_memory(a.y))
      a.y_direct = 1;
    if (a.bp_rB < 0 || a.bp_rB > grid || a.bp_rA < 0 || a.bp_rA > grid)
      return fail(DFK_ERR_CUDA, "internal: block plan remainder out of range");
    cudaError_t e = launch_stream(kModeBlock, L.tc, gemv_nb(nb), xm, am, a,
                                  grid, cfg.pdl != 0, ctx->stream, &a3m);
    if (e != cudaSuccess)
      return fail(DFK_ERR_CUDA,
                  std::string("block launch: ") + cudaGetErrorString(e));
    ctx->launches++;
  }
  return DFK_OK;
}

// ---------------------------------------------------------------------------
// Unfused comparators on cuBLASLt (bf16 in, fp32 accumulate).
// ---------------------------------------------------------------------------
// K-major copies for cuBLASLt, built lazily from the packs (only the parts
// the registered set has: stage-only sets, dfk_weights_create).
int ensure_unfused_s1(dfk_context_s* ctx, dfk_weights_s* w) {
  if (w->cat_t) return DFK_OK;
  if (!w->s1_pack) return fail(DFK_ERR_INVALID, "weights registered without W_gate / W_up");
  const size_t cat_bytes = static_cast<size_t>(2 * w->d_ff * w->d_model) * 2;
  if (cudaMalloc(&w->cat_t, cat_bytes) != cudaSuccess) {
    w->cat_t = nullptr;
    return fail(DFK_ERR_NOMEM, "unfused comparator weights");
  }
  DFK_CUDA(launch_unpack_stage1(w->s1_pack, w->d_model, w->d_ff, w->s1_tiles,
                                w->s1_kblocks, w->cat_t, ctx->stream));
  return DFK_OK;
}

int ensure_unfused_dn(dfk_context_s* ctx, dfk_weights_s* w) {
  if (w->down_t) return DFK_OK;
  if (!w->dn_pack) return fail(DFK_ERR_INVALID, "weights registered without W_down");
  const size_t down_bytes = static_cast<size_t>(w->d_ff * w->d_model) * 2;
  if (cudaMalloc(&w->down_t, down_bytes) != cudaSuccess) {
    w->down_t = nullptr;
    return fail(DFK_ERR_NOMEM, "unfused comparator weights");
  }
  DFK_CUDA(launch_unpack_down(w->dn_pack, w->d_model, w->d_ff, w->dn_tiles,
                              w->dn_kblocks, w->down_t, ctx->stream));
  return DFK_OK;
}

// C[n x m] (row-major, ldc) = B[n x k] (row-major, ldb) * A[m x k]^T where A
// is K-major [m x k] (lda).  In cuBLAS column-major terms: C_cm[m x n] =
// op_T(A_cm[k x m]) * B_cm[k x n].
int lt_gemm(dfk_context_s* ctx, const __nv_bfloat16* A, int64_t lda,
            const __nv_bfloat16* Bm, int64_t ldb, void* C, int64_t ldc,
            bool c_bf16, int64_t m, int64_t n, int64_t k) {
  if (!ctx->lt) {
    if (cublasLtCreate(&ctx->lt) != CUBLAS_STATUS_SUCCESS)
      return fail(DFK_ERR_CUDA, "cublasLtCreate");
  }
  const size_t ws_bytes = 32u << 20;
  DFK_TRY(ensure_buf(ctx, ctx->lt_ws, ws_bytes, false, ctx->stream));
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  const cudaDataType_t ct = c_bf16 ? CUDA_R_16BF : CUDA_R_32F;
  cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
  cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, k, m, lda);
  cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, k, n, ldb);
  cublasLtMatrixLayoutCreate(&lc, ct, m, n, ldc);
  auto key = std::make_tuple(m, n, k, c_bf16 ? 1 : 0);
  auto it = ctx->lt_algos.find(key);
  cublasLtMatmulAlgo_t algo;
  if (it == ctx->lt_algos.end()) {
    cublasLtMatmulPreference_t pref = nullptr;
    cublasLtMatmulPreferenceCreate(&pref);
    size_t wsb = ws_bytes;
    cublasLtMatmulPreferenceSetAttribute(
        pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
    cublasLtMatmulHeuristicResult_t res[8];
    int got = 0;
    cublasStatus_t st = cublasLtMatmulAlgoGetHeuristic(
        ctx->lt, op, la, lb, lc, lc, pref, 8, res, &got);
    cublasLtMatmulPreferenceDestroy(pref);
    if (st != CUBLAS_STATUS_SUCCESS || got == 0) {
      cublasLtMatmulDescDestroy(op);
      cublasLtMatrixLayoutDestroy(la);
      cublasLtMatrixLayoutDestroy(lb);
      cublasLtMatrixLayoutDestroy(lc);
      return fail(DFK_ERR_CUDA, "cuBLASLt: no algorithm for the unfused GEMM");
    }
    // Autotune the comparator: time every returned algorithm on these
    // operands (1 warm-up + 5 calls each, events on the context stream)
    // and keep the fastest -- the heuristic's first pick is often a
    // split-K kernel far from the best on skinny (decode) GEMMs.  Not while
    // the stream is being captured.
    int best = 0;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ctx->stream, &cs);
    if (got > 1 && cs == cudaStreamCaptureStatusNone && knobs().lt_tune) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const float alpha = 1.f, beta = 0.f;
      float best_ms = 1e30f;
      for (int i = 0; i < got; ++i) {
        bool ok = true;
        for (int r = 0; r < 6 && ok; ++r) {
          if (r == 1) cudaEventRecord(e0, ctx->stream);
          ok = cublasLtMatmul(ctx->lt, op, &alpha, A, la, Bm, lb, &beta, C, lc, C, lc,
                              &res[i].algo, ctx->lt_ws.p, ws_bytes,
                              ctx->stream) == CUBLAS_STATUS_SUCCESS;
        }
        cudaEventRecord(e1, ctx->stream);
        if (cudaEventSynchronize(e1) != cudaSuccess) ok = false;
        float ms = 0.f;
        if (ok && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess && ms < best_ms) {
          best_ms = ms;
          best = i;
        }
      }
      cudaGetLastError();
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    algo = res[best].algo;
    ctx->lt_algos.emplace(key, algo);
  } else {
    algo = it->second;
  }
  const float alpha = 1.f, beta = 0.f;
  cublasStatus_t st =
      cublasLtMatmul(ctx->lt, op, &alpha, A, la, Bm, lb, &beta, C, lc, C, lc,
                     &algo, ctx->lt_ws.p, ws_bytes, ctx->stream);
  cublasLtMatmulDescDestroy(op);
  cublasLtMatrixLayoutDestroy(la);
  cublasLtMatrixLayoutDestroy(lb);
  cublasLtMatrixLayoutDestroy(lc);
  if (st != CUBLAS_STATUS_SUCCESS)
    return fail(DFK_ERR_CUDA, "cublasLtMatmul failed (" +
                                  std::to_string(static_cast<int>(st)) + ")");
  ctx->launches++;
  return DFK_OK;
}

// Stage 1 of the unfused layouts into a2 (ld = d_ff).
int stage1_unfused(dfk_context_s* ctx, dfk_weights_s* w, const void* x,
                   int64_t B, __nv_bfloat16* a2, int64_t a2_ld, int variant) {
  DFK_TRY(ensure_unfused_s1(ctx, w));
  const int64_t df = w->d_ff, dm = w->d_model;
  const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
  if (variant == DFK_VARIANT_TWO_KERNEL) {
    // Grouped GEMM into [A_gate | A_1] (gate columns first), then silu-mul.
    DFK_TRY(ensure_buf(ctx, ctx->concat, static_cast<size_t>(B * 2 * df) * 2, false,
                       ctx->stream));
    auto* cc = static_cast<__nv_bfloat16*>(ctx->concat.p);
    DFK_TRY(lt_gemm(ctx, w->cat_t, dm, xb, dm, cc, 2 * df, true, 2 * df, B, dm));
    DFK_CUDA(launch_silu_mul(cc, 2 * df, cc + df, 2 * df, a2, B, df,
                             ctx->stream));
    ctx->launches++;
    (void)a2_ld;
    return DFK_OK;
  }
  // Four-kernel: A_gate, A_1, A_silu materialised.
  const size_t bytes = static_cast<size_t>(B * df) * 2;
  DFK_TRY(ensure_buf(ctx, ctx->concat, bytes, false, ctx->stream));
  DFK_TRY(ensure_buf(ctx, ctx->tmp1, bytes, false, ctx->stream));
  DFK_TRY(ensure_buf(ctx, ctx->tmp2, bytes, false, ctx->stream));
  auto* agate = static_cast<__nv_bfloat16*>(ctx->concat.p);
  auto* a1 = static_cast<__nv_bfloat16*>(ctx->tmp1.p);
  auto* asilu = static_cast<__nv_bfloat16*>(ctx->tmp2.p);
  DFK_TRY(lt_gemm(ctx, w->cat_t, dm, xb, dm, agate, df, true, df, B, dm));
  DFK_TRY(lt_gemm(ctx, w->cat_t + df * dm, dm, xb, dm, a1, df, true, df, B, dm));
  DFK_CUDA(launch_silu(agate, asilu, B * df, ctx->stream));
  DFK_CUDA(launch_mul(a1, asilu, a2, B * df, ctx->stream));
  ctx->launches += 2;
  return DFK_OK;
}

int down_unfused(dfk_context_s* ctx, dfk_weights_s* w, const void* a2,
                 int64_t B, void* y, bool y_bf16) {
  DFK_TRY(ensure_unfused_dn(ctx, w));
  return lt_gemm(ctx, w->down_t, w->d_ff, static_cast<const __nv_bfloat16*>(a2),
                 w->d_ff, y, w->d_model, y_bf16, w->d_model, B, w->d_ff);
}

// need_s1 / need_dn: the call uses the stage-1 / down weights (a set
// registered for one stage only cannot run the other, dfk_weights_create).
int check_handles(dfk_context_s* ctx, dfk_weights_s* w, bool need_s1 = true,
                  bool need_dn = true) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  if (!w) return fail(DFK_ERR_INVALID, "null weights");
  if (w->ctx != ctx)
    return fail(DFK_ERR_INVALID, "weights belong to another context");
  if (need_s1 && !w->s1_pack)
    return fail(DFK_ERR_INVALID, "weights registered without W_gate / W_up (down-only set)");
  if (need_dn && !w->dn_pack)
    return fail(DFK_ERR_INVALID, "weights registered without W_down (stage-1-only set)");
  return use_device(ctx);
}



size_t dtype_size(int dt) { return dt == DFK_F64 ? 8 : dt == DFK_F32 ? 4 : 2; }

}  // namespace

// ---------------------------------------------------------------------------
// Config resolution.
// ---------------------------------------------------------------------------
void default_config(dfk_context_s* ctx, dfk_weights_s* w, int64_t B,
                    dfk_config* out) {
  (void)ctx;
  // The single persistent block kernel with dynamic scheduling: the fastest
  // configuration in the measured sweeps at every batch (profiles/).  At
  // B = 1 on the smallest shards (<= 40 stage-1 tiles, e.g. Llama-8B or
  // Qwen-7B at TP 8) the warp-GEMV consumers beat tcgen05 by 7-10 %
  // (profiles/r2_chunk_sweep.md); tcgen05 everywhere else.
  const bool gemv = B == 1 && w->s1_pack && w->dn_pack && w->s1_tiles <= 40;
  std::memset(out, 0, sizeof(*out));
  out->variant = DFK_VARIANT_FUSED;
  out->s1_family = gemv ? DFK_FAMILY_GEMV : DFK_FAMILY_TC;
  out->down_family = gemv ? DFK_FAMILY_GEMV : DFK_FAMILY_TC;
  out->s1_split_k = 1;
  out->block_kernel = 1;
  out->dynamic_sched = 1;
  out->pdl = 1;
  std::snprintf(out->label, sizeof(out->label), "%s",
                config_label(*out).c_str());
}

int resolve_config(dfk_context_s* ctx, dfk_weights_s* w, int64_t B,
                   const dfk_config* in, dfk_config* out) {
  if (in) {
    *out = *in;
  } else {
    std::lock_guard<std::mutex> lk(ctx->mu);
    auto it = ctx->chosen.find(std::make_tuple(B, w->d_model, w->d_ff));
    if (it != ctx->chosen.end()) {
      *out = it->second;
    } else {
      default_config(ctx, w, B, out);
    }
  }
  if (out->variant < 0 || out->variant > 2)
    return fail(DFK_ERR_INVALID,
                "unknown variant " + std::to_string(out->variant));
  if (out->s1_family == DFK_FAMILY_AUTO) out->s1_family = DFK_FAMILY_TC;
  if (out->down_family == DFK_FAMILY_AUTO) out->down_family = DFK_FAMILY_TC;
  if (out->s1_family < 0 || out->s1_family > 2 || out->down_family < 0 ||
      out->down_family > 2)
    return fail(DFK_ERR_INVALID, "unknown kernel family");
  if (out->s1_split_k < 1) out->s1_split_k = 1;
  if (out->s1_stages < 0 || out->down_stages < 0 || out->s1_ctas < 0 ||
      out->down_ctas < 0)
    return fail(DFK_ERR_INVALID, "negative launch parameter");
  return DFK_OK;
}

int forward_impl(dfk_context_s* ctx, dfk_weights_s* w, const void* x,
                 int64_t B, void* y, int y_dtype, const dfk_config* cfg_in) {
  DFK_TRY(check_handles(ctx, w));
  DFK_TRY(check_batch(B));
  if (!x || !y) return fail(DFK_ERR_INVALID, "null activation pointer");
  if (y_dtype != DFK_F32 && y_dtype != DFK_BF16)
    return fail(DFK_ERR_INVALID, "y_dtype must be F32 or BF16");
  dfk_config cfg;
  DFK_TRY(resolve_config(ctx, w, B, cfg_in, &cfg));
  const int64_t a2_ld = round_up(w->d_ff, 8);
  DFK_TRY(ensure_buf(ctx, ctx->a2, static_cast<size_t>(B * a2_ld) * 2, false,
                     ctx->stream));
  auto* a2 = static_cast<__nv_bfloat16*>(ctx->a2.p);
  if (cfg.variant == DFK_VARIANT_FUSED && cfg.block_kernel) {
    return block_fused(ctx, w, x, B, a2, a2_ld, y, w->d_model,
                       y_dtype == DFK_BF16, cfg, nullptr);
  }
  if (cfg.variant == DFK_VARIANT_FUSED) {
    DFK_TRY(stage1_fused(ctx, w, x, B, a2, a2_ld, cfg));
    return down_fused(ctx, w, a2, a2_ld, B, y, w->d_model, y_dtype == DFK_BF16,
                      cfg);
  }
  // Unfused comparators want a dense X (ld = d_model) and dense A2.
  DFK_TRY(stage1_unfused(ctx, w, x, B, a2, w->d_ff, cfg.variant));
  return down_unfused(ctx, w, a2, B, y, y_dtype == DFK_BF16);
}

int block_fused_tp(dfk_context_s* ctx, dfk_weights_s* w, const void* x, int64_t B,
                   void* y, bool y_bf16, const dfk_config& cfg, const StreamArgs* tp) {
  const int64_t a2_ld = round_up(w->d_ff, 8);
  DFK_TRY(ensure_buf(ctx, ctx->a2, static_cast<size_t>(B * a2_ld) * 2, false,
                     ctx->stream));
  return block_fused(ctx, w, x, B, static_cast<__nv_bfloat16*>(ctx->a2.p), a2_ld, y,
                     w->d_model, y_bf16, cfg, tp);
}

}  // namespace dfk

using namespace dfk;

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

const char* dfk_last_error(void) { return g_last_error.c_str(); }

const char* dfk_version(void) { return "dfk-b200 0.1.0 (sm_100a)"; }

int dfk_device_count(int* n) {
  DFK_CUDA(cudaGetDeviceCount(n));
  return DFK_OK;
}

int dfk_context_create(int device, void* stream, dfk_context* out) {
  if (!out) return fail(DFK_ERR_INVALID, "null out");
  *out = nullptr;
  int n = 0;
  DFK_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n)
    return fail(DFK_ERR_INVALID, "device " + std::to_string(device) +
                                     " out of range (" + std::to_string(n) +
                                     " visible)");
  DFK_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  DFK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0) {
    return fail(DFK_ERR_UNSUPPORTED,
                std::string("this library is built for sm_100a (B200); device "
                            "is ") +
                    prop.name + " sm_" + std::to_string(prop.major) +
                    std::to_string(prop.minor));
  }
  // Load every kernel now (lazy loading would do it at first launch, where
  // it can wait for the device; see preload_aux_kernels).
  {
    cudaError_t e = preload_stream_kernels();
    if (e == cudaSuccess) e = preload_aux_kernels();
    if (e != cudaSuccess)
      return fail(DFK_ERR_CUDA, std::string("kernel preload: ") + cudaGetErrorString(e));
  }
  auto* ctx = new dfk_context_s();
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  ctx->max_smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
  ctx->l2_bytes = prop.l2CacheSize;
  ctx->name = prop.name;
  ctx->cc_major = prop.major;
  ctx->cc_minor = prop.minor;
  cudaDriverGetVersion(&ctx->driver_version);
  // Host-mapped error word the kernels raise when a cross-rank (or host
  // copy) wait gives up; dfk_context_sync reports and clears it.
  if (cudaHostAlloc(reinterpret_cast<void**>(&ctx->err_host), sizeof(int),
                    cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->err_dev), ctx->err_host, 0) !=
          cudaSuccess) {
    if (ctx->err_host) cudaFreeHost(ctx->err_host);
    delete ctx;
    return fail(DFK_ERR_CUDA, "cannot allocate the mapped error word");
  }
  *ctx->err_host = 0;
  if (stream) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete ctx;
      return fail(DFK_ERR_CUDA, cudaGetErrorString(e));
    }
    ctx->own_stream = true;
  }
  *out = ctx;
  return DFK_OK;
}

int dfk_context_destroy(dfk_context ctx) {
  if (!ctx) return DFK_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (DeviceBuf* b : {&ctx->a2, &ctx->xpad, &ctx->a2pad, &ctx->yacc, &ctx->flags, &ctx->sched,
                       &ctx->counters, &ctx->concat, &ctx->tmp1, &ctx->tmp2,
                       &ctx->lt_ws, &ctx->flush, &ctx->hx_dev, &ctx->hy_dev,
                       &ctx->dec[0], &ctx->dec[1], &ctx->dec_f32, &ctx->s1acc,
                       &ctx->s1cnt, &ctx->mat_scratch}) {
    if (b->p) cudaFree(b->p);
  }
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second.exec);
  ctx->graphs.clear();
  if (ctx->side_stream) {
    cudaStreamSynchronize(ctx->side_stream);
    cudaStreamDestroy(ctx->side_stream);
  }
  if (ctx->out_stream) {
    cudaStreamSynchronize(ctx->out_stream);
    cudaStreamDestroy(ctx->out_stream);
  }
  for (HostSlot& sl : ctx->host_slots) {
    if (sl.x.p) cudaFree(sl.x.p);
    if (sl.y.p) cudaFree(sl.y.p);
  }
  if (ctx->host_flags.p) cudaFree(ctx->host_flags.p);
  for (int r = 0; r < 8; ++r)
    if (ctx->tp_peer_ipc[r] && ctx->tp_peer[r]) cudaIpcCloseMemHandle(ctx->tp_peer[r]);
  if (ctx->tp_sym.p) cudaFree(ctx->tp_sym.p);
  for (dfk_weights_s* w : ctx->weights) free_weights(w);
  ctx->weights.clear();
  if (ctx->err_host) cudaFreeHost(ctx->err_host);
  if (ctx->hx_pinned) cudaFreeHost(ctx->hx_pinned);
  if (ctx->hy_pinned) cudaFreeHost(ctx->hy_pinned);
  if (ctx->lt) cublasLtDestroy(ctx->lt);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return DFK_OK;
}

int dfk_context_sync(dfk_context ctx) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  DFK_TRY(use_device(ctx));
  DFK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->side_stream) DFK_CUDA(cudaStreamSynchronize(ctx->side_stream));
  if (ctx->out_stream) DFK_CUDA(cudaStreamSynchronize(ctx->out_stream));
  if (ctx->err_host && *reinterpret_cast<volatile int*>(ctx->err_host)) {
    *ctx->err_host = 0;
    return fail(DFK_ERR_TIMEOUT,
                "a kernel gave up waiting (> 4 s) for another rank's fused all-reduce "
                "contribution or for the host X copy; the results of the calls since the "
                "last sync are wrong.  Re-create the symmetric workspaces "
                "(dfk_tp_sym_create + _open / _attach) on every rank before the next "
                "tensor-parallel call");
  }
  return DFK_OK;
}

int dfk_context_stream(dfk_context ctx, void** stream) {
  if (!ctx || !stream) return fail(DFK_ERR_INVALID, "null argument");
  *stream = ctx->stream;
  return DFK_OK;
}

int dfk_fingerprint(dfk_context ctx, char* buf, size_t len) {
  if (!ctx || !buf) return fail(DFK_ERR_INVALID, "null argument");
  int mem_clock = 0;
  cudaDeviceGetAttribute(&mem_clock, cudaDevAttrMemoryClockRate, ctx->device);
  std::ostringstream o;
  o << ctx->name << "|sm_" << ctx->cc_major << ctx->cc_minor << "|" << ctx->sm_count
    << "SM|memclk" << mem_clock << "|drv" << ctx->driver_version << "|tp"
    << tp_degree(ctx, nullptr);
  std::snprintf(buf, len, "%s", o.str().c_str());
  return DFK_OK;
}

int dfk_sm_count(dfk_context ctx, int* n) {
  if (!ctx || !n) return fail(DFK_ERR_INVALID, "null argument");
  *n = ctx->sm_count;
  return DFK_OK;
}

int dfk_weights_create(dfk_context ctx, const void* w_gate, const void* w_up,
                       const void* w_down, int64_t d_model, int64_t d_ff,
                       int32_t dtype, int32_t memory, int64_t ff_begin,
                       int64_t ff_end, dfk_weights* out) {
  if (!ctx || !out) return fail(DFK_ERR_INVALID, "null argument");
  *out = nullptr;
  DFK_TRY(use_device(ctx));
  if (d_model < 1 || d_ff < 1) {
    return fail(DFK_ERR_SHAPE, "MlpWeights: dimensions must be >= 1, got d_model=" +
                                   std::to_string(d_model) +
                                   " d_ff=" + std::to_string(d_ff));
  }
  if (ff_begin < 0 || ff_end > d_ff || ff_begin >= ff_end) {
    return fail(DFK_ERR_SHAPE, "shard [" + std::to_string(ff_begin) + ", " +
                                   std::to_string(ff_end) +
                                   ") is empty or outside [0, " +
                                   std::to_string(d_ff) + ")");
  }
  // Stage-only sets (run_fused_stage1 takes W_up / W_gate alone,
  // fused.hpp:61; down_projection W_down alone, swiglu.hpp:90): W_down NULL
  // or W_gate and W_up both NULL.
  const bool has_s1 = w_gate || w_up, has_dn = w_down != nullptr;
  if ((w_gate == nullptr) != (w_up == nullptr))
    return fail(DFK_ERR_INVALID, "W_gate and W_up must both be given or both be NULL");
  if (!has_s1 && !has_dn) return fail(DFK_ERR_INVALID, "no weight matrix given");
  if (dtype != DFK_F64 && dtype != DFK_F32 && dtype != DFK_BF16)
    return fail(DFK_ERR_INVALID, "unknown dtype");
  DFK_CUDA(cudaSetDevice(ctx->device));
  auto* w = new dfk_weights_s();
  w->ctx = ctx;
  w->d_model = d_model;
  w->d_ff = ff_end - ff_begin;
  w->ff_begin = ff_begin;
  w->d_ff_total = d_ff;
  w->s1_tiles = static_cast<int>(ceil_div64(w->d_ff, kS1Cols));
  w->s1_kblocks = static_cast<int>(ceil_div64(d_model, kBlockK));
  w->dn_tiles = static_cast<int>(ceil_div64(d_model, kDownCols));
  w->dn_kblocks = static_cast<int>(ceil_div64(w->d_ff, kBlockK));
  const size_t s1_bytes =
      static_cast<size_t>(w->s1_tiles) * w->s1_kblocks * kBlockBytes;
  const size_t dn_bytes =
      static_cast<size_t>(w->dn_tiles) * w->dn_kblocks * kBlockBytes;
  auto drop = [&](int status, const std::string& msg) {
    if (w->s1_pack) cudaFree(w->s1_pack);
    if (w->dn_pack) cudaFree(w->dn_pack);
    delete w;
    return fail(status, msg);
  };
  if ((has_s1 && cudaMalloc(&w->s1_pack, s1_bytes) != cudaSuccess) ||
      (has_dn && cudaMalloc(&w->dn_pack, dn_bytes) != cudaSuccess)) {
    cudaGetLastError();
    return drop(DFK_ERR_NOMEM, "weight pack allocation");
  }
  const void* srcs[3] = {w_gate, w_up, w_down};
  void* staging[3] = {nullptr, nullptr, nullptr};
  const size_t esz = dtype_size(dtype);
  if (memory == DFK_HOST) {
    const size_t n1 = static_cast<size_t>(d_model * d_ff) * esz;
    for (int i = 0; i < 3; ++i) {
      if (!srcs[i]) continue;
      if (cudaMalloc(&staging[i], n1) != cudaSuccess) {
        cudaGetLastError();
        for (void* p : staging) cudaFree(p);
        return drop(DFK_ERR_NOMEM, "weight staging allocation");
      }
      DFK_CUDA(cudaMemcpyAsync(staging[i], srcs[i], n1, cudaMemcpyHostToDevice,
                               ctx->stream));
      srcs[i] = staging[i];
    }
  }
  cudaError_t e1 = cudaSuccess, e2 = cudaSuccess;
  if (has_s1)
    e1 = launch_pack_stage1(srcs[0], srcs[1], dtype, d_model, d_ff, ff_begin, w->d_ff,
                            w->s1_tiles, w->s1_kblocks, w->s1_pack, ctx->stream);
  if (has_dn)
    e2 = launch_pack_down(srcs[2], dtype, d_model, ff_begin, w->d_ff, w->dn_tiles,
                          w->dn_kblocks, w->dn_pack, ctx->stream);
  cudaError_t e3 = cudaStreamSynchronize(ctx->stream);
  for (void* p : staging)
    if (p) cudaFree(p);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
    return drop(DFK_ERR_CUDA, std::string("weight prepack: ") +
                                  cudaGetErrorString(e1 != cudaSuccess   ? e1
                                                     : e2 != cudaSuccess ? e2
                                                                         : e3));
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->weights.insert(w);  // freed with the context if never destroyed
  }
  *out = w;
  return DFK_OK;
}

int dfk_weights_destroy(dfk_weights w) {
  if (!w) return DFK_OK;
  dfk_context_s* ctx = w->ctx;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!ctx->weights.erase(w)) return fail(DFK_ERR_INVALID, "unknown weights handle");
    // A new handle may reuse this address: graphs keyed by it are stale.
    ++ctx->generation;
  }
  free_weights(w);
  return DFK_OK;
}

int dfk_weights_shape(dfk_weights w, int64_t* d_model, int64_t* d_ff_shard,
                      int64_t* ff_begin) {
  if (!w) return fail(DFK_ERR_INVALID, "null weights");
  if (d_model) *d_model = w->d_model;
  if (d_ff_shard) *d_ff_shard = w->d_ff;
  if (ff_begin) *ff_begin = w->ff_begin;
  return DFK_OK;
}

int dfk_weights_bytes(dfk_weights w, int64_t* bytes) {
  if (!w || !bytes) return fail(DFK_ERR_INVALID, "null argument");
  *bytes = ((w->s1_pack ? static_cast<int64_t>(w->s1_tiles) * w->s1_kblocks : 0) +
            (w->dn_pack ? static_cast<int64_t>(w->dn_tiles) * w->dn_kblocks : 0)) *
           kBlockBytes;
  return DFK_OK;
}

int dfk_stage1(dfk_context ctx, dfk_weights w, const void* x, int64_t batch,
               void* a2, const dfk_config* cfg_in) {
  DFK_TRY(check_handles(ctx, w, true, false));
  DFK_TRY(check_batch(batch));
  if (!x || !a2) return fail(DFK_ERR_INVALID, "null activation pointer");
  dfk_config cfg;
  DFK_TRY(resolve_config(ctx, w, batch, cfg_in, &cfg));
  auto* out = static_cast<__nv_bfloat16*>(a2);
  if (cfg.variant == DFK_VARIANT_FUSED)
    return stage1_fused(ctx, w, x, batch, out, w->d_ff, cfg);
  return stage1_unfused(ctx, w, x, batch, out, w->d_ff, cfg.variant);
}

int dfk_down(dfk_context ctx, dfk_weights w, const void* a2, int64_t batch,
             void* y, int32_t y_dtype, const dfk_config* cfg_in) {
  DFK_TRY(check_handles(ctx, w, false, true));
  DFK_TRY(check_batch(batch));
  if (!a2 || !y) return fail(DFK_ERR_INVALID, "null activation pointer");
  if (y_dtype != DFK_F32 && y_dtype != DFK_BF16)
    return fail(DFK_ERR_INVALID, "y_dtype must be F32 or BF16");
  dfk_config cfg;
  DFK_TRY(resolve_config(ctx, w, batch, cfg_in, &cfg));
  if (cfg.variant == DFK_VARIANT_FUSED)
    return down_fused(ctx, w, a2, w->d_ff, batch, y, w->d_model,
                      y_dtype == DFK_BF16, cfg);
  return down_unfused(ctx, w, a2, batch, y, y_dtype == DFK_BF16);
}

int dfk_forward(dfk_context ctx, dfk_weights w, const void* x, int64_t batch,
                void* y, int32_t y_dtype, const dfk_config* cfg) {
  return forward_impl(ctx, w, x, batch, y, y_dtype, cfg);
}

int dfk_forward_host(dfk_context ctx, dfk_weights w, const void* x,
                     int32_t x_dtype, int64_t batch, void* y, int32_t y_dtype,
                     const dfk_config* cfg) {
  DFK_TRY(check_handles(ctx, w));
  DFK_TRY(check_batch(batch));
  if (!x || !y) return fail(DFK_ERR_INVALID, "null host pointer");
  DFK_CUDA(cudaSetDevice(ctx->device));
  const int64_t dm = w->d_model;
  const size_t xn = static_cast<size_t>(batch * dm);
  const size_t xb = xn * 2;
  const size_t yb = xn * 4;
  if (ctx->hx_pinned_bytes < xb) {
    if (ctx->hx_pinned) cudaFreeHost(ctx->hx_pinned);
    DFK_CUDA(cudaMallocHost(&ctx->hx_pinned, xb));
    ctx->hx_pinned_bytes = xb;
  }
  if (ctx->hy_pinned_bytes < yb) {
    if (ctx->hy_pinned) cudaFreeHost(ctx->hy_pinned);
    DFK_CUDA(cudaMallocHost(&ctx->hy_pinned, yb));
    ctx->hy_pinned_bytes = yb;
  }
  auto* hx = static_cast<uint16_t*>(ctx->hx_pinned);
  if (x_dtype != DFK_BF16 && x_dtype != DFK_F32 && x_dtype != DFK_F64)
    return fail(DFK_ERR_INVALID, "unknown x dtype");
  if (y_dtype != DFK_BF16 && y_dtype != DFK_F32 && y_dtype != DFK_F64)
    return fail(DFK_ERR_INVALID, "unknown y dtype");
  host_to_bf16(x, x_dtype, xn, hx);  // RNE, on the host-conversion pool
  DFK_TRY(ensure_buf(ctx, ctx->hx_dev, xb, false, ctx->stream));
  DFK_TRY(ensure_buf(ctx, ctx->hy_dev, yb, false, ctx->stream));
  DFK_CUDA(cudaMemcpyAsync(ctx->hx_dev.p, hx, xb, cudaMemcpyHostToDevice,
                           ctx->stream));
  if (tp_active(ctx)) {
    DFK_TRY(tp_block(ctx, w, ctx->hx_dev.p, batch,
                     static_cast<float*>(ctx->hy_dev.p), cfg));
  } else {
    DFK_TRY(forward_impl(ctx, w, ctx->hx_dev.p, batch, ctx->hy_dev.p, DFK_F32,
                         cfg));
  }
  DFK_CUDA(cudaMemcpyAsync(ctx->hy_pinned, ctx->hy_dev.p, yb,
                           cudaMemcpyDeviceToHost, ctx->stream));
  DFK_CUDA(cudaStreamSynchronize(ctx->stream));
  host_from_f32(static_cast<const float*>(ctx->hy_pinned), xn, y, y_dtype);
  return DFK_OK;
}

int dfk_forward_host_async(dfk_context ctx, dfk_weights w,
                           const void* x_pinned_bf16, int64_t batch,
                           float* y_pinned, const dfk_config* cfg) {
  DFK_TRY(check_handles(ctx, w));
  DFK_TRY(check_batch(batch));
  if (!x_pinned_bf16 || !y_pinned) return fail(DFK_ERR_INVALID, "null host pointer");
  const size_t xb = static_cast<size_t>(batch * w->d_model) * 2;
  const size_t yb = static_cast<size_t>(batch * w->d_model) * 4;
  dfk_config rc;
  DFK_TRY(resolve_config(ctx, w, batch, cfg, &rc));
  static const WaitValueFn wait_value = driver_fn<WaitValueFn>("cuStreamWaitValue32");
  static const WriteValueFn write_value = driver_fn<WriteValueFn>("cuStreamWriteValue32");
  // (one block launch per call: the GEMV family launches 8-row chunks, and
  // only a single launch carries the X-ready / Y-done flags)
  const int64_t one_launch = rc.s1_family == DFK_FAMILY_GEMV ? 8 : 256;
  if (!tp_active(ctx) && batch <= one_launch && rc.variant == DFK_VARIANT_FUSED &&
      rc.block_kernel && rc.dynamic_sched && rc.s1_split_k <= 1 && wait_value &&
      write_value && !knobs().host_stagek) {
    // Copy-engine X and Y: the H2D copy runs on a side stream as soon as its
    // ring slot is free (device flag x_free >= previous user's sequence no.)
    // and then publishes x_ready = seq; the block kernel -- still PDL-chained
    // to the previous block, nothing in between on the context stream --
    // waits for x_ready before its first X load, writes Y into the slot and
    // its last CTA publishes y_done = seq, on which the side stream's D2H
    // waits.  Both copies are off the block chain's critical path.
    if (!ctx->side_stream) {
      DFK_CUDA(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
      DFK_CUDA(cudaStreamCreateWithFlags(&ctx->out_stream, cudaStreamNonBlocking));
    }
    DFK_TRY(ensure_buf(ctx, ctx->host_flags, 3 * kHostSlots * sizeof(unsigned), true, ctx->stream));
    const int si = ctx->host_next;
    HostSlot& sl = ctx->host_slots[si];
    ctx->host_next = (ctx->host_next + 1) % kHostSlots;
    if (sl.x.bytes < xb || sl.y.bytes < yb) {
      DFK_CUDA(cudaStreamSynchronize(ctx->stream));
      DFK_CUDA(cudaStreamSynchronize(ctx->side_stream));
      DFK_CUDA(cudaStreamSynchronize(ctx->out_stream));
      const size_t nx = std::max<size_t>({xb, 2 * sl.x.bytes, 64 * 1024});
      const size_t ny = std::max<size_t>({yb, 2 * sl.y.bytes, 128 * 1024});
      for (HostSlot& o : ctx->host_slots) {
        DFK_TRY(ensure_buf(ctx, o.x, nx, false, ctx->stream));
        DFK_TRY(ensure_buf(ctx, o.y, ny, false, ctx->stream));
      }
      DFK_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    auto* flags = static_cast<unsigned*>(ctx->host_flags.p);
    unsigned* x_ready = flags + si;
    unsigned* x_free = flags + kHostSlots + si;
    unsigned* y_done = flags + 2 * kHostSlots + si;
    const unsigned seq = ++ctx->host_seq;
    if (seq > static_cast<unsigned>(kHostSlots)) {  // the slot's previous user is done
      if (wait_value(ctx->side_stream, reinterpret_cast<CUdeviceptr>(x_free),
                     seq - kHostSlots, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(DFK_ERR_CUDA, "cuStreamWaitValue32 failed");
    }
    DFK_CUDA(cudaMemcpyAsync(sl.x.p, x_pinned_bf16, xb, cudaMemcpyHostToDevice,
                             ctx->side_stream));
    if (write_value(ctx->side_stream, reinterpret_cast<CUdeviceptr>(x_ready), seq,
                    CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return fail(DFK_ERR_CUDA, "cuStreamWriteValue32 failed");
    ctx->pend_x_ready = x_ready;
    ctx->pend_x_free = x_free;
    ctx->pend_y_done = y_done;
    ctx->pend_x_seq = seq;
    const int st = forward_impl(ctx, w, sl.x.p, batch, sl.y.p, DFK_F32, &rc);
    ctx->pend_x_ready = nullptr;
    ctx->pend_x_free = nullptr;
    ctx->pend_y_done = nullptr;
    DFK_TRY(st);
    // Y leaves on its own stream, so that the next X copies never queue
    // behind this block's completion.  (x_free is published with y_done, so
    // the slot's Y is not overwritten before this copy: the next user's X
    // copy waits for x_free, its block for that X.)
    if (wait_value(ctx->out_stream, reinterpret_cast<CUdeviceptr>(y_done), seq,
                   CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail(DFK_ERR_CUDA, "cuStreamWaitValue32 failed");
    DFK_CUDA(cudaMemcpyAsync(y_pinned, sl.y.p, yb, cudaMemcpyDeviceToHost,
                             ctx->out_stream));
    return DFK_OK;
  }
  if (!tp_active(ctx) && xb % 16 == 0) {
    // Zero-copy chain: a staging kernel pulls X over PCIe into a ring slot
    // (PDL: overlapping the previous block), the block writes Y straight
    // into the caller's pinned buffer -- kernels only, no memcpy or event
    // between the blocks, so consecutive calls stay PDL-chained.  (A copy
    // stream + events variant measured slower: the events between kernels
    // break the PDL chain, tools/e2e_probe.py.)
    cudaPointerAttributes ax{}, ay{};
    DFK_CUDA(cudaPointerGetAttributes(&ax, x_pinned_bf16));
    DFK_CUDA(cudaPointerGetAttributes(&ay, y_pinned));
    if (!ax.devicePointer || !ay.devicePointer)
      return fail(DFK_ERR_INVALID, "forward_host_async needs pinned (cudaMallocHost) buffers");
    HostSlot& sl = ctx->host_slots[ctx->host_next];
    ctx->host_next = (ctx->host_next + 1) % kHostSlots;
    if (sl.x.bytes < xb) {
      // Grow every slot at once (geometrically): a reallocation waits for
      // the device, so it must not recur as batch sizes rotate over slots.
      DFK_CUDA(cudaStreamSynchronize(ctx->stream));
      const size_t nb = std::max<size_t>({xb, 2 * sl.x.bytes, 64 * 1024});
      for (HostSlot& o : ctx->host_slots) DFK_TRY(ensure_buf(ctx, o.x, nb, false, ctx->stream));
    }
    cudaError_t e = launch_stage_rows(ax.devicePointer, sl.x.p, static_cast<int64_t>(xb),
                                      ctx->stream);
    if (e != cudaSuccess) return fail(DFK_ERR_CUDA, cudaGetErrorString(e));
    ctx->launches++;
    return forward_impl(ctx, w, sl.x.p, batch, ay.devicePointer, DFK_F32, cfg);
  }
  // Stream order makes one staging pair safe: the next call's H2D runs after
  // this call's kernels, its kernels after this call's D2H.
  DFK_TRY(ensure_buf(ctx, ctx->hx_dev, xb, false, ctx->stream));
  DFK_TRY(ensure_buf(ctx, ctx->hy_dev, yb, false, ctx->stream));
  DFK_CUDA(cudaMemcpyAsync(ctx->hx_dev.p, x_pinned_bf16, xb,
                           cudaMemcpyHostToDevice, ctx->stream));
  if (tp_active(ctx)) {
    DFK_TRY(tp_block(ctx, w, ctx->hx_dev.p, batch,
                     static_cast<float*>(ctx->hy_dev.p), cfg));
  } else {
    DFK_TRY(forward_impl(ctx, w, ctx->hx_dev.p, batch, ctx->hy_dev.p, DFK_F32,
                         cfg));
  }
  DFK_CUDA(cudaMemcpyAsync(y_pinned, ctx->hy_dev.p, yb, cudaMemcpyDeviceToHost,
                           ctx->stream));
  return DFK_OK;
}

int dfk_balanced_range(int64_t extent, int64_t parts, int64_t index,
                       int64_t* begin, int64_t* end) {
  if (parts < 1) return fail(DFK_ERR_SHAPE, "balanced_ranges: parts must be >= 1");
  if (parts > extent)
    return fail(DFK_ERR_SHAPE, "balanced_ranges: cannot split extent " +
                                   std::to_string(extent) + " into " +
                                   std::to_string(parts) + " non-empty ranges");
  if (index < 0 || index >= parts) return fail(DFK_ERR_INVALID, "index out of range");
  const int64_t base = extent / parts, rem = extent % parts;
  const int64_t b = index * base + std::min(index, rem);
  *begin = b;
  *end = b + base + (index < rem ? 1 : 0);
  return DFK_OK;
}

int dfk_block_bytes(int64_t batch, int64_t d_model, int64_t d_ff,
                    int64_t* stage1, int64_t* stage2) {
  if (batch < 1 || d_model < 1 || d_ff < 1)
    return fail(DFK_ERR_SHAPE, "dims must be >= 1");
  // Fused single covering tile: X once, both weights once, A2 written once;
  // stage 2: A2 read once, W_down once, Y written once; 2 bytes/element.
  if (stage1) *stage1 = 2 * (batch * d_model + 2 * d_model * d_ff + batch * d_ff);
  if (stage2) *stage2 = 2 * (batch * d_ff + d_ff * d_model + batch * d_model);
  return DFK_OK;
}

int dfk_malloc(dfk_context ctx, size_t bytes, void** p) {
  if (!ctx || !p) return fail(DFK_ERR_INVALID, "null argument");
  DFK_CUDA(cudaSetDevice(ctx->device));
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
  if (e != cudaSuccess) return fail(DFK_ERR_NOMEM, cudaGetErrorString(e));
  return DFK_OK;
}

int dfk_free(dfk_context ctx, void* p) {
  if (ctx) cudaSetDevice(ctx->device);
  if (p) DFK_CUDA(cudaFree(p));
  return DFK_OK;
}

int dfk_host_alloc(size_t bytes, void** p) {
  DFK_CUDA(cudaMallocHost(p, bytes ? bytes : 16));
  return DFK_OK;
}

int dfk_host_free(void* p) {
  if (p) DFK_CUDA(cudaFreeHost(p));
  return DFK_OK;
}

int dfk_memcpy_h2d(dfk_context ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  DFK_TRY(use_device(ctx));
  DFK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return DFK_OK;
}

int dfk_memcpy_d2h(dfk_context ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  DFK_TRY(use_device(ctx));
  DFK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return DFK_OK;
}

int dfk_memset(dfk_context ctx, void* p, int value, size_t bytes) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  DFK_TRY(use_device(ctx));
  DFK_CUDA(cudaMemsetAsync(p, value, bytes, ctx->stream));
  return DFK_OK;
}

int dfk_fill_uniform_bf16(dfk_context ctx, void* p, int64_t n, uint64_t seed,
                          float lo, float hi) {
  if (!ctx || !p) return fail(DFK_ERR_INVALID, "null argument");
  DFK_TRY(use_device(ctx));
  DFK_CUDA(launch_fill_uniform_bf16(static_cast<__nv_bfloat16*>(p), n, seed, lo,
                                    hi, ctx->stream));
  return DFK_OK;
}

int dfk_event_create(void** ev) {
  cudaEvent_t e;
  DFK_CUDA(cudaEventCreate(&e));
  *ev = e;
  return DFK_OK;
}

int dfk_event_destroy(void* ev) {
  if (ev) DFK_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
  return DFK_OK;
}

int dfk_event_record(dfk_context ctx, void* ev) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  DFK_TRY(use_device(ctx));
  DFK_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), ctx->stream));
  return DFK_OK;
}

int dfk_event_elapsed_ms(void* start, void* stop, float* ms) {
  DFK_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(stop)));
  DFK_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start),
                                static_cast<cudaEvent_t>(stop)));
  return DFK_OK;
}

int dfk_flush_l2(dfk_context ctx) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  DFK_TRY(use_device(ctx));
  const size_t bytes = static_cast<size_t>(std::max(ctx->l2_bytes, 1 << 20)) * 2;
  DFK_TRY(ensure_buf(ctx, ctx->flush, bytes, false, ctx->stream));
  DFK_CUDA(launch_flush(ctx->flush.p, bytes, ctx->stream));
  return DFK_OK;
}

int dfk_set_trace(dfk_context ctx, void* buf, int64_t slots) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  if (buf && slots < static_cast<int64_t>(ctx->sm_count) * 2 * kTraceSlots)
    return fail(DFK_ERR_INVALID, "trace buffer needs >= 2 * SMs * 64 slots");
  ctx->trace = static_cast<unsigned long long*>(buf);
  ctx->trace_slots = slots;
  return DFK_OK;
}

int dfk_launch_count(dfk_context ctx, int64_t* n) {
  if (!ctx || !n) return fail(DFK_ERR_INVALID, "null argument");
  *n = ctx->launches;
  return DFK_OK;
}

int dfk_profiler_range(dfk_context ctx, int32_t start) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  DFK_CUDA(cudaStreamSynchronize(ctx->stream));
  DFK_CUDA(start ? cudaProfilerStart() : cudaProfilerStop());
  return DFK_OK;
}

}  // extern "C"
