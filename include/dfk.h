/*
 * dfk.h — C ABI of the B200-native fused SwiGLU-MLP path (DeepFusionKernel,
 * arXiv 2602.11808).
 *
 * This is the drop-in boundary for the reference's C++ operator API
 * (/root/reference/proj/include/deepfusion/{fused,swiglu,tp,tuner}.hpp).
 * Plain pointers and sizes only; no C++ or torch types cross it; no
 * exceptions cross it.  Every entry point returns a dfk_status (0 = OK) and
 * leaves a thread-local message in dfk_last_error() on failure.
 *
 * Mapping of the reference interface (file:line under
 * /root/reference/proj/) to the entry points that replace it:
 *
 *   run_fused_stage1   include/deepfusion/fused.hpp:61-63     -> dfk_stage1
 *   run_fused          include/deepfusion/fused.hpp:66-67     -> dfk_forward
 *   down_projection    include/deepfusion/swiglu.hpp:90-91    -> dfk_down
 *   run_stage1         include/deepfusion/fused.hpp:82-84     -> dfk_stage1
 *                                                               (cfg.variant)
 *   run_variant        include/deepfusion/fused.hpp:87-89     -> dfk_forward
 *                                                               (cfg.variant)
 *   run_four_kernel / run_two_kernel  swiglu.hpp:64-76        -> dfk_forward
 *                                       (DFK_VARIANT_FOUR/TWO_KERNEL)
 *   MlpWeights (+validate)  swiglu.hpp:49-57, swiglu.cpp:26-39 -> dfk_weights_create
 *   make_plan / run_tp_mlp  tp.hpp:54-79                      -> dfk_tp_sym_create /
 *                                                               _open / _attach +
 *                                                               dfk_tp_forward_fused
 *                                                               (all-reduce in the
 *                                                               kernel), or
 *                                                               dfk_tp_init* +
 *                                                               dfk_tp_forward (NCCL),
 *                                                               dfk_weights_create
 *                                                               (ff_begin/ff_end)
 *   simulated_all_reduce    tp.cpp:90-105                     -> the fused all-reduce
 *   time_decode_seconds     bench.cpp:98-115                  -> dfk_decode
 *   forward with host Matrix (the shim's run_fused)           -> dfk_forward_host,
 *                                                               dfk_forward_host_async
 *   balanced_ranges         tp.hpp:36, tp.cpp:8-29            -> dfk_balanced_range
 *   profile / select / Tuner::get_or_tune  tuner.hpp:103-137  -> dfk_tune
 *   cache_store / cache_lookup  tuner.hpp:102-113              -> dfk_cache_store /
 *                                                               dfk_cache_lookup (and
 *                                                               dfk_tune's cache_path)
 *   default_candidates      tuner.hpp:55                      -> dfk_candidates
 *   default_fingerprint     tuner.hpp:116                     -> dfk_fingerprint
 *   predict_traffic         traffic.hpp:60-71 (fused, single tile)
 *                                                             -> dfk_block_bytes
 *
 * Error classes mirror the reference's exceptions: ShapeError
 * (tensor.hpp:21-23) -> DFK_ERR_SHAPE; std::invalid_argument (unknown
 * variant, scheme mismatch) -> DFK_ERR_INVALID; "every candidate
 * disqualified" (tuner.cpp:185-188) -> DFK_ERR_GATE; CacheError
 * (tuner.hpp:97-99) -> DFK_ERR_CACHE.
 *
 * Data: activations are bf16 row-major on the device (X [B x d_model],
 * A2 [B x d_ff_shard]); Y is fp32 or bf16 [B x d_model].  Weights are
 * registered once in the reference layout (W_gate, W_up [d_model x d_ff],
 * W_down [d_ff x d_model], row-major; fp64 / fp32 / bf16; host or device)
 * and prepacked into the streaming layout.  All compute calls are
 * asynchronous on the context's stream; the caller synchronises.  One
 * context per GPU per host thread.
 */
#ifndef DFK_H_
#define DFK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFK_API __attribute__((visibility("default")))

typedef enum dfk_status {
  DFK_OK = 0,
  DFK_ERR_SHAPE = 1,       /* reference ShapeError */
  DFK_ERR_INVALID = 2,     /* reference std::invalid_argument */
  DFK_ERR_CUDA = 3,
  DFK_ERR_NCCL = 4,
  DFK_ERR_NOMEM = 5,
  DFK_ERR_UNSUPPORTED = 6,
  DFK_ERR_GATE = 7,        /* every scheduler candidate failed the gate */
  DFK_ERR_CACHE = 8,       /* reference CacheError */
  DFK_ERR_TIMEOUT = 9      /* a fused all-reduce wait on a peer gave up
                              (reported by dfk_context_sync)               */
} dfk_status;

typedef enum dfk_dtype { DFK_F64 = 0, DFK_F32 = 1, DFK_BF16 = 2 } dfk_dtype;
typedef enum dfk_memory { DFK_HOST = 0, DFK_DEVICE = 1 } dfk_memory;

/* Execution layout of the block (reference VariantTag, swiglu.hpp:16). */
typedef enum dfk_variant {
  DFK_VARIANT_FUSED = 0,       /* fused stage 1 + down (the product)        */
  DFK_VARIANT_TWO_KERNEL = 1,  /* cuBLASLt [W_gate|W_up] GEMM + silu_mul +
                                  cuBLASLt down: the unfused comparator     */
  DFK_VARIANT_FOUR_KERNEL = 2  /* 2 GEMMs + silu + mul + down               */
} dfk_variant;

/* Kernel family of a fused stage (0 = let the library choose). */
typedef enum dfk_family {
  DFK_FAMILY_AUTO = 0,
  DFK_FAMILY_TC = 1,    /* tcgen05 / TMEM tensor-core kernel ("F2")       */
  DFK_FAMILY_GEMV = 2   /* CUDA-core warp GEMV, batch <= 8 ("F1")         */
} dfk_family;

/* One scheduler candidate / launch configuration (the GPU counterpart of
 * KernelConfig + TileConfig, fused.hpp:25-47).  Zero-initialised fields mean
 * "library default". */
typedef struct dfk_config {
  int32_t variant;      /* dfk_variant                                     */
  int32_t s1_family;    /* dfk_family for the fused stage 1                */
  int32_t s1_stages;    /* smem pipeline depth (0 = deepest that fits)     */
  int32_t s1_ctas;      /* persistent CTAs (0 = one per SM)                */
  int32_t s1_split_k;   /* CTAs sharing one stage-1 tile (1 = none)        */
  int32_t down_family;  /* dfk_family for the down projection              */
  int32_t down_stages;
  int32_t down_ctas;    /* stream-K CTAs (0 = one per SM)                  */
  int32_t pdl;          /* 1 = programmatic dependent launch between the
                           two kernels (and across calls); 0 = plain       */
  int32_t mutant;       /* negative controls, tests only: 0 = none, 1 =
                           SiLU*up per K chunk (stream-K / split-K pieces;
                           verification.cpp:84-124), 2 = SiLU(A_gate)
                           round-tripped through a global buffer
                           (MaterializeIntermediate, :126-169)            */
  int32_t block_kernel; /* 1 = the whole block (stage 1 + down) in ONE
                           persistent kernel with per-tile A2 dependency
                           flags (the paper's single deeply fused kernel);
                           0 = two kernels (stage 1, then down)          */
  int32_t kbs;          /* 16 KiB weight blocks per pipeline stage (0 = auto) */
  int32_t dynamic_sched;/* 1 = CTAs pull work pieces from an atomic counter
                           (tiles, then fixed-size down chunks) instead of
                           the static byte-balanced plan                    */
  int32_t chunk_kb;     /* K blocks per dynamic down chunk (0 = auto)      */
  int32_t s1_chunk_kb;  /* K blocks per dynamic stage-1 piece: stream-K
                           over d_model with fp32 partial sums (0 = auto:
                           split only when the shard has fewer stage-1
                           tiles than CTAs)                                */
  int32_t s1_tail;      /* dynamic block kernel on shards with more stage-1
                           tiles than CTAs: the first wave of tiles runs
                           whole, every later tile is split into s1_tail
                           K parts (stream-K), spreading the last stage-1
                           wave over all CTAs (0 = auto: 3 at batch > 16,
                           off below; 1 = off)                            */
  char label[64];       /* scheduler label, e.g. "fused_tc_s12_pdl"        */
} dfk_config;

typedef struct dfk_context_s* dfk_context;
typedef struct dfk_weights_s* dfk_weights;

/* --- library / context ------------------------------------------------- */
DFK_API const char* dfk_last_error(void);
DFK_API const char* dfk_version(void);
DFK_API int dfk_device_count(int* n);
/* stream: a cudaStream_t to run on, or NULL for a context-owned stream. */
DFK_API int dfk_context_create(int device, void* stream, dfk_context* out);
DFK_API int dfk_context_destroy(dfk_context ctx);
DFK_API int dfk_context_sync(dfk_context ctx);
DFK_API int dfk_context_stream(dfk_context ctx, void** stream);
/* Free-text device descriptor used as the tuning-cache fingerprint
 * (the GPU counterpart of default_fingerprint, tuner.cpp:392-406). */
DFK_API int dfk_fingerprint(dfk_context ctx, char* buf, size_t len);
DFK_API int dfk_sm_count(dfk_context ctx, int* n);

/* --- weights --------------------------------------------------------- */
/* Registers one block's weights in the reference layout and prepacks them.
 * [ff_begin, ff_end) selects a tensor-parallel shard of d_ff (pass 0, d_ff
 * for the whole block): W_gate/W_up columns and W_down rows of that range
 * (tp.cpp:140-167).  Stage-only sets: w_down NULL registers stage 1 alone
 * (run_fused_stage1's W_up / W_gate, fused.hpp:61-63; dfk_stage1 only),
 * w_gate and w_up both NULL registers the down projection alone
 * (down_projection's W_down, swiglu.hpp:90-91; dfk_down only); calls that
 * need the missing part fail with DFK_ERR_INVALID.  Errors: DFK_ERR_SHAPE
 * for dims < 1 or an empty / out-of-range shard. */
DFK_API int dfk_weights_create(dfk_context ctx, const void* w_gate,
                               const void* w_up, const void* w_down,
                               int64_t d_model, int64_t d_ff, int32_t dtype,
                               int32_t memory, int64_t ff_begin,
                               int64_t ff_end, dfk_weights* out);
DFK_API int dfk_weights_destroy(dfk_weights w);
DFK_API int dfk_weights_shape(dfk_weights w, int64_t* d_model,
                              int64_t* d_ff_shard, int64_t* ff_begin);
/* Bytes of packed weights resident in HBM for this handle. */
DFK_API int dfk_weights_bytes(dfk_weights w, int64_t* bytes);

/* --- the hot path (device pointers, asynchronous) ---------------------- */
/* A2 = (X W_up) * silu(X W_gate): X bf16 [B x d_model], A2 bf16
 * [B x d_ff_shard].  cfg NULL = scheduler's choice for B. */
DFK_API int dfk_stage1(dfk_context ctx, dfk_weights w, const void* x,
                       int64_t batch, void* a2, const dfk_config* cfg);
/* Y = A2 W_down: A2 bf16 [B x d_ff_shard], Y (y_dtype F32/BF16)
 * [B x d_model]. */
DFK_API int dfk_down(dfk_context ctx, dfk_weights w, const void* a2,
                     int64_t batch, void* y, int32_t y_dtype,
                     const dfk_config* cfg);
/* Whole block: Y = stage-2(stage-1(X)); A2 lives in context scratch.  An
 * fp32 Y in device memory is zeroed by the kernel and accumulated in place
 * ("direct Y"); X may overlap Y (in-place callers get the workspace path). */
DFK_API int dfk_forward(dfk_context ctx, dfk_weights w, const void* x,
                        int64_t batch, void* y, int32_t y_dtype,
                        const dfk_config* cfg);
/* Reference-facing call with HOST buffers (synchronous): converts X
 * (x_dtype F64/F32/BF16) to bf16, copies it in, runs dfk_forward (or
 * the TP block -- dfk_tp_forward_fused when the symmetric workspaces are
 * set up, else dfk_tp_forward when the context has a TP communicator),
 * copies Y out and
 * converts it to y_dtype. */
DFK_API int dfk_forward_host(dfk_context ctx, dfk_weights w, const void* x,
                             int32_t x_dtype, int64_t batch, void* y,
                             int32_t y_dtype, const dfk_config* cfg);

/* Asynchronous host-buffer call for pipelined callers: X is bf16 in PINNED
 * host memory, Y is fp32 in PINNED host memory.  With the (default) dynamic
 * block kernel the copies never sit between two blocks on the context
 * stream: X goes H2D on a side stream into a device ring slot and publishes
 * a device flag the block waits on; the block's last CTA publishes "Y done"
 * and a second side stream copies Y out.  Other layouts: a PDL-chained
 * staging kernel pulls X and Y is written to the pinned buffer directly;
 * under TP, H2D(X), the TP block, D2H(Y) in stream order.  Buffers must stay
 * valid until dfk_context_sync (which waits for the side streams too). */
DFK_API int dfk_forward_host_async(dfk_context ctx, dfk_weights w,
                                   const void* x_pinned_bf16, int64_t batch,
                                   float* y_pinned, const dfk_config* cfg);

/* Decode loop (time_decode_seconds, bench.cpp:98-115): `steps` passes over
 * the `n_layers` blocks `layers` (same d_model), x <- Y after every block as
 * a bf16 chain; the last block's Y lands in y_out (bf16 [B x d_model],
 * device).  Under TP every block is a dfk_tp_forward_fused (or, with only
 * an NCCL communicator, a dfk_tp_forward).  use_graph != 0
 * captures the whole sequence into a CUDA graph on first use (after one
 * eager pass that sizes every scratch buffer) and replays it on later calls
 * with the same (layers, batch, steps, x, y_out, resolved config).
 * Asynchronous on the context stream. */
DFK_API int dfk_decode(dfk_context ctx, const dfk_weights* layers,
                       int32_t n_layers, const void* x, int64_t batch,
                       int32_t steps, void* y_out, const dfk_config* cfg,
                       int32_t use_graph);

/* --- scheduler (tuner.cpp semantics) ----------------------------------- */
/* Candidate grid for (weights, B): fills up to `cap` configs, returns the
 * count in *n (default_candidates, tuner.cpp:59-88). */
/* The configuration a compute call with `cfg` runs at this batch: cfg
 * itself, or (NULL) the scheduler's stored decision for the shape, else the
 * library default (the dynamic block kernel; warp-GEMV at B = 1 on shards
 * with <= 40 stage-1 tiles). */
DFK_API int dfk_resolve_config(dfk_context ctx, dfk_weights w, int64_t batch,
                               const dfk_config* cfg, dfk_config* out);
DFK_API int dfk_candidates(dfk_context ctx, dfk_weights w, int64_t batch,
                           dfk_config* out, int32_t cap, int32_t* n);
/* The same grid for a shape (B, d_model, d_ff shard) without registered
 * weights (the C++ shim's gpu_candidates). */
DFK_API int dfk_candidates_shape(dfk_context ctx, int64_t batch, int64_t d_model,
                                 int64_t d_ff, dfk_config* out, int32_t cap,
                                 int32_t* n);
/* Profiles every candidate on the context's GPU (CUDA-event timing: one
 * gate run, `warmup` >= 1 untimed runs, `runs` >= 3 timed runs, lower
 * median), disqualifies those deviating from the unfused cuBLASLt reference
 * by more than the bf16 gate (max|dY| / max|Y_ref| > 1e-2), selects by
 * (median, fusion preference, label), stores it for later NULL-cfg calls,
 * and persists it in the JSON cache at cache_path (NULL/"" = memory only;
 * format_version 1, flock-guarded, keyed by (B, d_model, d_ff, TP degree,
 * GPU fingerprint)).  A cache hit skips profiling.  *from_cache is set to
 * 1 on a hit.  results_json (optional) receives the ScheduleEntry as JSON. */
DFK_API int dfk_tune(dfk_context ctx, dfk_weights w, int64_t batch,
                     const char* cache_path, int32_t warmup, int32_t runs,
                     dfk_config* chosen, int32_t* from_cache,
                     char* results_json, size_t results_len);
/* The tuning cache on its own (cache_lookup / cache_store, tuner.hpp:102-113):
 * one JSON document {"format_version": 1, "entries": [...]} whose entries
 * are ScheduleEntry objects keyed by (shape.batch, shape.d_model,
 * shape.d_ff, fingerprint).  Lookup of an absent file or key sets *found = 0;
 * a corrupt file or another format_version is DFK_ERR_CACHE.  *needed
 * (optional) receives the entry's size incl. the NUL; a too-small buffer is
 * DFK_ERR_INVALID (entry_json may be NULL to query the size).  Store inserts
 * or replaces the entry with the same key; safe across threads and
 * processes, readers never see a partially written file. */
DFK_API int dfk_cache_lookup(const char* path, int64_t batch, int64_t d_model,
                             int64_t d_ff, const char* fingerprint,
                             char* entry_json, size_t len, size_t* needed,
                             int32_t* found);
DFK_API int dfk_cache_store(const char* path, const char* entry_json);
/* The configuration a NULL-cfg call with this B would use. */
DFK_API int dfk_select_config(dfk_context ctx, dfk_weights w, int64_t batch,
                              dfk_config* out);

/* --- tensor parallelism over NCCL -------------------------------------- */
/* ncclUniqueId is 128 bytes. */
DFK_API int dfk_tp_unique_id(void* id128);
/* Multi-process (one rank per GPU): every rank calls with the same id. */
DFK_API int dfk_tp_init(dfk_context ctx, const void* id128, int rank,
                        int nranks);
/* Single process driving `n` contexts on n devices (ncclCommInitAll). */
DFK_API int dfk_tp_init_all(dfk_context* ctxs, int n);
DFK_API int dfk_tp_rank(dfk_context ctx, int* rank, int* nranks);
/* Bracket per-device calls when ONE thread drives several ranks
 * (ncclGroupStart / ncclGroupEnd). */
DFK_API int dfk_tp_group_start(void);
DFK_API int dfk_tp_group_end(void);
/* Fused stage 1 + down on this rank's shard into fp32 partial Y, then one
 * in-place ncclAllReduce(sum) of B x d_model on the context stream (the one
 * collective of the compound scheme, tp.cpp:140-167). */
DFK_API int dfk_tp_forward(dfk_context ctx, dfk_weights w, const void* x,
                           int64_t batch, float* y, const dfk_config* cfg);
/* --- fused TP all-reduce over NVLink peer memory ----------------------- */
/* The block's one collective inside the block kernel:
 * down tile t is owned by rank t % P; every rank red.adds its fp32 partial
 * sums into the owner's workspace over NVLink, the CTA completing a tile
 * writes the full-sum Y into every rank's workspace, and each rank's launch
 * ends once all of its Y tiles are written.  Replaces dfk_tp_forward's
 * separate ncclAllReduce (tp.cpp:140-167 / simulated_all_reduce :90-105).
 *
 * dfk_tp_sym_create: allocates this rank's symmetric workspace for
 *   batch <= max_batch (<= 256) and d_model (% 4 == 0); writes its 64-byte
 *   CUDA IPC handle to ipc_handle64 (may be NULL).
 * dfk_tp_sym_open: multi-process -- handles = nranks x 64 bytes in rank
 *   order (every rank's dfk_tp_sym_create output, exchanged by the caller).
 * dfk_tp_sym_attach: one process driving n contexts (on n devices, or
 *   several contexts on ONE device as an emulation of n ranks).
 * dfk_tp_forward_fused: this rank's shard -- the balanced_ranges(d_ff, P)
 *   shard of its rank (anything else is DFK_ERR_INVALID) -- and Y (y_dtype
 *   F32 or BF16 [B x d_model], device) = the full sum over ranks, written
 *   by the block kernel itself: ONE launch per block, nothing after it.
 *   Every rank must issue it with the same batch.  A rank waits at most 4 s
 *   for its peers; then the launch ends with a wrong Y and the next
 *   dfk_context_sync returns DFK_ERR_TIMEOUT (the context stays usable;
 *   re-create the symmetric workspaces).  When ONE process drives several
 *   ranks, allocate every buffer before issuing the ranks' calls (a
 *   cudaMalloc may wait for the device, i.e. for a rank that waits for a
 *   peer not launched yet). */
DFK_API int dfk_tp_sym_create(dfk_context ctx, int64_t max_batch,
                              int64_t d_model, void* ipc_handle64);
DFK_API int dfk_tp_sym_open(dfk_context ctx, const void* handles, int rank,
                            int nranks);
DFK_API int dfk_tp_sym_attach(dfk_context* ctxs, int n);
DFK_API int dfk_tp_forward_fused(dfk_context ctx, dfk_weights w,
                                 const void* x, int64_t batch, void* y,
                                 int32_t y_dtype, const dfk_config* cfg);

/* balanced_ranges(extent, parts)[index] (tp.cpp:8-29). */
DFK_API int dfk_balanced_range(int64_t extent, int64_t parts, int64_t index,
                               int64_t* begin, int64_t* end);

/* --- traffic model ------------------------------------------------------ */
/* Algorithmic bytes of one fused block call at 2 B/element: the reference's
 * fused single-tile model, stage 1 + stage 2 (traffic.cpp:70-76, 82-94),
 * with d_ff the (shard) width. */
DFK_API int dfk_block_bytes(int64_t batch, int64_t d_model, int64_t d_ff,
                            int64_t* stage1, int64_t* stage2);

/* --- device memory / timing plumbing ----------------------------------- */
DFK_API int dfk_malloc(dfk_context ctx, size_t bytes, void** p);
DFK_API int dfk_free(dfk_context ctx, void* p);
DFK_API int dfk_host_alloc(size_t bytes, void** p); /* pinned */
DFK_API int dfk_host_free(void* p);
DFK_API int dfk_memcpy_h2d(dfk_context ctx, void* dst, const void* src,
                           size_t bytes);
DFK_API int dfk_memcpy_d2h(dfk_context ctx, void* dst, const void* src,
                           size_t bytes);
DFK_API int dfk_memset(dfk_context ctx, void* p, int value, size_t bytes);
/* Host-side element conversions of the reference-facing calls (the
 * reference's Matrix operands are fp64, tensor.hpp:73-128): round-to-nearest-
 * even to bf16 bits (NaN kept quiet, as the device rounds), or widen fp32 /
 * bf16 to the destination dtype.  Vectorised, on the calling thread. */
DFK_API int dfk_host_to_bf16(const void* src, int32_t src_dtype, size_t n,
                             uint16_t* dst);
DFK_API int dfk_host_from_f32(const float* src, size_t n, void* dst,
                              int32_t dst_dtype);
DFK_API int dfk_host_from_bf16(const uint16_t* src, size_t n, void* dst,
                               int32_t dst_dtype);
/* Fills a device bf16 buffer with uniform values in [lo, hi) (synthetic
 * bench inputs; counter-based hash, seed-deterministic). */
DFK_API int dfk_fill_uniform_bf16(dfk_context ctx, void* p, int64_t n,
                                  uint64_t seed, float lo, float hi);
DFK_API int dfk_event_create(void** ev);
DFK_API int dfk_event_destroy(void* ev);
DFK_API int dfk_event_record(dfk_context ctx, void* ev);
DFK_API int dfk_event_elapsed_ms(void* start, void* stop, float* ms);
/* Writes `bytes` of junk to a scratch buffer larger than L2 (flush). */
DFK_API int dfk_flush_l2(dfk_context ctx);
/* Kernel timeline tracing (diagnostics): while `buf` is non-NULL every
 * streaming-kernel launch of this context writes per-CTA globaltimer stamps
 * (64 x uint64 per CTA: start, producer done, consumer done, then per piece
 * issue / retire) into the device buffer `buf` of `slots` uint64.  NULL
 * turns tracing off (the default; zero cost). */
DFK_API int dfk_set_trace(dfk_context ctx, void* buf, int64_t slots);
/* Number of hot-path kernel launches issued by this context so far. */
DFK_API int dfk_launch_count(dfk_context ctx, int64_t* n);
/* Synchronises the context stream, then cudaProfilerStart (start != 0) or
 * cudaProfilerStop: brackets the launches an `ncu --profile-from-start off`
 * capture sees (the traffic-model assertion, tests/test_traffic_ncu.py). */
DFK_API int dfk_profiler_range(dfk_context ctx, int32_t start);

#ifdef __cplusplus
}
#endif

#endif /* DFK_H_ */
