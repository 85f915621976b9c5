// internal.h — library-private state behind the dfk.h handles.
#pragma once

#include <cublasLt.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "dfk.h"

namespace dfk {

// Error plumbing: thread-local message + status, no exceptions across the
// ABI.
struct Error {
  int status;
  std::string msg;
};
void set_error(int status, const std::string& msg);
int fail(int status, const std::string& msg);

#define DFK_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess)                                                 \
      return ::dfk::fail(DFK_ERR_CUDA, std::string(#call) + ": " +         \
                                           cudaGetErrorString(e_));        \
  } while (0)

#define DFK_TRY(call)             \
  do {                            \
    int s_ = (call);              \
    if (s_ != DFK_OK) return s_;  \
  } while (0)

struct DeviceBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// One X staging slot of the host-buffer forward (dfk_forward_host_async).
struct HostSlot {
  DeviceBuf x, y;
};
constexpr int kHostSlots = 8;

// A captured decode sequence (decode.cpp) and its kernel launch count.
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
  uint64_t generation = 0;  // ctx->generation when captured
};

}  // namespace dfk

struct dfk_context_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 0;
  int max_smem_optin = 0;
  int l2_bytes = 0;
  std::string name;
  int cc_major = 0, cc_minor = 0;
  int driver_version = 0;
  int64_t launches = 0;
  // Bumped by every scratch (re)allocation and weight-set destruction: the
  // addresses a captured decode graph baked in are valid while it holds.
  uint64_t generation = 0;

  // Scratch (grown on demand, never shrunk).
  dfk::DeviceBuf a2;       // internal A2 of dfk_forward
  dfk::DeviceBuf xpad;     // padded activations for unaligned shapes
  dfk::DeviceBuf a2pad;    // padded A2 for dfk_down with unaligned d_ff
  dfk::DeviceBuf yacc;     // fp32 down accumulator (kept all-zero)
  dfk::DeviceBuf counters; // per-tile down arrival counters (kept zero)
  dfk::DeviceBuf flags;    // per-stage-1-tile completion flags (block kernel)
  dfk::DeviceBuf sched;    // dynamic-scheduler counters (kept zero between launches)
  dfk::DeviceBuf s1acc;    // stage-1 stream-K fp32 partial sums (kept all-zero)
  dfk::DeviceBuf s1cnt;    // stage-1 stream-K per-tile arrival counters (kept zero)
  dfk::DeviceBuf mat_scratch;  // MaterializeIntermediate control's A_silu (tests)
  unsigned epoch = 0;      // block-kernel launch epoch (flag value)
  unsigned long long* trace = nullptr;  // dfk_set_trace buffer
  int64_t trace_slots = 0;
  dfk::DeviceBuf concat;   // unfused comparator intermediates
  dfk::DeviceBuf tmp1, tmp2;
  dfk::DeviceBuf lt_ws;    // cuBLASLt workspace
  dfk::DeviceBuf flush;    // L2 flush buffer
  dfk::DeviceBuf hx_dev, hy_dev;  // forward_host device staging
  dfk::HostSlot host_slots[dfk::kHostSlots];
  int host_next = 0;
  // Copy-engine X path of the host-buffer forward: side stream, per-slot
  // device flags (x_ready / x_free, uint32 [kHostSlots] each), sequence no.,
  // and the flags of the call being launched (consumed by block_fused).
  cudaStream_t side_stream = nullptr;   // X H2D copies
  cudaStream_t out_stream = nullptr;    // Y D2H copies
  dfk::DeviceBuf host_flags;
  unsigned host_seq = 0;
  const unsigned* pend_x_ready = nullptr;
  unsigned* pend_x_free = nullptr;
  unsigned* pend_y_done = nullptr;
  unsigned pend_x_seq = 0;
  void* hx_pinned = nullptr;
  size_t hx_pinned_bytes = 0;
  void* hy_pinned = nullptr;
  size_t hy_pinned_bytes = 0;

  cublasLtHandle_t lt = nullptr;
  std::map<std::tuple<int64_t, int64_t, int64_t, int>, cublasLtMatmulAlgo_t>
      lt_algos;

  // TMA descriptors keyed by (ptr, inner extent, rows, row stride, box rows).
  std::map<std::tuple<uintptr_t, int64_t, int64_t, int64_t, int>, CUtensorMap>
      tmaps;

  // NCCL tensor parallelism.
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;

  // Fused TP all-reduce (tp.cpp): this rank's symmetric workspace
  // (IPC-exportable) and every rank's workspace base as seen from here.
  dfk::DeviceBuf tp_sym;
  int64_t tp_max_b = 0, tp_dm = 0;
  int tp_sym_rank = 0, tp_sym_size = 0;
  // Host-mapped error word (cudaHostAllocMapped): kernels set it when a
  // cross-rank wait times out; dfk_context_sync reports and clears it.
  int* err_host = nullptr;
  int* err_dev = nullptr;
  void* tp_peer[8] = {};
  bool tp_peer_ipc[8] = {};
  // Some peer rank runs on THIS GPU (tests emulate ranks this way): its
  // kernels must be able to become resident next to ours, so fused-TP
  // launches take at most sm_count / P CTAs and let the next launch in the
  // stream start only after their Y is complete (see the kernel's PDL
  // trigger).
  bool tp_colocated = false;

  // Decode loop (decode.cpp): bf16 ping-pong activations, fp32 TP partial,
  // captured sequences keyed by (layers, batch, steps, buffers, config).
  dfk::DeviceBuf dec[2];
  dfk::DeviceBuf dec_f32;
  std::map<std::string, dfk::GraphEntry> graphs;

  // Weight handles registered on this context (freed with it).
  std::set<dfk_weights_s*> weights;

  // Scheduler decisions: (batch, d_model, d_ff shard) -> config.
  std::map<std::tuple<int64_t, int64_t, int64_t>, dfk_config> chosen;
  std::mutex mu;
};

struct dfk_weights_s {
  dfk_context_s* ctx = nullptr;
  int64_t d_model = 0, d_ff = 0, ff_begin = 0, d_ff_total = 0;
  // Stage 1: tiles of 64 A2 columns, K blocks over d_model.
  int s1_tiles = 0, s1_kblocks = 0;
  uint8_t* s1_pack = nullptr;
  // Down: tiles of 128 Y columns, K blocks over d_ff.
  int dn_tiles = 0, dn_kblocks = 0;
  uint8_t* dn_pack = nullptr;
  // Unfused comparator (built lazily from the packs): K-major bf16
  // W_cat^T [2 d_ff x d_model] (gate rows first) and W_down^T
  // [d_model x d_ff].
  __nv_bfloat16* cat_t = nullptr;
  __nv_bfloat16* down_t = nullptr;
};

namespace dfk {

// Kernels in aux_kernels.cu.
cudaError_t launch_pack_stage1(const void* w_gate, const void* w_up, int dtype,
                               int64_t d_model, int64_t d_ff_total,
                               int64_t ff_begin, int64_t d_ff, int tiles,
                               int kblocks, uint8_t* dst, cudaStream_t s);
cudaError_t launch_pack_down(const void* w_down, int dtype, int64_t d_model,
                             int64_t ff_begin, int64_t d_ff, int tiles,
                             int kblocks, uint8_t* dst, cudaStream_t s);
cudaError_t launch_unpack_stage1(const uint8_t* pack, int64_t d_model,
                                 int64_t d_ff, int tiles, int kblocks,
                                 __nv_bfloat16* cat_t, cudaStream_t s);
cudaError_t launch_unpack_down(const uint8_t* pack, int64_t d_model,
                               int64_t d_ff, int tiles, int kblocks,
                               __nv_bfloat16* down_t, cudaStream_t s);
cudaError_t launch_pad_rows(const __nv_bfloat16* src, int64_t rows,
                            int64_t cols, int64_t ld_src, __nv_bfloat16* dst,
                            int64_t ld_dst, cudaStream_t s);
cudaError_t launch_silu_mul(const __nv_bfloat16* gate, int64_t ld_gate,
                            const __nv_bfloat16* up, int64_t ld_up,
                            __nv_bfloat16* out, int64_t rows, int64_t cols,
                            cudaStream_t s);
cudaError_t launch_silu(const __nv_bfloat16* in, __nv_bfloat16* out,
                        int64_t n, cudaStream_t s);
cudaError_t launch_mul(const __nv_bfloat16* a, const __nv_bfloat16* b,
                       __nv_bfloat16* out, int64_t n, cudaStream_t s);
cudaError_t launch_fill_uniform_bf16(__nv_bfloat16* p, int64_t n,
                                     uint64_t seed, float lo, float hi,
                                     cudaStream_t s);
cudaError_t launch_flush(void* p, size_t bytes, cudaStream_t s);
cudaError_t launch_f32_to_bf16(const float* in, __nv_bfloat16* out, int64_t n,
                               cudaStream_t s);
cudaError_t preload_aux_kernels();
cudaError_t launch_stage_rows(const void* src, void* dst, int64_t bytes,
                              cudaStream_t s);

// Makes ctx's device current (one host thread may drive contexts on several
// devices, e.g. the C++ shim's run_tp_mlp); every entry point that launches
// or copies calls it.
inline int use_device(dfk_context_s* ctx);

// api.cu helpers used by the scheduler / TP translation units.
int resolve_config(dfk_context_s* ctx, dfk_weights_s* w, int64_t B,
                   const dfk_config* in, dfk_config* out);
void default_config(dfk_context_s* ctx, dfk_weights_s* w, int64_t B,
                    dfk_config* out);
int forward_impl(dfk_context_s* ctx, dfk_weights_s* w, const void* x,
                 int64_t B, void* y, int y_dtype, const dfk_config* cfg);
// An unregistered device copy of w's packs (the scheduler's rotating
// weight sets: sub-L2 shards are timed cold, as in a layer chain), and its
// release.
int clone_weights(dfk_context_s* ctx, const dfk_weights_s* w, dfk_weights_s** out);
void release_clone(dfk_weights_s* w);
// Tensor-parallel degree a context / weight set stands for (the NCCL or
// fused-TP rank count, or d_ff_total / d_ff of a balanced shard).
int tp_degree(const dfk_context_s* ctx, const dfk_weights_s* w);
struct StreamArgs;
// One tensor-parallel block into fp32 Y (tp.cpp): the fused all-reduce when
// the symmetric workspaces are set up, else the NCCL all-reduce, else
// (single rank) the plain block.
int tp_block(dfk_context_s* ctx, dfk_weights_s* w, const void* x, int64_t B,
             float* y, const dfk_config* cfg);
// The fused-TP block into Y of either dtype (F32 / BF16).
int tp_forward_fused_impl(dfk_context_s* ctx, dfk_weights_s* w, const void* x,
                          int64_t B, void* y, int y_dtype, const dfk_config* cfg);
bool tp_active(const dfk_context_s* ctx);
// The block kernel with the fused TP all-reduce (tp.cpp): `tp` carries the
// tp_* fields of StreamArgs; y is this rank's symmetric output.
int block_fused_tp(dfk_context_s* ctx, dfk_weights_s* w, const void* x, int64_t B,
                   void* y, bool y_bf16, const dfk_config& cfg, const StreamArgs* tp);
int ensure_buf(dfk_context_s* ctx, DeviceBuf& b, size_t bytes, bool zero, cudaStream_t s);
std::string config_label(const dfk_config& c);
// Host-side conversions on the worker pool (host_convert.cpp).
void host_to_bf16(const void* src, int dtype, size_t n, uint16_t* dst);
void host_from_f32(const float* src, size_t n, void* dst, int dtype);
void host_from_bf16(const uint16_t* src, size_t n, void* dst, int dtype);
// Tuning cache (tuning_cache.cpp): lookup (false + *err set on a bad file)
// and insert-or-replace ("" on success, else the error).
bool cache_find(const std::string& path, int64_t B, int64_t dm, int64_t df,
                const std::string& fp, std::string* hit, std::string* err);
std::string cache_put(const std::string& path, const std::string& entry_text);

}  // namespace dfk

namespace dfk {
inline int use_device(dfk_context_s* ctx) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != ctx->device) {
    const cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess)
      return fail(DFK_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  return DFK_OK;
}
}  // namespace dfk
