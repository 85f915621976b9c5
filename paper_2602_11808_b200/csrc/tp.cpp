// tp.cpp — tensor parallelism over NCCL (the compound scheme of
// /root/reference/proj/src/tp.cpp:140-167): W_gate/W_up are column-sharded
// and W_down row-sharded over balanced_ranges(d_ff, P) (tp.cpp:8-29, done by
// dfk_weights_create's [ff_begin, ff_end)), each rank runs the fused stage 1
// and the down projection on its shard into an fp32 partial Y, and ONE
// ncclAllReduce(sum) of B x d_model per block combines them (the reference's
// simulated_all_reduce, tp.cpp:90-105; NCCL's summation order differs from
// device order, so results match within tolerance, not bitwise).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "layout.cuh"
#include "stream_kernels.cuh"

using namespace dfk;

namespace {

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(DFK_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

// One symmetric workspace per rank, identical layout on every rank (so a
// peer's buffers are at the same offsets from its base): fp32 down
// accumulator [max_b x t2*128], per-tile K-block counters, per-tile done
// words, and the full-sum Y slot [max_b x d_model] fp32.
struct SymLayout {
  size_t yacc, cnt, done, y, total;
  int t2;
};

size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

SymLayout sym_layout(int64_t max_b, int64_t dm) {
  SymLayout L;
  L.t2 = static_cast<int>((dm + kDownCols - 1) / kDownCols);
  size_t off = 0;
  L.yacc = off;
  off = align256(off + static_cast<size_t>(max_b) * L.t2 * kDownCols * 4);
  L.cnt = off;
  off = align256(off + static_cast<size_t>(L.t2) * 4);
  L.done = off;
  off = align256(off + static_cast<size_t>(L.t2) * 4);
  L.y = off;
  off = align256(off + static_cast<size_t>(max_b * dm) * 4);
  L.total = off;
  return L;
}

void close_peers(dfk_context_s* ctx) {
  for (int r = 0; r < 8; ++r) {
    if (ctx->tp_peer_ipc[r] && ctx->tp_peer[r]) cudaIpcCloseMemHandle(ctx->tp_peer[r]);
    ctx->tp_peer[r] = nullptr;
    ctx->tp_peer_ipc[r] = false;
  }
  ctx->tp_colocated = false;
}

}  // namespace

namespace dfk {

bool tp_active(const dfk_context_s* ctx) {
  return ctx->tp_sym_size > 1 || (ctx->comm && ctx->nranks > 1);
}

int tp_block(dfk_context_s* ctx, dfk_weights_s* w, const void* x, int64_t B,
             float* y, const dfk_config* cfg) {
  if (ctx->tp_sym_size > 1) return tp_forward_fused_impl(ctx, w, x, B, y, DFK_F32, cfg);
  return dfk_tp_forward(ctx, w, x, B, y, cfg);
}

int tp_forward_fused_impl(dfk_context_s* ctx, dfk_weights_s* w, const void* x,
                          int64_t batch, void* y, int y_dtype, const dfk_config* cfg) {
  if (!ctx || !w) return fail(DFK_ERR_INVALID, "null handle");
  if (w->ctx != ctx) return fail(DFK_ERR_INVALID, "weights belong to another context");
  if (!w->s1_pack || !w->dn_pack)
    return fail(DFK_ERR_INVALID, "the TP block needs all three weight matrices");
  if (!x || !y) return fail(DFK_ERR_INVALID, "null activation pointer");
  if (batch < 1) return fail(DFK_ERR_SHAPE, "batch must be >= 1");
  if (y_dtype != DFK_F32 && y_dtype != DFK_BF16)
    return fail(DFK_ERR_INVALID, "y_dtype must be F32 or BF16");
  if (ctx->tp_sym_size < 1 || !ctx->tp_sym.p)
    return fail(DFK_ERR_INVALID, "dfk_tp_sym_create / _open / _attach first");
  const int P = ctx->tp_sym_size;
  if (P == 1) return forward_impl(ctx, w, x, batch, y, y_dtype, cfg);
  if (batch > ctx->tp_max_b)
    return fail(DFK_ERR_SHAPE, "batch exceeds the symmetric workspace's max_batch");
  if (w->d_model != ctx->tp_dm)
    return fail(DFK_ERR_SHAPE, "weights' d_model differs from the symmetric workspace");
  // A tile is complete when the K blocks of ALL ranks' shards have arrived;
  // every rank derives that total from balanced_ranges, so each rank must
  // hold exactly its balanced shard (tp.cpp:8-29, make_plan :55-61).
  int64_t mb = 0, me = 0;
  DFK_TRY(dfk_balanced_range(w->d_ff_total, P, ctx->tp_sym_rank, &mb, &me));
  if (w->ff_begin != mb || w->ff_begin + w->d_ff != me)
    return fail(DFK_ERR_INVALID,
                "fused TP: rank " + std::to_string(ctx->tp_sym_rank) + " holds d_ff [" +
                    std::to_string(w->ff_begin) + ", " + std::to_string(w->ff_begin + w->d_ff) +
                    ") but the all-reduce expects its balanced_ranges shard [" +
                    std::to_string(mb) + ", " + std::to_string(me) +
                    ") (use dfk_tp_forward for other plans)");
  dfk_config c;
  DFK_TRY(resolve_config(ctx, w, batch, cfg, &c));
  c.variant = DFK_VARIANT_FUSED;  // the all-reduce lives in the block kernel
  c.block_kernel = 1;
  c.dynamic_sched = 1;
  c.s1_split_k = 1;
  // Down K blocks contributed to every tile by all ranks (shards may differ
  // by one column, balanced_ranges tp.cpp:8-29).
  int total_kb = 0;
  for (int r = 0; r < P; ++r) {
    int64_t b = 0, e = 0;
    DFK_TRY(dfk_balanced_range(w->d_ff_total, P, r, &b, &e));
    total_kb += static_cast<int>((e - b + kBlockK - 1) / kBlockK);
  }
  const SymLayout L = sym_layout(ctx->tp_max_b, ctx->tp_dm);
  StreamArgs t = {};
  t.tp_rank = ctx->tp_sym_rank;
  t.tp_size = P;
  t.tp_total_kb = total_kb;
  t.yacc_ld = L.t2 * kDownCols;
  for (int r = 0; r < P; ++r) {
    auto* base = static_cast<uint8_t*>(ctx->tp_peer[r]);
    if (!base) return fail(DFK_ERR_INVALID, "peer workspace missing");
    t.tp_yacc[r] = reinterpret_cast<float*>(base + L.yacc);
    t.tp_cnt[r] = reinterpret_cast<int*>(base + L.cnt);
    t.tp_done[r] = reinterpret_cast<int*>(base + L.done);
    t.tp_y[r] = reinterpret_cast<float*>(base + L.y);
  }
  DFK_CUDA(cudaSetDevice(ctx->device));
  return block_fused_tp(ctx, w, x, batch, y, y_dtype == DFK_BF16, c, &t);
}

}  // namespace dfk

extern "C" {

int dfk_tp_unique_id(void* id128) {
  if (!id128) return fail(DFK_ERR_INVALID, "null id buffer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id128, &id, sizeof(id));
  return DFK_OK;
}

int dfk_tp_init(dfk_context ctx, const void* id128, int rank, int nranks) {
  if (!ctx || !id128) return fail(DFK_ERR_INVALID, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(DFK_ERR_INVALID, "bad rank/nranks");
  DFK_CUDA(cudaSetDevice(ctx->device));
  if (ctx->comm) {
    ncclCommDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  ctx->rank = rank;
  ctx->nranks = nranks;
  return DFK_OK;
}

int dfk_tp_init_all(dfk_context* ctxs, int n) {
  if (!ctxs || n < 1) return fail(DFK_ERR_INVALID, "bad context list");
  std::vector<int> devs(n);
  std::vector<ncclComm_t> comms(n);
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i]) return fail(DFK_ERR_INVALID, "null context in list");
    devs[i] = ctxs[i]->device;
  }
  ncclResult_t r = ncclCommInitAll(comms.data(), n, devs.data());
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitAll");
  for (int i = 0; i < n; ++i) {
    if (ctxs[i]->comm) ncclCommDestroy(ctxs[i]->comm);
    ctxs[i]->comm = comms[i];
    ctxs[i]->rank = i;
    ctxs[i]->nranks = n;
  }
  return DFK_OK;
}

int dfk_tp_rank(dfk_context ctx, int* rank, int* nranks) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  if (rank) *rank = ctx->rank;
  if (nranks) *nranks = ctx->nranks;
  return DFK_OK;
}

int dfk_tp_group_start(void) {
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  return DFK_OK;
}

int dfk_tp_group_end(void) {
  ncclResult_t r = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return DFK_OK;
}

int dfk_tp_forward(dfk_context ctx, dfk_weights w, const void* x,
                   int64_t batch, float* y, const dfk_config* cfg) {
  if (!ctx || !w) return fail(DFK_ERR_INVALID, "null handle");
  DFK_TRY(forward_impl(ctx, w, x, batch, y, DFK_F32, cfg));
  if (ctx->comm && ctx->nranks > 1) {
    ncclResult_t r =
        ncclAllReduce(y, y, static_cast<size_t>(batch * w->d_model), ncclFloat,
                      ncclSum, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  }
  return DFK_OK;
}

// ---------------------------------------------------------------------------
// Fused TP all-reduce over NVLink peer memory.
// ---------------------------------------------------------------------------
int dfk_tp_sym_create(dfk_context ctx, int64_t max_batch, int64_t d_model,
                      void* ipc_handle64) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  if (max_batch < 1 || max_batch > 256 || d_model < 4 || d_model % 4)
    return fail(DFK_ERR_SHAPE, "fused TP needs 1 <= max_batch <= 256 and d_model % 4 == 0");
  DFK_CUDA(cudaSetDevice(ctx->device));
  close_peers(ctx);
  if (ctx->tp_sym.p) {
    cudaFree(ctx->tp_sym.p);
    ctx->tp_sym = {};
  }
  const SymLayout L = sym_layout(max_batch, d_model);
  DFK_CUDA(cudaMalloc(&ctx->tp_sym.p, L.total));
  ctx->tp_sym.bytes = L.total;
  DFK_CUDA(cudaMemsetAsync(ctx->tp_sym.p, 0, L.total, ctx->stream));
  DFK_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->tp_max_b = max_batch;
  ctx->tp_dm = d_model;
  ctx->tp_sym_rank = 0;
  ctx->tp_sym_size = 1;
  ctx->tp_peer[0] = ctx->tp_sym.p;
  if (ipc_handle64) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    cudaIpcMemHandle_t h;
    DFK_CUDA(cudaIpcGetMemHandle(&h, ctx->tp_sym.p));
    std::memcpy(ipc_handle64, &h, sizeof(h));
  }
  return DFK_OK;
}

int dfk_tp_sym_open(dfk_context ctx, const void* handles, int rank, int nranks) {
  if (!ctx || !handles) return fail(DFK_ERR_INVALID, "null argument");
  if (!ctx->tp_sym.p) return fail(DFK_ERR_INVALID, "dfk_tp_sym_create first");
  if (nranks < 1 || nranks > kMaxTp || rank < 0 || rank >= nranks)
    return fail(DFK_ERR_INVALID, "bad rank/nranks (fused TP supports up to 8 ranks)");
  DFK_CUDA(cudaSetDevice(ctx->device));
  close_peers(ctx);
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) {
      ctx->tp_peer[r] = ctx->tp_sym.p;
      continue;
    }
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      close_peers(ctx);
      return fail(DFK_ERR_CUDA, std::string("cudaIpcOpenMemHandle(rank ") +
                                    std::to_string(r) + "): " + cudaGetErrorString(e));
    }
    ctx->tp_peer[r] = p;
    ctx->tp_peer_ipc[r] = true;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, p) == cudaSuccess) {
      if (pa.device == ctx->device) ctx->tp_colocated = true;
    } else {
      cudaGetLastError();
    }
  }
  ctx->tp_sym_rank = rank;
  ctx->tp_sym_size = nranks;
  return DFK_OK;
}

int dfk_tp_sym_attach(dfk_context* ctxs, int n) {
  if (!ctxs || n < 1 || n > kMaxTp) return fail(DFK_ERR_INVALID, "bad context list");
  for (int i = 0; i < n; ++i) {
    if (!ctxs[i] || !ctxs[i]->tp_sym.p)
      return fail(DFK_ERR_INVALID, "every context needs dfk_tp_sym_create first");
    if (ctxs[i]->tp_max_b != ctxs[0]->tp_max_b || ctxs[i]->tp_dm != ctxs[0]->tp_dm)
      return fail(DFK_ERR_SHAPE, "symmetric workspaces differ in max_batch / d_model");
  }
  for (int i = 0; i < n; ++i) {
    DFK_CUDA(cudaSetDevice(ctxs[i]->device));
    close_peers(ctxs[i]);
    for (int j = 0; j < n; ++j) {
      if (j != i && ctxs[j]->device == ctxs[i]->device) ctxs[i]->tp_colocated = true;
      if (ctxs[j]->device != ctxs[i]->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(ctxs[j]->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else if (e != cudaSuccess) {
          return fail(DFK_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") +
                                        cudaGetErrorString(e));
        }
      }
      ctxs[i]->tp_peer[j] = ctxs[j]->tp_sym.p;
    }
    ctxs[i]->tp_sym_rank = i;
    ctxs[i]->tp_sym_size = n;
  }
  return DFK_OK;
}

int dfk_tp_forward_fused(dfk_context ctx, dfk_weights w, const void* x,
                         int64_t batch, void* y, int32_t y_dtype, const dfk_config* cfg) {
  return tp_forward_fused_impl(ctx, w, x, batch, y, y_dtype, cfg);
}

}  // extern "C"
