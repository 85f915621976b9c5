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

using namespace dfk;

namespace {

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(DFK_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

}  // namespace

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

}  // extern "C"
