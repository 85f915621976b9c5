// decode.cpp — the multi-layer decode loop (the reference's
// time_decode_seconds, /root/reference/proj/src/bench.cpp:98-115: `steps`
// passes over L layers, x <- Y after every block) on the GPU, optionally
// captured ONCE into a CUDA graph and replayed.
//
// The chain is bf16 (Y of block l is X of block l+1, rounded RNE), which is
// what a decoder feeds its next layer.  Each block is one persistent
// kernel launch (or the configured layout), chained by programmatic
// dependent launch; under TP every block ends in its all-reduce.
//
// Graph replay and the block kernel's stage-1 completion flags: a launch
// waits for flags == its epoch, and epochs are baked into the captured
// launches.  A captured sequence has >= 2 launches with distinct epochs, so
// at the start of every launch the flags hold the PREVIOUS launch's epoch
// (the graph's last one, or a newer eager launch's) -- never its own.
// Single-call sequences are therefore never captured.  When the layers'
// stage-1 tile counts differ, the graph starts with a memset of the flags
// (tiles only one layer has would otherwise keep that layer's epoch from
// the previous replay).  Every graph records ctx->generation at capture and
// is re-captured when a scratch buffer has been reallocated since.
#include <cuda_runtime.h>

#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "internal.h"

using namespace dfk;

namespace {

// One block of the chain: Y (bf16) = MLP(X); under TP the fp32 partial is
// all-reduced and rounded to bf16.
int chain_block(dfk_context_s* ctx, dfk_weights_s* w, const void* x,
                int64_t B, void* y_bf16, const dfk_config* cfg) {
  // Fused all-reduce: the block kernel writes the all-reduced bf16 Y itself.
  if (ctx->tp_sym_size > 1)
    return tp_forward_fused_impl(ctx, w, x, B, y_bf16, DFK_BF16, cfg);
  if (tp_active(ctx)) {  // NCCL comparator: fp32 partial, all-reduce, round
    const size_t n = static_cast<size_t>(B * w->d_model);
    DFK_TRY(ensure_buf(ctx, ctx->dec_f32, n * 4, false, ctx->stream));
    float* yf = static_cast<float*>(ctx->dec_f32.p);
    DFK_TRY(tp_block(ctx, w, x, B, yf, cfg));
    cudaError_t e = launch_f32_to_bf16(yf, static_cast<__nv_bfloat16*>(y_bf16),
                                       static_cast<int64_t>(n), ctx->stream);
    if (e != cudaSuccess) return fail(DFK_ERR_CUDA, cudaGetErrorString(e));
    ctx->launches++;
    return DFK_OK;
  }
  return forward_impl(ctx, w, x, B, y_bf16, DFK_BF16, cfg);
}

int run_chain(dfk_context_s* ctx, dfk_weights_s* const* layers, int L,
              const void* x, int64_t B, int steps, void* y_out,
              const dfk_config* cfg, bool reset_flags = false) {
  const int64_t total = static_cast<int64_t>(L) * steps;
  if (reset_flags && ctx->flags.p)
    DFK_CUDA(cudaMemsetAsync(ctx->flags.p, 0, ctx->flags.bytes, ctx->stream));
  const size_t bytes = static_cast<size_t>(B * layers[0]->d_model) * 2;
  // Every scratch buffer of the chain exists before the first launch: a
  // cudaMalloc between launches may wait for the device, which under the
  // fused TP all-reduce would wait for this rank's peers (themselves waiting
  // for our next launch when one process drives several ranks).
  DFK_TRY(ensure_buf(ctx, ctx->dec[0], bytes, false, ctx->stream));
  DFK_TRY(ensure_buf(ctx, ctx->dec[1], bytes, false, ctx->stream));
  if (tp_active(ctx) && ctx->tp_sym_size <= 1)
    DFK_TRY(ensure_buf(ctx, ctx->dec_f32, bytes * 2, false, ctx->stream));
  const void* cur = x;
  int64_t k = 0;
  for (int s = 0; s < steps; ++s) {
    for (int l = 0; l < L; ++l, ++k) {
      void* out;
      if (k == total - 1 && y_out != cur) {
        out = y_out;
      } else {
        DeviceBuf& b = ctx->dec[k & 1];
        DFK_TRY(ensure_buf(ctx, b, bytes, false, ctx->stream));
        out = b.p;
        if (out == cur) {  // never read and write the same buffer
          DeviceBuf& o = ctx->dec[(k + 1) & 1];
          DFK_TRY(ensure_buf(ctx, o, bytes, false, ctx->stream));
          out = o.p;
        }
      }
      DFK_TRY(chain_block(ctx, layers[l], cur, B, out, cfg));
      cur = out;
    }
  }
  if (cur != y_out)
    DFK_CUDA(cudaMemcpyAsync(y_out, cur, bytes, cudaMemcpyDeviceToDevice,
                             ctx->stream));
  return DFK_OK;
}

std::string graph_key(dfk_context_s* ctx, dfk_weights_s* const* layers, int L,
                      const void* x, int64_t B, int steps, const void* y_out,
                      const dfk_config* cfg) {
  std::ostringstream o;
  o << B << ':' << steps << ':' << x << ':' << y_out << ':';
  for (int l = 0; l < L; ++l) o << layers[l] << ',';
  // The resolved configuration (a NULL cfg follows later tuning decisions).
  dfk_config r;
  if (resolve_config(ctx, layers[0], B, cfg, &r) == DFK_OK) o << config_label(r);
  if (cfg) o << ":s" << cfg->s1_stages << cfg->down_stages << cfg->kbs << cfg->chunk_kb;
  return o.str();
}

}  // namespace

extern "C" {

int dfk_decode(dfk_context ctx, const dfk_weights* layers, int32_t n_layers,
               const void* x, int64_t batch, int32_t steps, void* y_out,
               const dfk_config* cfg, int32_t use_graph) {
  if (!ctx) return fail(DFK_ERR_INVALID, "null context");
  if (!layers || n_layers < 1) return fail(DFK_ERR_INVALID, "need >= 1 layer");
  if (steps < 1) return fail(DFK_ERR_INVALID, "steps must be >= 1");
  if (!x || !y_out) return fail(DFK_ERR_INVALID, "null activation pointer");
  if (batch < 1)
    return fail(DFK_ERR_SHAPE, "batch must be >= 1, got " + std::to_string(batch));
  std::vector<dfk_weights_s*> ws(static_cast<size_t>(n_layers));
  for (int l = 0; l < n_layers; ++l) {
    ws[l] = layers[l];
    if (!ws[l]) return fail(DFK_ERR_INVALID, "null layer handle");
    if (ws[l]->ctx != ctx)
      return fail(DFK_ERR_INVALID, "layer belongs to another context");
    if (!ws[l]->s1_pack || !ws[l]->dn_pack)
      return fail(DFK_ERR_INVALID, "a decode layer needs all three weight matrices");
    if (ws[l]->d_model != ws[0]->d_model)
      return fail(DFK_ERR_SHAPE, "layers disagree on d_model (x <- Y chain)");
  }
  DFK_CUDA(cudaSetDevice(ctx->device));
  const int64_t total = static_cast<int64_t>(n_layers) * steps;
  if (!use_graph || total < 2)
    return run_chain(ctx, ws.data(), n_layers, x, batch, steps, y_out, cfg);

  const std::string key =
      graph_key(ctx, ws.data(), n_layers, x, batch, steps, y_out, cfg);
  auto it = ctx->graphs.find(key);
  bool recapture = false;
  if (it != ctx->graphs.end() && it->second.generation != ctx->generation) {
    // A scratch buffer was reallocated (or a weight set destroyed) since the
    // capture: the baked addresses may be stale.  Drop and re-capture.
    cudaGraphExecDestroy(it->second.exec);
    ctx->graphs.erase(it);
    it = ctx->graphs.end();
    recapture = true;
  }
  if (it == ctx->graphs.end()) {
    // Eager pass first: grows every scratch buffer, builds the TMA
    // descriptors and opts the kernels in to their shared memory, so that
    // the capture below records launches only.  A re-capture under TP skips
    // it (buffers only grow, so they are sized already; an extra eager
    // sequence on one rank would not be matched by its peers).
    if (!(recapture && tp_active(ctx)))
      DFK_TRY(run_chain(ctx, ws.data(), n_layers, x, batch, steps, y_out, cfg));
    // Layers with different stage-1 tile counts: a layer's flags beyond the
    // others' tiles would still hold its own baked epoch from the previous
    // replay, so every replay starts from zeroed flags.
    bool uneven = false;
    for (int l = 1; l < n_layers; ++l) uneven |= ws[l]->s1_tiles != ws[0]->s1_tiles;
    const int64_t l0 = ctx->launches;
    DFK_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    const int st = run_chain(ctx, ws.data(), n_layers, x, batch, steps, y_out, cfg, uneven);
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
    if (st != DFK_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (ec != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      return fail(DFK_ERR_CUDA, std::string("decode graph capture: ") +
                                    cudaGetErrorString(ec));
    }
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess)
      return fail(DFK_ERR_CUDA, std::string("decode graph instantiate: ") +
                                    cudaGetErrorString(ei));
    if (ctx->graphs.size() >= 64) {
      for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second.exec);
      ctx->graphs.clear();
    }
    it = ctx->graphs.emplace(key, GraphEntry{ex, ctx->launches - l0, ctx->generation}).first;
    ctx->launches = l0;  // counted on replay
  }
  DFK_CUDA(cudaGraphLaunch(it->second.exec, ctx->stream));
  ctx->launches += it->second.launches;
  return DFK_OK;
}

}  // extern "C"
