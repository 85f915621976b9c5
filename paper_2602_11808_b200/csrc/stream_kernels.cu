// stream_kernels.cu — the hot path: weight-streaming kernels for the fused
// SwiGLU MLP on sm_100a.
//
// One kernel template covers every stage of the block and both consumer
// families:
//
//   kModeStage1  A2 = (X W_up) * silu(X W_gate)  (fused.cpp:74-168,
//                DeepFusionKernel: gate and up accumulate side by side, the
//                SiLU*up epilogue runs once per element after the FULL K
//                reduction, A2 is the only global write)
//   kModeDown    Y = A2 W_down                   (swiglu.cpp:214-226)
//   kModeBlock   both in ONE persistent launch (run_fused, fused.cpp:209-216)
//
//   tcgen05 family  weights are the MMA M=128 operand, the batch is MMA N
//                   (swap-AB), fp32 accumulators in TMEM, epilogue through
//                   tcgen05.ld
//   GEMV family     8 CUDA-core warps dot the same smem stages with fp32
//                   FMAs and warp-shuffle reductions (batch <= 8)
//
// Skeleton (warp-specialised, persistent, one CTA per SM):
//   warp 0      producer: weight K blocks (16 KiB, pre-swizzled in HBM) with
//               1-D bulk copies (cp.async.bulk, L2 evict_first) + the
//               activation rows of the same K blocks with 2-D TMA (128B
//               swizzle); `kbs` blocks per ring stage (32 KiB copies stream
//               at ~7 TB/s, tools/stream_probe.cu).  The first ring's weight
//               copies are issued BEFORE griddepcontrol.wait, so under PDL
//               they overlap the previous kernel's tail.
//   warp 1      tcgen05: one lane issues 4 MMAs (M128 x N x K16) per K block
//               and tcgen05.commit's the slot back to the producer.
//   warps 2-5   tcgen05 epilogue (TMEM lane quarter = warp % 4).
//   warps 1-8   GEMV family math warps (no TMEM).
//
// Work is a sequence of "pieces" (one tile, a contiguous K-block range):
//   stage-1 pieces are whole tiles (64 A2 columns x all of d_model) handed
//   out round-robin, so partial gate/up sums never leave the SM;
//   down pieces come from a stream-K split of the flattened (tile, K block)
//   space: partial sums go to an fp32 workspace with red.global.add and the
//   CTA completing a tile's last piece converts it to the output dtype and
//   re-zeroes the workspace (no memset, ever).
//   kModeBlock orders the down space wave-major (all K blocks whose stage-1
//   tile is computed in round-robin wave 0 first, ...) and gives each CTA a
//   byte-balanced share: CTAs with fewer stage-1 tiles take more down work,
//   starting on K blocks whose A2 is already published.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

#include "layout.cuh"
#include "ptx.cuh"
#include "stream_kernels.cuh"

namespace dfk {

namespace {

constexpr int kTcThreads = 192;    // producer, MMA, 4 epilogue warps
constexpr int kGemvThreads = 288;  // producer + 8 math warps
constexpr int kGemvWarps = 8;
constexpr int kMaxKbs = 4;

// ---------------------------------------------------------------------------
// Work plan.
// ---------------------------------------------------------------------------
struct Piece {
  int down;  // 0 = stage-1 tile, 1 = down piece
  int tile;
  int kb0, kb1;
};

struct Plan {
  int mode;
  int G, c;
  int split;        // CTAs per stage-1 tile (cluster size), 1 = none
  int q, Q;         // cluster index of this CTA, number of clusters
  int krank;        // rank in the cluster = K part of each stage-1 tile
  int n1;           // stage-1 tiles of this CTA
  int rank;         // this CTA's rank (kModeDown: c; kModeBlock: light first)
  int64_t a0, a1;   // kModeBlock group-A range of this CTA
  int64_t u0, u1;   // down range (kModeDown: whole space; kModeBlock: group B)
  int64_t U2;       // total down units
};

// Group-B (or plain stream-K) range start of rank k.
__device__ __forceinline__ int64_t start_b(const StreamArgs& a, const Plan& p,
                                           int64_t k) {
  if (p.mode == kModeDown) return p.U2 * k / p.G;
  return k * a.bp_bl + (k < a.bp_rB ? k : a.bp_rB);
}

// Group-A range start of rank k (k in [0, G]).
__device__ __forceinline__ int64_t start_a(const StreamArgs& a, int64_t k) {
  const int64_t kl = k < a.bp_L ? k : a.bp_L;
  return kl * a.bp_al + (k - kl) * a.bp_ah + (k < a.bp_rA ? k : a.bp_rA);
}

__device__ __forceinline__ Plan make_plan(const StreamArgs& a, int mode) {
  Plan p;
  p.mode = mode;
  p.G = gridDim.x;
  p.c = blockIdx.x;
  p.U2 = static_cast<int64_t>(a.t2) * a.kb2;
  p.split = (mode != kModeDown && a.split_k > 1) ? a.split_k : 1;
  p.Q = p.G / p.split;
  p.q = p.c / p.split;
  p.krank = p.c % p.split;
  p.n1 = mode != kModeDown && p.q < a.t1 ? (a.t1 - 1 - p.q) / p.Q + 1 : 0;
  p.a0 = p.a1 = 0;
  p.u0 = p.u1 = 0;
  p.rank = p.c;
  if (mode == kModeStage1) return p;
  if (mode == kModeBlock) {
    p.rank = p.c >= a.bp_r ? p.c - a.bp_r : a.bp_L + p.c;
    p.a0 = start_a(a, p.rank);
    p.a1 = start_a(a, p.rank + 1);
  }
  p.u0 = start_b(a, p, p.rank);
  p.u1 = start_b(a, p, p.rank + 1);
  return p;
}

struct PieceIter {
  int i = 0;
  int grp = 0;        // 0 = stage 1, 1 = group A, 2 = group B / stream-K
  int64_t u = -1;
  __device__ __forceinline__ bool next(const StreamArgs& a, const Plan& p,
                                       Piece& out) {
    if (grp == 0) {
      if (i < p.n1) {
        out.down = 0;
        out.tile = p.q + i * p.Q;
        out.kb0 = p.krank * a.kb1 / p.split;
        out.kb1 = (p.krank + 1) * a.kb1 / p.split;
        ++i;
        return true;
      }
      if (p.mode == kModeStage1) return false;
      grp = p.mode == kModeBlock ? 1 : 2;
      u = -1;
    }
    if (grp == 1) {
      if (u < 0) u = p.a0;
      if (u < p.a1) {
        const int t = static_cast<int>(u / a.bp_nA);
        const int kb = static_cast<int>(u % a.bp_nA);
        const int64_t seg_end = static_cast<int64_t>(t + 1) * a.bp_nA;
        const int64_t end = seg_end < p.a1 ? seg_end : p.a1;
        out.down = 1;
        out.tile = t;
        out.kb0 = kb;
        out.kb1 = kb + static_cast<int>(end - u);
        u = end;
        ++i;
        return true;
      }
      grp = 2;
      u = -1;
    }
    if (u < 0) u = p.u0;
    if (u >= p.u1) return false;
    const int nseg = p.mode == kModeDown ? a.kb2 : a.bp_nB;
    const int kofs = p.mode == kModeDown ? 0 : a.bp_kB0;
    const int t = static_cast<int>(u / nseg);
    const int kb = kofs + static_cast<int>(u % nseg);
    const int64_t seg_end = static_cast<int64_t>(t + 1) * nseg;
    const int64_t end = seg_end < p.u1 ? seg_end : p.u1;
    out.down = 1;
    out.tile = t;
    out.kb0 = kb;
    out.kb1 = kb + static_cast<int>(end - u);
    u = end;
    ++i;
    return true;
  }
};

// ---------------------------------------------------------------------------
// Dynamic scheduling: piece index -> piece, and the smem piece queue that
// carries the producer's choices to the MMA / epilogue / math warps.
// ---------------------------------------------------------------------------
struct PieceQueue {
  int4 q[kPieceQueue];
  uint64_t full[kPieceQueue];
  uint64_t empty[kPieceQueue];
};

__device__ __forceinline__ int dyn_chunks(const StreamArgs& a) {
  return (a.kb2 + a.chunk_kb - 1) / a.chunk_kb;
}

// Stage-1 pieces per tile (stream-K over d_model when s1_chunk < kb1).
__device__ __forceinline__ int s1_pieces(const StreamArgs& a) {
  return a.s1_chunk > 0 && a.s1_chunk < a.kb1 ? (a.kb1 + a.s1_chunk - 1) / a.s1_chunk
                                               : 1;
}

// Piece index -> piece.  Stage-1 pieces first, tile-major (every K chunk of
// tile 0, then tile 1, ...), so tiles complete in order; then the down
// pieces, chunk-major (all t2 tiles of K chunk 0, then chunk 1, ...), so the
// earliest-published A2 is consumed first.
__device__ __forceinline__ bool decode_dyn(const StreamArgs& a, int mode,
                                           int64_t idx, Piece& out) {
  const int s1c = s1_pieces(a);
  const bool tail = a.s1_tail > 1;
  const int64_t n1 =
      mode == kModeDown ? 0
      : tail ? a.s1_whole + static_cast<int64_t>(a.t1 - a.s1_whole) * a.s1_tail
             : static_cast<int64_t>(a.t1) * s1c;
  const int64_t n2 =
      mode != kModeStage1 ? static_cast<int64_t>(a.t2) * dyn_chunks(a) : 0;
  if (idx < n1) {
    out.down = 0;
    if (tail) {
      if (idx < a.s1_whole) {
        out.tile = static_cast<int>(idx);
        out.kb0 = 0;
        out.kb1 = a.kb1;
      } else {
        const int j = static_cast<int>(idx - a.s1_whole);
        const int part = j % a.s1_tail;
        out.tile = a.s1_whole + j / a.s1_tail;
        out.kb0 = part * a.kb1 / a.s1_tail;
        out.kb1 = (part + 1) * a.kb1 / a.s1_tail;
      }
      return true;
    }
    out.tile = static_cast<int>(idx / s1c);
    const int kc = static_cast<int>(idx % s1c);
    out.kb0 = s1c > 1 ? kc * a.s1_chunk : 0;
    out.kb1 = s1c > 1 ? min(a.kb1, out.kb0 + a.s1_chunk) : a.kb1;
    return true;
  }
  idx -= n1;
  if (idx >= n2) return false;
  const int kc = static_cast<int>(idx / a.t2);
  out.down = 1;
  out.tile = static_cast<int>(idx % a.t2);
  out.kb0 = kc * a.chunk_kb;
  out.kb1 = min(a.kb2, out.kb0 + a.chunk_kb);
  return true;
}

// Balanced stream-K: the qi-th piece of CTA c of G (see StreamArgs::bal).
// Stage-1 pieces first, then down pieces, each range split at tile
// boundaries of its flattened (tile, K block) space.
__device__ __forceinline__ bool bal_range_piece(int64_t r0, int64_t r1, int kbt, int qi,
                                                int* tile, int* kb0, int* kb1, int* n) {
  if (r1 <= r0) {
    *n = 0;
    return false;
  }
  const int t0 = static_cast<int>(r0 / kbt);
  *n = static_cast<int>((r1 - 1) / kbt) - t0 + 1;
  if (qi >= *n) return false;
  const int t = t0 + qi;
  const int64_t lo = static_cast<int64_t>(t) * kbt;
  *tile = t;
  *kb0 = static_cast<int>((r0 > lo ? r0 : lo) - lo);
  *kb1 = static_cast<int>((r1 < lo + kbt ? r1 : lo + kbt) - lo);
  return true;
}

__device__ __forceinline__ bool bal_piece(const StreamArgs& a, int mode, int64_t c,
                                          int64_t G, int qi, Piece& out) {
  int n1 = 0;
  if (mode != kModeDown) {
    const int64_t U1 = static_cast<int64_t>(a.t1) * a.kb1;
    if (bal_range_piece(U1 * c / G, U1 * (c + 1) / G, a.kb1, qi, &out.tile, &out.kb0,
                        &out.kb1, &n1)) {
      out.down = 0;
      return true;
    }
  }
  if (mode == kModeStage1) return false;
  const int64_t U2 = static_cast<int64_t>(a.t2) * a.kb2;
  int n2 = 0;
  if (bal_range_piece(U2 * c / G, U2 * (c + 1) / G, a.kb2, qi - n1, &out.tile, &out.kb0,
                      &out.kb1, &n2)) {
    out.down = 1;
    return true;
  }
  return false;
}

// Down piece idx of the dynamic queue (chunk-major, see decode_dyn).
__device__ __forceinline__ bool decode_dyn_down(const StreamArgs& a, int64_t idx,
                                                Piece& out) {
  if (idx < 0 || idx >= static_cast<int64_t>(a.t2) * dyn_chunks(a)) return false;
  const int kc = static_cast<int>(idx / a.t2);
  out.down = 1;
  out.tile = static_cast<int>(idx % a.t2);
  out.kb0 = kc * a.chunk_kb;
  out.kb1 = min(a.kb2, out.kb0 + a.chunk_kb);
  return true;
}

// The consumers' view of the piece sequence (static plan or queue).
struct PieceReader {
  int i = 0;
  PieceIter it;
  // single: the calling thread alone consumes the slot; otherwise the whole
  // warp calls and lane 0 releases it.
  __device__ __forceinline__ bool next(const StreamArgs& a, const Plan& p,
                                       PieceQueue* pq, bool single,
                                       Piece& out) {
    if (!a.dynamic) {
      const bool ok = it.next(a, p, out);
      if (ok) ++i;
      return ok;
    }
    const int slot = i % kPieceQueue;
    mbar_wait(&pq->full[slot], static_cast<uint32_t>((i / kPieceQueue) & 1));
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(&pq->q[slot]))
                 : "memory");
    if (single) {
      mbar_arrive(&pq->empty[slot]);
    } else {
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&pq->empty[slot]);
    }
    ++i;
    if (v.w < 0) return false;
    out.tile = v.x;
    out.kb0 = v.y;
    out.kb1 = v.z;
    out.down = v.w;
    return true;
  }
};

// Number of non-empty ranges [start(k), start(k+1)), k in [0, n), that
// intersect [lo, hi); start is monotone.
template <typename StartFn>
__device__ __forceinline__ int pieces_in(StartFn start, int n, int64_t lo,
                                         int64_t hi) {
  if (hi <= lo || n <= 0) return 0;
  // k0 = largest k with start(k) <= lo, k1 = largest k with start(k) <= hi-1.
  auto rank_of = [&](int64_t u) {
    int l = 0, h = n - 1;
    while (l < h) {
      const int mid = (l + h + 1) >> 1;
      if (start(mid) <= u) l = mid; else h = mid - 1;
    }
    return l;
  };
  const int k0 = rank_of(lo), k1 = rank_of(hi - 1);
  int cnt = 0;
  for (int k = k0; k <= k1; ++k)
    if (start(k + 1) > start(k)) ++cnt;
  return cnt;
}

// How many pieces (flushes) down tile t receives in total.
__device__ __forceinline__ int down_tile_pieces(const StreamArgs& a,
                                                const Plan& p, int t) {
  if (a.dynamic) return dyn_chunks(a);
  auto sb = [&](int64_t k) { return start_b(a, p, k); };
  if (p.mode == kModeDown) {
    const int64_t lo = static_cast<int64_t>(t) * a.kb2;
    return pieces_in(sb, p.G, lo, lo + a.kb2);
  }
  int n = 0;
  if (a.bp_nA > 0) {
    auto sa = [&](int64_t k) { return start_a(a, k); };
    const int64_t lo = static_cast<int64_t>(t) * a.bp_nA;
    n += pieces_in(sa, p.G, lo, lo + a.bp_nA);
  }
  const int64_t lo = static_cast<int64_t>(t) * a.bp_nB;
  n += pieces_in(sb, p.G, lo, lo + a.bp_nB);
  return n;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void trace_stamp(const StreamArgs& a, int slot) {
  if (a.trace && slot < kTraceSlots)
    a.trace[static_cast<int64_t>(blockIdx.x) * kTraceSlots + slot] = gtimer();
}

__device__ __forceinline__ void trace_put(const StreamArgs& a, int slot,
                                          unsigned long long v) {
  if (a.trace && slot < kTraceSlots)
    a.trace[static_cast<int64_t>(blockIdx.x) * kTraceSlots + slot] = v;
}

// Release/acquire fence at gpu scope (MEMBAR.ALL.GPU; __threadfence() is
// fence.sc.gpu, MEMBAR.SC.GPU): every counter / flag protocol here is a
// release-acquire pattern, none needs sequential consistency.
// Finalize loops (last arriver of a tile) issue this many 16-byte L2 loads
// per thread before the first store.  8 measured -0.5 us at N = 64 on small
// TP shards but +0.6 us at N <= 16 (the larger unrolled body runs from a cold
// instruction cache), profiles/r1c_epilogue.md.
constexpr int kFinDepth = 4;

// Counter increment with release (this CTA's writes, gathered by the CTA
// barrier before it) and acquire (the other pieces' writes, for the last
// arriver) semantics in one instruction: replaces fence + atomicAdd + fence.
__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Cross-rank waits give up after 4 s: the error word (host-mapped, read by
// dfk_context_sync) is set and the wait returns false, so the launch ends
// -- with a wrong Y -- instead of hanging the GPU or trapping (a trap would
// leave the context unusable).  Any thread that sees the error set stops
// waiting at once.
__device__ __forceinline__ bool tp_wait_timed_out(const StreamArgs& a,
                                                  unsigned long long t0) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (t - t0 < 1000000ull) return false;  // fast path: no host-memory read
  if (a.tp_error && *reinterpret_cast<volatile int*>(a.tp_error)) return true;
  if (t - t0 > 4000000000ull) {
    if (a.tp_error) atomicExch_system(a.tp_error, 1);
    return true;
  }
  return false;
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Down epilogue tail: publish this CTA's piece of tile t; the CTA adding the
// last piece converts the tile to the output dtype and re-zeroes it.
// Fused-TP tail of a down piece of tile t (nk K blocks): see StreamArgs.
__device__ __forceinline__ void tp_finish_tile(const StreamArgs& a, int t, int nk,
                                               int tid, int nthr, int* smem_flag) {
  const int o = t % a.tp_size;
  named_bar(1, nthr);  // then one system-scope fence: see down_finish_tile
  if (tid == 0) {
    int old;  // release + acquire at system scope (peers' red.adds), one instruction
    asm volatile("atom.add.acq_rel.sys.s32 %0, [%1], %2;"
                 : "=r"(old) : "l"(a.tp_cnt[o] + t), "r"(nk) : "memory");
    *smem_flag = (old + nk == a.tp_total_kb) ? 1 : 0;  // acquire shared by the barrier
  }
  named_bar(1, nthr);
  if (*smem_flag) {
    // The full sums of tile t (owner o's workspace, possibly remote) go to
    // every rank's Y slot (the all-gather, by push), the workspace is
    // re-zeroed, and every rank's done word of tile t is raised; each rank
    // then copies the tile into its caller's Y (tp_collect_y).
    float* acc = a.tp_yacc[o];
    const int col0 = t * kDownCols;
    const int nvec = a.B * (kDownCols / 4);
    for (int base = tid; base < nvec; base += kFinDepth * nthr) {
      float4 v[kFinDepth];
      float4* q[kFinDepth];
#pragma unroll
      for (int u = 0; u < kFinDepth; ++u) {
        const int idx = base + u * nthr;
        q[u] = nullptr;
        if (idx < nvec) {
          const int n = idx / (kDownCols / 4), j = col0 + (idx % (kDownCols / 4)) * 4;
          q[u] = reinterpret_cast<float4*>(acc + static_cast<int64_t>(n) * a.yacc_ld + j);
          v[u] = __ldcg(q[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kFinDepth; ++u) {
        const int idx = base + u * nthr;
        if (idx < nvec) {
          const int n = idx / (kDownCols / 4), j = col0 + (idx % (kDownCols / 4)) * 4;
          if (j < a.out_cols) {  // out_cols is a multiple of 4 in TP mode
            for (int r = 0; r < a.tp_size; ++r)
              __stcg(reinterpret_cast<float4*>(a.tp_y[r] + n * a.y_ld + j), v[u]);
          }
          __stcg(q[u], make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
    }
    if (tid == 0) a.tp_cnt[o][t] = 0;
    named_bar(1, nthr);
    if (tid < a.tp_size) {  // release every rank's tile (cumulative through the barrier)
      __threadfence_system();
      atomicAdd_system(a.tp_done[tid] + t, 1);
    }
  }
  named_bar(1, nthr);
}

// End of a fused-TP block launch (every CTA, all threads): CTA c copies the
// tiles t = c, c + G, ... of this rank's full-sum Y slot into the caller's Y
// (fp32 or bf16) once the finalising CTA (on any rank) has raised the tile's
// done word, then re-arms it.  The kernel therefore ends with Y complete:
// one launch per tensor-parallel block, no copy or conversion after it.
__device__ __forceinline__ void tp_collect_y(const StreamArgs& a, int* smem_flag) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  int* done = a.tp_done[a.tp_rank];
  const float* ys = a.tp_y[a.tp_rank];
  for (int t = blockIdx.x; t < a.t2; t += gridDim.x) {
    if (tid == 0) {
      unsigned long long t0;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
      while (ld_acquire_sys(done + t) == 0)
        if (tp_wait_timed_out(a, t0)) break;
      done[t] = 0;  // consumed: the next finalisation is the next launch's
    }
    __syncthreads();  // the acquire is shared through the barrier
    const int col0 = t * kDownCols;
    const int nvec = a.B * (kDownCols / 4);
    for (int idx = tid; idx < nvec; idx += nthr) {
      const int n = idx / (kDownCols / 4), j = col0 + (idx % (kDownCols / 4)) * 4;
      if (j >= a.out_cols) continue;
      const float4 v = __ldcg(reinterpret_cast<const float4*>(ys + n * a.y_ld + j));
      if (a.y_bf16) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.y) + n * a.y_ld + j) = pk;
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.y) + n * a.y_ld + j) = v;
      }
    }
  }
  (void)smem_flag;
}

// 16 accumulator values of one lane (its output row `lane`, batch rows
// c0 .. c0+15) added into a [n][ld] fp32 workspace whose lane-consecutive
// addresses are consecutive floats: groups of 4 lanes transpose 4 x 4 blocks
// (two shuffle butterflies) so that each lane adds 4 consecutive floats of
// one batch row with a single red.global.add.v4.f32.  `col0` = the address of
// the group's first column for batch row 0 (16-byte aligned, ld % 4 == 0).
template <bool kSys = false>
__device__ __forceinline__ void red_rows_v4(float (&v)[16], float* col0, int64_t ld,
                                            int c0, int nvalid, int lane) {
  const int li = lane & 3;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float* x = v + 4 * b;
#pragma unroll
    for (int st = 1; st <= 2; st <<= 1) {
      const bool hi = (lane & st) != 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r & st) continue;
        const float send = hi ? x[r] : x[r | st];
        const float recv = __shfl_xor_sync(0xffffffffu, send, st);
        if (hi) x[r] = recv; else x[r | st] = recv;
      }
    }
    const int n = c0 + 4 * b + li;
    if (kSys)
      red_add_sys_v4_f32_if(col0 + static_cast<int64_t>(n) * ld, x[0], x[1], x[2], x[3],
                            n < nvalid);
    else
      red_add_v4_f32_if(col0 + static_cast<int64_t>(n) * ld, x[0], x[1], x[2], x[3], n < nvalid);
  }
}

// Direct Y (StreamArgs::y_direct), run by the nthr epilogue / math threads
// of every CTA once per launch: after griddepcontrol.wait (the previous
// launch may still read or write Y) zero this CTA's 1/G slice of Y and count
// it on sched[2].  Slices start on 128-byte lines (8 float4), so a warp's
// 512-byte store covers whole sectors (unaligned slices cost a partial sector
// per warp store: +30 KB of L2 writes at B = 64).
__device__ __forceinline__ void direct_y_zero(const StreamArgs& a, int tid, int nthr) {
  pdl_wait();
  const int64_t nv = static_cast<int64_t>(a.B) * (a.out_cols / 4);
  const int64_t v0 = (nv * blockIdx.x / gridDim.x) & ~int64_t{7};
  const int64_t v1 =
      blockIdx.x + 1 == gridDim.x ? nv : (nv * (blockIdx.x + 1) / gridDim.x) & ~int64_t{7};
  const int q4 = a.out_cols / 4;
  for (int64_t v = v0 + tid; v < v1; v += nthr) {
    const int64_t n = v / q4, j = (v % q4) * 4;
    __stcg(reinterpret_cast<float4*>(reinterpret_cast<float*>(a.y) + n * a.y_ld + j),
           make_float4(0.f, 0.f, 0.f, 0.f));
  }
  named_bar(1, nthr);  // then one cumulative release: see down_finish_tile
  if (tid == 0) {
    fence_acq_rel_gpu();
    atomicAdd(a.sched + 2, 1);
  }
}

// Before a CTA's first reduction into Y: every slice is zero (long true by
// then -- every CTA zeroes right after the PDL wait, the first down piece
// comes after stage-1 streaming).
__device__ __forceinline__ void direct_y_wait(const StreamArgs& a, int tid, int nthr) {
  if (tid == 0)
    while (static_cast<int>(ld_acquire(reinterpret_cast<const unsigned*>(a.sched + 2))) <
           static_cast<int>(gridDim.x)) {
    }
  named_bar(1, nthr);
}

__device__ __forceinline__ float* down_acc(const StreamArgs& a, int t) {
  return a.tp_size > 1 ? a.tp_yacc[t % a.tp_size] : a.yacc;
}

__device__ __forceinline__ void down_finish_tile(const StreamArgs& a,
                                                 const Plan& p, int t, int nk,
                                                 int tid, int nthr, int* smem_flag,
                                                 bool stamp = false) {
  if (a.tp_size > 1) {
    tp_finish_tile(a, t, nk, tid, nthr, smem_flag);
    return;
  }
  // Release pattern: every thread's red.adds are ordered before the CTA
  // barrier; ONE thread's gpu-scope fence (cumulative through the barrier)
  // then orders them all before its counter increment.
  named_bar(1, nthr);
  if (tid == 0) {
    if (stamp) trace_stamp(a, 41);
    if (stamp) trace_stamp(a, 42);
    // dynamic: count K blocks (pieces of a tile may differ in size)
    const int old = atom_add_acq_rel_gpu(&a.counters[t], a.dynamic ? nk : 1);
    const int last = a.dynamic ? (old + nk == a.kb2 ? 1 : 0)
                               : (old == down_tile_pieces(a, p, t) - 1 ? 1 : 0);
    if (stamp) trace_stamp(a, 43);
    *smem_flag = last;  // the acquire is shared through the barrier below
  }
  named_bar(1, nthr);
  if (stamp && tid == 0) trace_put(a, 45, *smem_flag);
  if (*smem_flag) {
    // 128 columns x B rows, 4 consecutive floats per thread and iteration;
    // loads are issued kFinDepth deep before any store (the reads are L2 round trips).
    const int col0 = t * kDownCols;
    const int nvec = a.B * (kDownCols / 4);
    for (int base = tid; base < nvec; base += kFinDepth * nthr) {
      float4 v[kFinDepth];
      float4* q[kFinDepth];
#pragma unroll
      for (int u = 0; u < kFinDepth; ++u) {
        const int idx = base + u * nthr;
        q[u] = nullptr;
        if (idx < nvec) {
          const int n = idx / (kDownCols / 4), j = col0 + (idx % (kDownCols / 4)) * 4;
          q[u] = reinterpret_cast<float4*>(a.yacc + static_cast<int64_t>(n) * a.yacc_ld + j);
          v[u] = __ldcg(q[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kFinDepth; ++u) {
        const int idx = base + u * nthr;
        if (idx < nvec) {
          const int n = idx / (kDownCols / 4), j = col0 + (idx % (kDownCols / 4)) * 4;
          const float vv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
          if (a.y_vec4 && j + 3 < a.out_cols) {
            // one 16-byte store (Y may live in mapped host memory: whole
            // PCIe write lines instead of 4-byte partial ones)
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.y) + n * a.y_ld + j) = v[u];
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (j + e < a.out_cols) {
                if (a.y_bf16) {
                  reinterpret_cast<__nv_bfloat16*>(a.y)[n * a.y_ld + j + e] =
                      __float2bfloat16_rn(vv[e]);
                } else {
                  reinterpret_cast<float*>(a.y)[n * a.y_ld + j + e] = vv[e];
                }
              }
            }
          }
          __stcg(q[u], make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
    }
    if (tid == 0) a.counters[t] = 0;
  }
  named_bar(1, nthr);
  if (stamp && tid == 0) trace_stamp(a, 44);
}

// Stage-1 epilogue tail in kModeBlock: make this tile's A2 stores visible to
// other SMs' TMA reads, then publish the tile's completion flag.
__device__ __forceinline__ void s1_publish(const StreamArgs& a, int tile,
                                           int tid, int nthr) {
  // Every writer orders its generic A2 stores before later async-proxy
  // reads; the barrier gathers them at CTA scope and one cumulative
  // release (tid 0) publishes them at gpu scope.
  fence_proxy_async_global();
  named_bar(1, nthr);
  if (tid == 0) st_release(a.flags + tile, a.epoch);
}

// Stage-1 stream-K: add this CTA's partial gate/up sums of tile t (one
// value per (row, n)) to the fp32 workspace.  mutant == 1 (the reference's
// SiluPerKChunk negative control, verification.cpp:84-124) instead adds
// SiLU(gate_part) * up_part into the gate slot: must fail parity.
__device__ __forceinline__ float* s1acc_at(const StreamArgs& a, int t, int n) {
  return a.s1acc + (static_cast<int64_t>(t) * a.n_pad + n) * kBlockRows;
}

// Tail of a partial stage-1 piece: the CTA adding the tile's last piece
// turns the full sums into A2, re-zeroes the workspace and publishes.
__device__ __forceinline__ void s1_finish_tile(const StreamArgs& a, int t, int nk,
                                               int tid, int nthr,
                                               int* smem_flag, bool stamp = false) {
  named_bar(1, nthr);  // then one fence: see down_finish_tile
  if (tid == 0) {
    if (stamp) trace_stamp(a, 46);
    if (stamp) trace_stamp(a, 47);
    // K blocks of the tile's pieces so far (pieces may differ in size)
    const int old = atom_add_acq_rel_gpu(&a.s1cnt[t], nk);
    const int last = (old + nk == a.kb1) ? 1 : 0;
    if (stamp) trace_stamp(a, 48);
    *smem_flag = last;  // the acquire is shared through the barrier below
  }
  named_bar(1, nthr);
  if (stamp && tid == 0) trace_put(a, 51, *smem_flag);
  if (*smem_flag) {
    // Work item (n, c4): A2 columns 4*c4 .. 4*c4+3 of batch row n; its gate
    // sums are 4 consecutive workspace rows, the up sums the 4 rows 16 below.
    // Loads are issued kFinDepth items deep before any store (L2 round trips).
    const int total = a.B * (kS1Cols / 4);
    for (int base = tid; base < total; base += kFinDepth * nthr) {
      float4 g[kFinDepth], u[kFinDepth];
      float* ptr[kFinDepth];
#pragma unroll
      for (int k = 0; k < kFinDepth; ++k) {
        const int idx = base + k * nthr;
        ptr[k] = nullptr;
        if (idx < total) {
          const int n = idx >> 4, c4 = idx & 15;
          ptr[k] = s1acc_at(a, t, n) + 32 * (c4 >> 2) + 4 * (c4 & 3);
          g[k] = __ldcg(reinterpret_cast<const float4*>(ptr[k]));
          u[k] = __ldcg(reinterpret_cast<const float4*>(ptr[k] + 16));
        }
      }
#pragma unroll
      for (int k = 0; k < kFinDepth; ++k) {
        const int idx = base + k * nthr;
        if (idx < total) {
          const int n = idx >> 4, c4 = idx & 15;
          const float gv[4] = {g[k].x, g[k].y, g[k].z, g[k].w};
          const float uv[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
          float h[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) h[e] = a.mutant == 1 ? gv[e] : silu_f(gv[e]) * uv[e];
          const int col = t * kS1Cols + 4 * c4;
          __nv_bfloat16* dst = a.a2 + static_cast<int64_t>(n) * a.a2_ld + col;
          if (col + 3 < a.cols_valid) {  // a2_ld % 8 == 0: 8-byte aligned
            __nv_bfloat162 lo = __floats2bfloat162_rn(h[0], h[1]);
            __nv_bfloat162 hi = __floats2bfloat162_rn(h[2], h[3]);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(dst) = pk;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (col + e < a.cols_valid) dst[e] = __float2bfloat16_rn(h[e]);
          }
          __stcg(reinterpret_cast<float4*>(ptr[k]), make_float4(0.f, 0.f, 0.f, 0.f));
          __stcg(reinterpret_cast<float4*>(ptr[k] + 16), make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
    }
    if (tid == 0) a.s1cnt[t] = 0;
    if (stamp && tid == 0) trace_stamp(a, 49);
    if (a.flags) s1_publish(a, t, tid, nthr);
    if (stamp && tid == 0) trace_stamp(a, 50);
  }
  named_bar(1, nthr);
}

// ---------------------------------------------------------------------------
// Producer (all of warp 0; lane 0 issues the copies).  In kModeBlock the
// warp checks the stage-1 completion flags a down piece depends on
// cooperatively (32 acquire loads in flight), once per piece.
// ---------------------------------------------------------------------------
struct ReadyCache {
  int lo = 0, hi = 0;  // flags of stage-1 tiles [lo, hi) known published
};

__device__ __forceinline__ void ensure_ready(const StreamArgs& a,
                                            ReadyCache& rc, int lo, int hi) {
  if (!a.flags || (lo >= rc.lo && hi <= rc.hi)) return;
  const int lane = static_cast<int>(lane_id());
  for (int j = lo + lane; j < hi; j += 32) {
    while (ld_acquire(a.flags + j) != a.epoch) {
    }
  }
  __syncwarp();
  fence_proxy_async_global();
  rc.lo = lo;
  rc.hi = hi;
}

// Non-blocking form of ensure_ready (whole warp): true, and the range
// cached, when every flag in [lo, hi) is published.
__device__ __forceinline__ bool check_ready(const StreamArgs& a, ReadyCache& rc,
                                            int lo, int hi) {
  if (!a.flags || (lo >= rc.lo && hi <= rc.hi)) return true;
  bool ok = true;
  for (int j = lo + static_cast<int>(lane_id()); j < hi; j += 32)
    ok = ok && ld_acquire(a.flags + j) == a.epoch;
  ok = __all_sync(0xffffffffu, ok);
  if (ok) {
    fence_proxy_async_global();
    rc.lo = lo;
    rc.hi = hi;
  }
  return ok;
}

__device__ __forceinline__ void produce(const StreamArgs& a, const Plan& p,
                                        const CUtensorMap* xmap,
                                        const CUtensorMap* amap, const CUtensorMap* a3map,
                                        uint8_t* smem,
                                        int stage_bytes, uint64_t* full,
                                        uint64_t* empty, PieceQueue* pq, int4* pend) {
  const bool leader = lane_id() == 0;
  const uint64_t policy = policy_evict_first();
  const uint32_t xblk = static_cast<uint32_t>(a.n_pad) * 128u;
  const uint32_t wbytes_all = static_cast<uint32_t>(a.kbs) * kBlockBytes;
  // Stages whose weight copies are issued but whose activation loads wait:
  // before griddepcontrol.wait (PDL), or -- down pieces -- until the stage-1
  // tiles they read have published.  Weight streaming never waits for
  // either: it runs ahead until the ring wraps onto a deferred stage.
  // pend[] lives in shared memory (one entry per ring slot, written by the
  // leader lane): a per-thread array indexed at run time would be a local
  // memory stack frame whose write-backs add ~0.6 MB of L2 stores per launch.
  // Entry: x = slot | nb << 8 | down << 12 | qi << 16, y = kb,
  // z = pk0 | pk1 << 16 (the down piece's A2 K-block range).
  int npend = 0;
  int64_t pend0_it = 0;  // ring stage of pend[0]
  ReadyCache rc;
  int64_t it = 0;
  bool waited = false;
  PieceIter pi;
  bool x_ok = a.x_ready == nullptr;
  auto act_loads = [&](uint8_t* xs, int kb, int nb, int down, uint64_t* bar) {
    if (!down && !x_ok) {  // (whole warp) the side stream's X copy landed?
      unsigned long long t0;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
      // gpu scope: the flag and the X bytes are written by this GPU's copy
      // engine / stream front end, visible in its L2
      while (static_cast<int>(ld_acquire(a.x_ready) - a.x_seq) < 0)
        if (tp_wait_timed_out(a, t0)) break;
      fence_proxy_async_global();
      x_ok = true;
    }
    if (!leader) return;
    if (down ? a.a3d : a.x3d) {
      tma_load_3d(xs, down ? a3map : xmap, 0, 0, kb, bar);
      return;
    }
    for (int b = 0; b < nb; ++b) {
      tma_load_2d(xs + b * xblk, down ? amap : xmap, (kb + b) * kBlockK, 0, bar);
    }
  };
  Piece first{};
  int first_issued = 0;  // K blocks of the first piece already in the ring
  // Issue every deferred activation load: griddepcontrol.wait first (before
  // it, the next pf_kb K blocks of the first piece go to L2), then block on
  // the readiness of each deferred down stage.
  auto flush = [&]() {
    if (!waited) {
      if (leader && a.pf_kb > 0 && first.kb1 > first.kb0) {
        const uint8_t* wb = first.down ? a.w2 : a.w1;
        const int kbt = first.down ? a.kb2 : a.kb1;
        const int k0 = first.kb0 + first_issued;
        const int k1 = min(first.kb1, k0 + a.pf_kb);
        for (int kb = k0; kb < k1; kb += 4) {
          const int nb = min(4, k1 - kb);
          bulk_prefetch_l2(wb + (static_cast<int64_t>(first.tile) * kbt + kb) *
                                    static_cast<int64_t>(kBlockBytes),
                           static_cast<uint32_t>(nb) * kBlockBytes);
        }
      }
      pdl_wait();
      waited = true;
    }
    __syncwarp();  // the leader's pend[] writes
    for (int j = 0; j < npend; ++j) {
      const int4 e = pend[j];
      const int slot = e.x & 0xff, nb = (e.x >> 8) & 0xf, down = (e.x >> 12) & 1,
                qi = e.x >> 16, kb = e.y, pk0 = e.z & 0xffff, pk1 = (e.z >> 16) & 0xffff;
      if (down) ensure_ready(a, rc, pk0, pk1);
      if (leader && kb == pk0 && qi < 8) trace_stamp(a, 32 + qi);
      act_loads(smem + static_cast<int64_t>(slot) * stage_bytes + wbytes_all, kb, nb, down,
                &full[slot]);
    }
    __syncwarp();  // every lane has read pend[] before it is rewritten
    npend = 0;
  };
  for (int qi = 0;; ++qi) {
    Piece pc;
    bool valid;
    if (!a.dynamic) {
      valid = pi.next(a, p, pc);
    } else {
      if (a.bal) {
        valid = bal_piece(a, p.mode, blockIdx.x, gridDim.x, qi, pc);
      } else if (p.split > 1) {
        // Dynamic + cluster split-K (small shards): CTA c < t1 x split
        // starts with K part c % split of stage-1 tile c / split (its
        // cluster reduces the parts through DSMEM); every other piece is a
        // down piece -- the first static for the remaining CTAs, then the
        // queue.
        const int n1s = a.t1 * p.split;
        if (qi == 0 && static_cast<int>(blockIdx.x) < n1s) {
          pc.down = 0;
          pc.tile = p.q;
          pc.kb0 = p.krank * a.kb1 / p.split;
          pc.kb1 = (p.krank + 1) * a.kb1 / p.split;
          valid = true;
        } else {
          int64_t didx = static_cast<int64_t>(blockIdx.x) - n1s;
          if (qi > 0) {
            if (!waited) flush();  // no global atomics before the previous grid ends
            int got = 0;
            if (leader) got = atomicAdd(a.sched, 1);
            didx = static_cast<int64_t>(gridDim.x) - n1s + __shfl_sync(0xffffffffu, got, 0);
          }
          valid = decode_dyn_down(a, didx, pc);
        }
      } else {
        int64_t idx = blockIdx.x;
        if (qi > 0) {
          if (!waited) flush();  // no global atomics before the previous grid ends
          int got = 0;
          if (leader) got = atomicAdd(a.sched, 1);
          idx = static_cast<int64_t>(gridDim.x) + __shfl_sync(0xffffffffu, got, 0);
        }
        valid = decode_dyn(a, p.mode, idx, pc);
      }
      const int slot = qi % kPieceQueue;
      if (qi >= kPieceQueue) {
        if (leader)
          mbar_wait(&pq->empty[slot],
                    static_cast<uint32_t>(((qi / kPieceQueue) & 1) ^ 1));
        __syncwarp();
      }
      if (leader) {
        pq->q[slot] = make_int4(pc.tile, pc.kb0, pc.kb1, valid ? pc.down : -1);
        mbar_arrive(&pq->full[slot]);
      }
    }
    if (!valid) break;
    if (qi == 0) first = pc;
    if (leader) trace_stamp(a, 3 + 2 * qi);
    if (leader && qi < 8)
      trace_put(a, 24 + qi,
                (static_cast<unsigned long long>(pc.down) << 48) |
                    (static_cast<unsigned long long>(pc.kb1 - pc.kb0) << 32) |
                    static_cast<unsigned long long>(pc.tile));    const uint8_t* wbase = pc.down ? a.w2 : a.w1;
    const int kbt = pc.down ? a.kb2 : a.kb1;
    for (int kb = pc.kb0; kb < pc.kb1; kb += a.kbs, ++it) {
      const int nb = min(a.kbs, pc.kb1 - kb);
      const int slot = static_cast<int>(it % a.stages);
      const uint32_t phase = static_cast<uint32_t>((it / a.stages) & 1);
      if (it >= a.stages) {
        // The slot about to be reused holds a deferred stage: its consumer
        // cannot finish before we issue its activations.
        if (npend > 0 && pend0_it <= it - a.stages) flush();
        if (leader) mbar_wait(&empty[slot], phase ^ 1u);
        __syncwarp();
        // trace_rel: when the producer saw stage (it - stages) released
        if (leader && a.trace && a.trace_rel && it - a.stages >= a.trace_s0 &&
            it - a.stages < a.trace_s0 + 12)
          trace_stamp(a, 40 + static_cast<int>(it - a.stages - a.trace_s0));
      }
      uint8_t* st = smem + static_cast<int64_t>(slot) * stage_bytes;
      if (leader) {
        // (a 3-D X box always brings kbs K blocks' rows, OOB included)
        mbar_arrive_expect_tx(&full[slot],
                              static_cast<uint32_t>(nb) * kBlockBytes +
                                  static_cast<uint32_t>((pc.down ? a.a3d : a.x3d) ? a.kbs : nb) *
                                      static_cast<uint32_t>(a.xrows) * 128u);
        // nb consecutive K blocks of one tile are contiguous in the pack.
        bulk_g2s(st,
                 wbase + (static_cast<int64_t>(pc.tile) * kbt + kb) *
                             static_cast<int64_t>(kBlockBytes),
                 static_cast<uint32_t>(nb) * kBlockBytes, &full[slot], policy);
        if (a.trace && !a.trace_rel && a.trace_s0 >= 0 && it >= a.trace_s0 &&
            it < a.trace_s0 + 12)
          trace_stamp(a, 40 + static_cast<int>(it - a.trace_s0));
      }
      // Activation loads stay in stage order: defer while anything is
      // deferred, before the PDL wait, or while this down piece's A2 is not
      // yet published (non-blocking check).
      if (!waited || npend > 0 || (pc.down && !check_ready(a, rc, pc.kb0, pc.kb1))) {
        if (qi == 0 && !waited) first_issued += nb;
        if (npend == 0) pend0_it = it;
        if (leader)
          pend[npend] = make_int4(slot | (nb << 8) | (pc.down << 12) | (qi << 16), kb,
                                  pc.kb0 | (pc.kb1 << 16), 0);
        ++npend;
        continue;
      }
      if (leader && kb == pc.kb0 && qi < 8) trace_stamp(a, 32 + qi);
      act_loads(st + wbytes_all, kb, nb, pc.down, &full[slot]);
    }
  }
  if (leader) trace_stamp(a, 1);
  flush();  // fewer stages of work than ring slots / deferred tail
}

// ---------------------------------------------------------------------------
// GEMV math warps (batch <= NB).  Lane = (q, c): c = 16-byte chunk of the
// 64-wide K block, q = one of the 4 rows this warp handles per pass; pass p
// covers the 32-row group p of the 128-row block.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int gemv_row(int p, int mw, int q) {
  // q 0,1 -> gate rows 2mw+q; q 2,3 -> the matching up rows (16 apart), so
  // the gate/up pair of one A2 column is lane ^ 16.
  return p * 32 + (q < 2 ? 2 * mw + q : 16 + 2 * mw + (q - 2));
}

template <int NB>
__device__ __forceinline__ void gemv_consume(const StreamArgs& a, const Plan& p,
                                             uint8_t* smem, int stage_bytes,
                                             uint64_t* full, uint64_t* empty,
                                             int* smem_flag, PieceQueue* pq) {
  const int mw = static_cast<int>(warp_id()) - 1;
  const int lane = static_cast<int>(lane_id());
  const int q = lane >> 3, c = lane & 7;
  const int tid = mw * 32 + lane;
  const int nthr = kGemvWarps * 32;
  const int wbytes_all = a.kbs * kBlockBytes;
  const int xblk = a.n_pad * 128;
  int64_t it = 0;
  bool y_zeroed = false;
  if (a.y_direct) direct_y_zero(a, tid, nthr);
  PieceReader pi;
  Piece pc;
  while (pi.next(a, p, pq, false, pc)) {
    float acc[4][NB];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int n = 0; n < NB; ++n) acc[r][n] = 0.f;

    for (int kb = pc.kb0; kb < pc.kb1; kb += a.kbs, ++it) {
      const int nb = min(a.kbs, pc.kb1 - kb);
      const int slot = static_cast<int>(it % a.stages);
      const uint32_t phase = static_cast<uint32_t>((it / a.stages) & 1);
      mbar_wait(&full[slot], phase);
      const uint8_t* st = smem + static_cast<int64_t>(slot) * stage_bytes;
      for (int b = 0; b < nb; ++b) {
        const uint8_t* ws = st + b * kBlockBytes;
        const uint8_t* xs = st + wbytes_all + b * xblk;
        float xf[NB][8];
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const uint4 xv = *reinterpret_cast<const uint4*>(
              xs + n * 128 + ((c ^ (n & 7)) << 4));
          xf[n][0] = bf16lo(xv.x); xf[n][1] = bf16hi(xv.x);
          xf[n][2] = bf16lo(xv.y); xf[n][3] = bf16hi(xv.y);
          xf[n][4] = bf16lo(xv.z); xf[n][5] = bf16hi(xv.z);
          xf[n][6] = bf16lo(xv.w); xf[n][7] = bf16hi(xv.w);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int row = gemv_row(r, mw, q);
          const uint4 wv = *reinterpret_cast<const uint4*>(
              ws + row * 128 + ((c ^ (row & 7)) << 4));
          float wf[8];
          wf[0] = bf16lo(wv.x); wf[1] = bf16hi(wv.x);
          wf[2] = bf16lo(wv.y); wf[3] = bf16hi(wv.y);
          wf[4] = bf16lo(wv.z); wf[5] = bf16hi(wv.z);
          wf[6] = bf16lo(wv.w); wf[7] = bf16hi(wv.w);
#pragma unroll
          for (int n = 0; n < NB; ++n)
#pragma unroll
            for (int e = 0; e < 8; ++e)
              acc[r][n] = fmaf(wf[e], xf[n][e], acc[r][n]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        float v = acc[r][n];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        acc[r][n] = v;
      }

    if (!pc.down && (pc.kb0 > 0 || pc.kb1 < a.kb1)) {
      // stream-K piece: partial sums to the workspace
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = gemv_row(r, mw, q);
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          float v = acc[r][n];
          if (a.mutant == 1) {
            const float up = __shfl_xor_sync(0xffffffffu, v, 16);
            v = q < 2 ? silu_f(v) * up : 0.f;
          }
          if (c == 0 && n < a.B) atomicAdd(s1acc_at(a, pc.tile, n) + row, v);
        }
      }
      s1_finish_tile(a, pc.tile, pc.kb1 - pc.kb0, tid, nthr, smem_flag);
    } else if (!pc.down) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int col = pc.tile * kS1Cols + r * 16 + 2 * mw + q;
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const float up = __shfl_xor_sync(0xffffffffu, acc[r][n], 16);
          if (c == 0 && q < 2 && n < a.B && col < a.cols_valid) {
            a.a2[n * a.a2_ld + col] =
                __float2bfloat16_rn(silu_f(acc[r][n]) * up);
          }
        }
      }
      if (a.flags) s1_publish(a, pc.tile, tid, nthr);
    } else {
      if (a.y_direct && !y_zeroed) {
        direct_y_wait(a, tid, nthr);
        y_zeroed = true;
      }
      float* ybase = a.y_direct ? reinterpret_cast<float*>(a.y) : down_acc(a, pc.tile);
      const int64_t ld = a.y_direct ? a.y_ld : a.yacc_ld;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int j = pc.tile * kDownCols + gemv_row(r, mw, q);
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          if (c == 0 && n < a.B && j < a.out_cols) {
            float* dst = ybase + static_cast<int64_t>(n) * ld + j;
            if (a.tp_size > 1)
              atomicAdd_system(dst, acc[r][n]);
            else
              atomicAdd(dst, acc[r][n]);
          }
        }
      }
      if (!a.y_direct) down_finish_tile(a, p, pc.tile, pc.kb1 - pc.kb0, tid, nthr, smem_flag);
    }
    if (tid == 0) trace_stamp(a, 2 + 2 * pi.i);
  }
  if (tid == 0) trace_stamp(a, 2);
}

// ---------------------------------------------------------------------------
// tcgen05 MMA issuer (one lane of warp 1).
// ---------------------------------------------------------------------------
// One ring stage of MMAs: NB K blocks x 4 K16 steps, fully unrolled, the
// smem descriptors advanced by constant adds (the start-address field is
// addr >> 4 in the low bits), MMA i into accumulator chain i % NACC.  The
// single issuing thread is on the streaming critical path (a slot is freed
// only when its MMAs retire), so this loop is kept branch- and divide-free.
template <int NB, int NACC>
__device__ __forceinline__ void mma_stage(uint32_t d, uint64_t dw, uint64_t dx,
                                          uint32_t idesc, uint32_t xblk16,
                                          uint32_t chain_cols, bool zero) {
#pragma unroll
  for (int b = 0; b < NB; ++b) {
#pragma unroll
    for (int k = 0; k < kBlockK / 16; ++k) {
      constexpr int kSteps = kBlockK / 16;
      const int i = b * kSteps + k;
      const uint64_t ad = dw + static_cast<uint64_t>((b * kBlockBytes + k * 32) >> 4);
      const uint64_t bd = dx + static_cast<uint64_t>(b * xblk16 + ((k * 32) >> 4));
      tc_mma_bf16(d + static_cast<uint32_t>(i % NACC) * chain_cols, ad, bd, idesc,
                  (zero && i < NACC) ? 0u : 1u);
    }
  }
}

template <int NACC>
__device__ __forceinline__ void mma_stage_nb(int nb, uint32_t d, uint64_t dw, uint64_t dx,
                                             uint32_t idesc, uint32_t xblk16,
                                             uint32_t chain_cols, bool zero) {
  switch (nb) {
    case 1: mma_stage<1, NACC>(d, dw, dx, idesc, xblk16, chain_cols, zero); break;
    case 2: mma_stage<2, NACC>(d, dw, dx, idesc, xblk16, chain_cols, zero); break;
    case 3: mma_stage<3, NACC>(d, dw, dx, idesc, xblk16, chain_cols, zero); break;
    default: mma_stage<4, NACC>(d, dw, dx, idesc, xblk16, chain_cols, zero); break;
  }
}

template <int NACC>
__device__ __forceinline__ void mma_loop(const StreamArgs& a, const Plan& p,
                                         uint8_t* smem, int stage_bytes,
                                         uint64_t* full, uint64_t* empty,
                                         uint64_t* tfull, uint64_t* tempty,
                                         uint32_t tmem_base, PieceQueue* pq) {
  const uint32_t idesc = umma_idesc_bf16(128, static_cast<uint32_t>(a.n_pad));
  const uint32_t xblk16 = static_cast<uint32_t>(a.n_pad) * 128u / 16u;
  const uint32_t xblk16_3d = static_cast<uint32_t>(a.xrows) * 128u / 16u;  // packed X (x3d)
  const uint32_t wbytes_all = static_cast<uint32_t>(a.kbs) * kBlockBytes;
  const uint32_t chain_cols = static_cast<uint32_t>(a.n_pad);
  const uint64_t desc0 = umma_desc_sw128(0);
  const uint32_t smem0 = smem_u32(smem);
  int64_t it = 0;
  int acc_it = 0;
  PieceReader pi;
  Piece pc;
  while (pi.next(a, p, pq, true, pc)) {
    const int ab = acc_it & 1;
    const uint32_t aph = static_cast<uint32_t>((acc_it >> 1) & 1);
    mbar_wait(&tempty[ab], aph ^ 1u);
    tc_fence_after();
    const uint32_t d = tmem_base + static_cast<uint32_t>(ab * NACC * a.n_pad);
    int slot = static_cast<int>(it % a.stages);
    uint32_t phase = static_cast<uint32_t>((it / a.stages) & 1);
    for (int kb = pc.kb0; kb < pc.kb1; kb += a.kbs, ++it) {
      const int nb = min(a.kbs, pc.kb1 - kb);
      mbar_wait(&full[slot], phase);
      if (a.trace && !a.trace_rel && a.trace_s0 >= 0 && it >= a.trace_s0 &&
          it < a.trace_s0 + 12)
        trace_stamp(a, 52 + static_cast<int>(it - a.trace_s0));
      tc_fence_after();
      const uint32_t sbase = smem0 + static_cast<uint32_t>(slot * stage_bytes);
      const uint64_t dw = desc0 + (sbase >> 4);
      const uint64_t dx = desc0 + ((sbase + wbytes_all) >> 4);
      mma_stage_nb<NACC>(nb, d, dw, dx, idesc,
                         (pc.down ? a.a3d : a.x3d) ? xblk16_3d : xblk16, chain_cols,
                         kb == pc.kb0);
      tc_commit(&empty[slot]);
      // trace_rel: the stage's MMAs and commit are issued
      if (a.trace && a.trace_rel && it >= a.trace_s0 && it < a.trace_s0 + 12)
        trace_stamp(a, 52 + static_cast<int>(it - a.trace_s0));
      if (++slot == a.stages) {
        slot = 0;
        phase ^= 1u;
      }
    }
    tc_commit(&tfull[ab]);
    ++acc_it;
  }
}

__device__ __forceinline__ void mma_issue(const StreamArgs& a, const Plan& p,
                                          uint8_t* smem, int stage_bytes,
                                          uint64_t* full, uint64_t* empty,
                                          uint64_t* tfull, uint64_t* tempty,
                                          uint32_t tmem_base, PieceQueue* pq) {
  switch (a.nacc) {
    case 4: mma_loop<4>(a, p, smem, stage_bytes, full, empty, tfull, tempty, tmem_base, pq); break;
    case 2: mma_loop<2>(a, p, smem, stage_bytes, full, empty, tfull, tempty, tmem_base, pq); break;
    default: mma_loop<1>(a, p, smem, stage_bytes, full, empty, tfull, tempty, tmem_base, pq);
  }
}

// ---------------------------------------------------------------------------
// tcgen05 epilogue (warps 2-5; TMEM lanes 32*(warp%4) .. +31).
// ---------------------------------------------------------------------------
// Stage-1 epilogue of a K-split tile (cluster of p.split CTAs).  Each
// non-leader writes its partial gate/up accumulators into ITS OWN slot
// red[rank-1][row][n] of the leader's shared memory with st.async (16-byte
// DSMEM stores whose completion is counted in bytes on the leader's
// red_full mbarrier: no fences, no per-thread arrivals); the leader adds the
// slots to its own partial, runs SiLU*up, writes A2 and releases every
// non-leader's red_free barrier.  Partial sums never leave the SMs.
// mutant == 1 applies SiLU*up per K part instead (the reference's
// SiluPerKChunk negative control, verification.cpp:84-124): must fail parity.
__device__ __forceinline__ void s1_split_epilogue(const StreamArgs& a,
                                                  const Plan& p, int tile,
                                                  uint32_t taddr, int row,
                                                  int lane, int tid, float* red,
                                                  uint64_t* red_full,
                                                  uint64_t* red_free,
                                                  int split_iter) {
  int is_up, cofs;
  s1_row_map(row, &is_up, &cofs);
  const int col = tile * kS1Cols + cofs;
  const uint32_t par = static_cast<uint32_t>(split_iter & 1);
  const bool mutant = a.mutant == 1;
  const int rs = split_row_floats(a.n_pad);
  const int slot_floats = 128 * rs;
  if (p.krank != 0) {
    float* mine = red + (p.krank - 1) * slot_floats + row * rs;
    if (row == 0 && split_iter == 0) trace_stamp(a, 61);
    mbar_wait_cluster(red_free, par ^ 1u);
    if (row == 0 && split_iter == 0) trace_stamp(a, 62);
    for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
      float v[16];
      tmem_ld16(taddr + c0, v);
      if (mutant) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float up = __shfl_xor_sync(0xffffffffu, v[e], 16);
          v[e] = is_up ? 0.f : silu_f(v[e]) * up;
        }
      }
#pragma unroll
      for (int e = 0; e < 16; e += 4)
        st_async_f4(mine + c0 + e, red_full, 0, v[e], v[e + 1], v[e + 2], v[e + 3]);
    }
    if (row == 0 && split_iter == 0) trace_stamp(a, 63);
    return;
  }
  // Leader: arm the byte count of this phase, wait for every partner slot.
  if (tid == 0)
    mbar_arrive_expect_tx(red_full, static_cast<uint32_t>((p.split - 1) * 128 * a.n_pad * 4));
  if (row == 0 && split_iter == 0) trace_stamp(a, 61);
  mbar_wait_cluster(red_full, par);
  if (row == 0 && split_iter == 0) trace_stamp(a, 62);
  if ((row & 31) == 0 && split_iter == 0) trace_stamp(a, 44 + (row >> 5));
  for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
    float other[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) other[e] = 0.f;
    for (int r = 1; r < p.split; ++r) {
      const float* src = red + (r - 1) * slot_floats + row * rs + c0;
#pragma unroll
      for (int e = 0; e < 16; e += 4) {
        const float4 t = ld_shared_f4(src + e);
        other[e] += t.x;
        other[e + 1] += t.y;
        other[e + 2] += t.z;
        other[e + 3] += t.w;
      }
    }
    float v[16];
    tmem_ld16(taddr + c0, v);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      float out;
      if (!mutant) {
        const float g_or_u = v[e] + other[e];
        const float up = __shfl_xor_sync(0xffffffffu, g_or_u, 16);
        out = silu_f(g_or_u) * up;
      } else {
        const float up = __shfl_xor_sync(0xffffffffu, v[e], 16);
        out = silu_f(v[e]) * up + other[e];
      }
      const int n = c0 + e;
      if (!is_up && n < a.B && col < a.cols_valid) {
        a.a2[n * a.a2_ld + col] = __float2bfloat16_rn(out);
      }
    }
  }
  // Release the slots: one arrival per leader epilogue warp on every
  // partner's red_free (the release orders this warp's slot reads).
  if ((row & 31) == 0 && split_iter == 0) trace_stamp(a, 48 + (row >> 5));
  __syncwarp();
  if (lane == 0)
    for (int r = 1; r < p.split; ++r) mbar_arrive_cluster(red_free, r);
  if ((row & 31) == 0 && split_iter == 0) trace_stamp(a, 52 + (row >> 5));
}

__device__ __forceinline__ void tc_epilogue(const StreamArgs& a, const Plan& p,
                                            uint64_t* tfull, uint64_t* tempty,
                                            uint32_t tmem_base,
                                            int* smem_flag, PieceQueue* pq,
                                            float* red, uint64_t* red_full,
                                            uint64_t* red_free, const CUtensorMap* amap,
                                            uint8_t* a2st) {
  const int w = static_cast<int>(warp_id());
  const int quarter = w & 3;
  const int lane = static_cast<int>(lane_id());
  const int row = quarter * 32 + lane;
  const int tid = (w - 2) * 32 + lane;
  int acc_it = 0;
  int split_iter = 0;
  bool dn_stamped = false;
  bool y_zeroed = false;  // direct Y: every CTA's slice is zero (seen once)
  if (a.y_direct) direct_y_zero(a, tid, 128);
  PieceReader pi;
  Piece pc;
  while (pi.next(a, p, pq, false, pc)) {
    const int ab = acc_it & 1;
    const uint32_t aph = static_cast<uint32_t>((acc_it >> 1) & 1);
    mbar_wait(&tfull[ab], aph);
    if (tid == 0 && acc_it == 0) trace_stamp(a, 19);
    tc_fence_after();
    const int nacc = a.nacc > 0 ? a.nacc : 1;
    const uint32_t astr = static_cast<uint32_t>(a.n_pad);
    const uint32_t taddr = tmem_base +
                           (static_cast<uint32_t>(quarter * 32) << 16) +
                           static_cast<uint32_t>(ab * nacc * a.n_pad);
    if (!pc.down && p.split > 1) {
      s1_split_epilogue(a, p, pc.tile, taddr, row, lane, tid, red, red_full, red_free,
                        split_iter++);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      if (a.flags && p.krank == 0) s1_publish(a, pc.tile, tid, 128);
      if (tid == 0) trace_stamp(a, 2 + 2 * pi.i);
      ++acc_it;
      continue;
    }
    if (!pc.down && (pc.kb0 > 0 || pc.kb1 < a.kb1)) {
      const bool s1_stamp = a.trace && a.trace_s0 < 0 && acc_it == 0;
      if (s1_stamp && tid == 0) trace_stamp(a, 52);
      // stream-K piece: partial gate/up sums to the workspace (one
      // predicated red.add per element, straight-line)
      float* base = s1acc_at(a, pc.tile, 0) + row;
      for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
        float v[16];
        tmem_ld16_sum(taddr + c0, nacc, astr, v);
        if (a.mutant == 1) {  // negative control: SiLU per K part
          int is_up, cofs;
          s1_row_map(row, &is_up, &cofs);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float up = __shfl_xor_sync(0xffffffffu, v[e], 16);
            v[e] = is_up ? 0.f : silu_f(v[e]) * up;
          }
        }
        if (a.red_v4) {
          red_rows_v4(v, base - (lane & 3), kBlockRows, c0, a.B, lane);
        } else {
          float* bc = base + static_cast<int64_t>(c0) * kBlockRows;
#pragma unroll
          for (int e = 0; e < 16; ++e)
            red_add_f32_if(bc + e * kBlockRows, v[e], c0 + e < a.B);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      s1_finish_tile(a, pc.tile, pc.kb1 - pc.kb0, tid, 128, smem_flag, s1_stamp);
    } else if (!pc.down && a.a2_tma) {
      // A2 tile -> swizzled smem [n][64 cols] bf16 -> one TMA store.  The
      // barrier first: the previous tile's store has been waited for by tid 0.
      int is_up, cofs;
      s1_row_map(row, &is_up, &cofs);
      // Lane pairs (l, l ^ 16) hold gate / up of the same column for 16
      // batch rows; one exchange of 8 values gives each lane 8 (gate, up)
      // pairs: the gate lane finishes rows n = 4j + {0, 1}, the up lane
      // n = 4j + {2, 3} (rows 2 apart: the two lanes' 32-byte row segments
      // fall in different banks of the swizzled tile).  Branch-free, eight
      // independent SiLU chains, eight shared stores per 16 rows.
      const uint32_t st_base = smem_u32(a2st) + static_cast<uint32_t>((cofs & 7) << 1);
      const int chunk = cofs >> 3;
      named_bar(1, 128);
      for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
        float v[16];
        tmem_ld16_sum(taddr + c0, nacc, astr, v);
        if (tid == 0 && acc_it == 0 && c0 == 0) trace_stamp(a, 23);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int ng = (i & 1) + ((i >> 1) << 2);  // gate lane's row
          const float send = is_up ? v[ng] : v[ng + 2];
          const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
          const float g = is_up ? recv : v[ng];
          const float u = is_up ? v[ng + 2] : recv;
          const int n = c0 + ng + (is_up ? 2 : 0);
          // row n, column cofs: 16-byte chunk (cofs / 8) XOR (n & 7)
          st_shared_u16(st_base + static_cast<uint32_t>(n * 128 + ((chunk ^ (n & 7)) << 4)),
                        __bfloat16_as_ushort(__float2bfloat16_rn(silu_f(g) * u)));
        }
      }
      if (tid == 0 && acc_it == 0) trace_stamp(a, 31);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      fence_proxy_async_shared();
      named_bar(1, 128);
      if (tid == 0) {
        if (acc_it == 0) trace_stamp(a, 20);
        tma_store_2d(amap, a2st, pc.tile * kS1Cols, 0);
        bulk_commit();
        bulk_wait_all();
        if (acc_it == 0) trace_stamp(a, 21);
        if (a.flags) {
          // The bulk group's completion made the A2 writes visible to this
          // thread; the proxy fence orders them (async proxy) before the
          // release store, whose cumulativity publishes them to every
          // consumer that acquires the flag (and fences its own async proxy
          // before loading A2 by TMA, ensure_ready / check_ready).
          fence_proxy_async_global();
          st_release(a.flags + pc.tile, a.epoch);
        }
        if (acc_it == 0) trace_stamp(a, 22);
      }
    } else if (!pc.down) {
      int is_up, cofs;
      s1_row_map(row, &is_up, &cofs);
      const int col = pc.tile * kS1Cols + cofs;
      for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
        float v[16];
        tmem_ld16_sum(taddr + c0, nacc, astr, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float up = __shfl_xor_sync(0xffffffffu, v[e], 16);
          const int n = c0 + e;
          if (!is_up && n < a.B && col < a.cols_valid) {
            float act = silu_f(v[e]);
            if (a.mutant == 2) {
              // MaterializeIntermediate negative control
              // (verification.cpp:126-169): SiLU(A_gate) round-trips through
              // a global buffer -- same numbers, extra global traffic.
              float* slot = a.mat_scratch + static_cast<int64_t>(n) * a.cols_valid + col;
              asm volatile("st.global.cg.f32 [%0], %1;" ::"l"(slot), "f"(act) : "memory");
              asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(act) : "l"(slot) : "memory");
            }
            a.a2[n * a.a2_ld + col] = __float2bfloat16_rn(act * up);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      if (a.flags) s1_publish(a, pc.tile, tid, 128);
    } else {
      // One predicated red.global.add per (row j, batch n): straight-line
      // code (the epilogue runs from a cold instruction cache once per piece).
      const bool stamp = a.trace && a.trace_s0 < 0 && !dn_stamped;
      dn_stamped = dn_stamped || stamp;
      if (stamp && tid == 0) trace_stamp(a, 40);
      const int j = pc.tile * kDownCols + row;
      const bool jok = j < a.out_cols;
      if (a.y_direct && !y_zeroed) {
        direct_y_wait(a, tid, 128);
        y_zeroed = true;
      }
      float* yp = a.y_direct ? reinterpret_cast<float*>(a.y) + j : down_acc(a, pc.tile) + j;
      const int64_t ld = a.y_direct ? a.y_ld : a.yacc_ld;
      // v4 reductions over whole 4-column groups (the condition is
      // warp-uniform: the shuffles involve all 32 lanes); under the fused TP
      // all-reduce always, at system scope (the owner's workspace may be on
      // another GPU: 4x fewer NVLink reductions)
      const bool tp = a.tp_size > 1;
      const bool vec = (a.red_v4 || tp || a.y_direct) &&
                       __all_sync(0xffffffffu, j - (lane & 3) + 3 < a.out_cols);
      for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
        float v[16];
        tmem_ld16_sum(taddr + c0, nacc, astr, v);
        if (vec) {
          if (tp)
            red_rows_v4<true>(v, yp - (lane & 3), ld, c0, a.B, lane);
          else
            red_rows_v4(v, yp - (lane & 3), ld, c0, a.B, lane);
        } else {
          float* yc = yp + c0 * ld;
          if (tp) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              red_add_sys_f32_if(yc + e * ld, v[e], jok && c0 + e < a.B);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) red_add_f32_if(yc + e * ld, v[e], jok && c0 + e < a.B);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      if (!a.y_direct)
        down_finish_tile(a, p, pc.tile, pc.kb1 - pc.kb0, tid, 128, smem_flag, stamp);
    }
    if (tid == 0) trace_stamp(a, 2 + 2 * pi.i);
    ++acc_it;
  }
  if (tid == 0) trace_stamp(a, 2);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* ptr) {
  return reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(ptr) + 1023) & ~static_cast<uintptr_t>(1023));
}

// ---------------------------------------------------------------------------
// The kernel.
// ---------------------------------------------------------------------------
template <int kMode, bool kTC, int NB>
__global__ void __launch_bounds__(kTC ? kTcThreads : kGemvThreads, 1)
    stream_kernel(const __grid_constant__ CUtensorMap xmap,
                  const __grid_constant__ CUtensorMap amap,
                  const __grid_constant__ CUtensorMap a3map,
                  const StreamArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int stage_bytes = stream_stage_bytes(a.n_pad, a.kbs);
  // A2 staging tile right after the ring (1024-aligned: the 128B swizzle)
  uint8_t* a2st = smem + a.stages * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(a2st + a2_stage_bytes(a.n_pad, a.a2_tma));
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  PieceQueue* pq = reinterpret_cast<PieceQueue*>(
      (reinterpret_cast<uintptr_t>(tempty + 2) + 15) & ~static_cast<uintptr_t>(15));
  uint64_t* red_full = reinterpret_cast<uint64_t*>(pq + 1);
  uint64_t* red_free = red_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_free + 1);
  int* smem_flag = reinterpret_cast<int*>(tmem_slot + 1);
  // The producer's deferred-stage list (one int4 per ring slot), then the
  // split-K reduction buffer, 16-byte aligned.
  int4* pend = reinterpret_cast<int4*>(
      (reinterpret_cast<uintptr_t>(smem_flag + 4) + 15) & ~static_cast<uintptr_t>(15));
  float* red = reinterpret_cast<float*>(pend + a.stages);
  const bool split = kMode != kModeDown && a.split_k > 1;

  const uint32_t w = warp_id();
  if (w == 0 && lane_id() == 0) {
    if (kMode != kModeDown) prefetch_tmap(&xmap);
    if (kMode != kModeStage1) prefetch_tmap(&amap);
    if (kMode != kModeStage1 && a.a3d) prefetch_tmap(&a3map);
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTC ? 1 : kGemvWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    for (int i = 0; i < kPieceQueue; ++i) {
      mbar_init(&pq->full[i], 1);
      mbar_init(&pq->empty[i], kTC ? 5 : kGemvWarps);
    }
    if (split) {
      mbar_init(red_full, 1);  // the leader's expect_tx; partners count bytes
      mbar_init(red_free, 4);  // one per leader epilogue warp
    }
    fence_barrier_init();
  }

  uint32_t tmem_cols = 0;
  if constexpr (kTC) {
    tmem_cols = 32;
    const int nacc = a.nacc > 0 ? a.nacc : 1;
    while (tmem_cols < static_cast<uint32_t>(2 * nacc * a.n_pad)) tmem_cols <<= 1;
    if (w == 1) tmem_alloc(tmem_slot, tmem_cols);
  }
  __syncthreads();
  if (split) cluster_sync();  // barriers initialised + buffer zeroed cluster-wide
  tc_fence_after();
  const uint32_t tmem_base = kTC ? *tmem_slot : 0u;
  const Plan plan = make_plan(a, kMode);
  if (threadIdx.x == 0) trace_stamp(a, 0);

  // Let the next kernel in the stream get scheduled as SMs drain; it only
  // touches our outputs after its own griddepcontrol.wait.
  const bool late_trigger = kMode == kModeBlock && a.tp_size > 1 && a.tp_late_trigger;
  if (!late_trigger) pdl_launch_dependents();

  if (w == 0) {
    produce(a, plan, &xmap, &amap, &a3map, smem, stage_bytes, full, empty, pq, pend);
  } else if constexpr (kTC) {
    if (w == 1) {
      if (lane_id() == 0)
        mma_issue(a, plan, smem, stage_bytes, full, empty, tfull, tempty,
                  tmem_base, pq);
    } else {
      tc_epilogue(a, plan, tfull, tempty, tmem_base, smem_flag, pq, red, red_full,
                  red_free, &amap, a2st);
    }
  } else {
    gemv_consume<NB>(a, plan, smem, stage_bytes, full, empty, smem_flag, pq);
  }

  __syncthreads();
  // Fused TP all-reduce: this rank's Y tiles into the caller's buffer.
  if (kMode == kModeBlock && a.tp_size > 1) {
    tp_collect_y(a, smem_flag);
    __syncthreads();
    if (late_trigger) pdl_launch_dependents();
  }
  if (a.dynamic && threadIdx.x == 0) {
    // The last CTA out re-arms the work counter for the next launch.
    if (atom_add_acq_rel_gpu(a.sched + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      if (a.x_free) {  // device-scope release: read by stream waits / copy engines
        st_release(a.x_free, a.x_seq);
        if (a.y_done) st_release(a.y_done, a.x_seq);
      }
      a.sched[0] = 0;
      a.sched[1] = 0;
      a.sched[2] = 0;
      fence_acq_rel_gpu();
    }
  }
  if (split) cluster_sync();  // no CTA leaves while peers may touch its smem
  if constexpr (kTC) {
    if (w == 1) {
      __syncwarp();
      tc_fence_after();
      tmem_dealloc(tmem_base, tmem_cols);
    }
  }
}

// Opt every kernel instantiation in to the device's full dynamic shared
// memory once (the per-launch amount is set in the launch config).
cudaError_t allow_max_smem(const void* kern) {
  // Function attributes are per device (context): cache by (device, kernel),
  // under a lock (contexts may be created from several host threads).
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, kern})) return cudaSuccess;
  int max_optin = 0;
  e = cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin);
  if (e == cudaSuccess) done.insert({dev, kern});
  return e;
}

template <int kMode, bool kTC, int NB>
cudaError_t launch_one(const CUtensorMap& xmap, const CUtensorMap& amap,
                       const CUtensorMap& a3map, const StreamArgs& a, int grid, int smem,
                       bool pdl, cudaStream_t stream) {
  auto kern = stream_kernel<kMode, kTC, NB>;
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kTC ? kTcThreads : kGemvThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (a.split_k > 1 && kMode != kModeDown) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = static_cast<unsigned>(a.split_k);
    attrs[na].val.clusterDim.y = 1;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, xmap, amap, a3map, a);
}

template <int kMode>
cudaError_t launch_mode(bool tc, int nb, const CUtensorMap& xmap,
                        const CUtensorMap& amap, const CUtensorMap& a3map,
                        const StreamArgs& a, int grid, int smem, bool pdl, cudaStream_t s) {
  if (tc) return launch_one<kMode, true, 0>(xmap, amap, a3map, a, grid, smem, pdl, s);
  switch (nb) {
    case 1: return launch_one<kMode, false, 1>(xmap, amap, a3map, a, grid, smem, pdl, s);
    case 2: return launch_one<kMode, false, 2>(xmap, amap, a3map, a, grid, smem, pdl, s);
    case 4: return launch_one<kMode, false, 4>(xmap, amap, a3map, a, grid, smem, pdl, s);
    case 8: return launch_one<kMode, false, 8>(xmap, amap, a3map, a, grid, smem, pdl, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// Force-load (see preload_aux_kernels) and opt in every instantiation.
cudaError_t preload_stream_kernels() {
  const void* fns[] = {
#define DFK_K(m) \
  reinterpret_cast<const void*>(stream_kernel<m, true, 0>),  \
      reinterpret_cast<const void*>(stream_kernel<m, false, 1>), \
      reinterpret_cast<const void*>(stream_kernel<m, false, 2>), \
      reinterpret_cast<const void*>(stream_kernel<m, false, 4>), \
      reinterpret_cast<const void*>(stream_kernel<m, false, 8>)
      DFK_K(kModeStage1), DFK_K(kModeDown), DFK_K(kModeBlock)
#undef DFK_K
  };
  for (const void* f : fns) {
    cudaFuncAttributes at;
    cudaError_t e = cudaFuncGetAttributes(&at, f);
    if (e == cudaSuccess) e = allow_max_smem(f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// How many clusters of `split` CTAs (with this kernel's smem) can be
// co-resident; clusters beyond it would run in a second wave (and, in the
// block kernel, spin on flags of tiles whose CTAs are not resident yet).
int stream_max_clusters(int mode, int split, int smem) {
  if (split <= 1) return 1 << 30;
  auto kern = mode == kModeBlock ? stream_kernel<kModeBlock, true, 0>
                                 : stream_kernel<kModeStage1, true, 0>;
  allow_max_smem(reinterpret_cast<const void*>(kern));
  if (split > 8)
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(split * 64));
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = static_cast<unsigned>(split);
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return n > 0 ? n : 1;
}

int stream_smem_bytes(int n_pad, int stages, int kbs, int split_k, int a2_tma) {
  return 1024 + stages * stream_stage_bytes(n_pad, kbs) + a2_stage_bytes(n_pad, a2_tma) + (2 * stages + 4) * 8 +
         static_cast<int>(sizeof(PieceQueue)) + 128 + 16 * stages + split_red_bytes(n_pad, split_k);
}

cudaError_t launch_stream(int mode, bool tc, int nb_gemv,
                          const CUtensorMap& xmap, const CUtensorMap& amap,
                          const StreamArgs& a, int grid, bool pdl,
                          cudaStream_t stream, const CUtensorMap* a3map) {
  if (a.a3d && !a3map) return cudaErrorInvalidValue;
  const CUtensorMap& a3 = a3map ? *a3map : amap;
  if (a.kbs < 1 || a.kbs > kMaxKbs || a.stages < 2 || a.stages > 32)
    return cudaErrorInvalidValue;
  if (a.split_k > 1 && (!tc || a.split_k > 8 || grid % a.split_k != 0 ||
                        (a.dynamic && (mode != kModeBlock || a.bal ||
                                       a.t1 * a.split_k > grid))))
    return cudaErrorInvalidValue;
  if (a.nacc > 4 || (a.nacc > 1 && (a.split_k > 1 || 2 * a.nacc * a.n_pad > 512)))
    return cudaErrorInvalidValue;
  if (a.a2_tma && (!tc || a.split_k > 1 || mode == kModeDown)) return cudaErrorInvalidValue;
  const int smem = stream_smem_bytes(a.n_pad, a.stages, a.kbs,
                                     mode == kModeDown ? 1 : a.split_k, a.a2_tma);
  switch (mode) {
    case kModeStage1:
      return launch_mode<kModeStage1>(tc, nb_gemv, xmap, amap, a3, a, grid, smem, pdl, stream);
    case kModeDown:
      return launch_mode<kModeDown>(tc, nb_gemv, xmap, amap, a3, a, grid, smem, pdl, stream);
    case kModeBlock:
      return launch_mode<kModeBlock>(tc, nb_gemv, xmap, amap, a3, a, grid, smem, pdl, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace dfk
