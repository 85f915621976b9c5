// stream_kernels.cuh — argument block shared by the host launchers
// (api.cu) and the weight-streaming kernels (stream_kernels.cu).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace dfk {

// kModeStage1: fused gate/up GEMM + SiLU*up epilogue -> A2 (one kernel).
// kModeDown:   A2 W_down, stream-K over (tile, K block) -> Y.
// kModeBlock:  the whole block in ONE persistent kernel: every CTA first
//              streams its stage-1 tiles, then down pieces; a down piece's
//              A2 block is loaded only after the stage-1 tile that produced
//              it published its completion flag (epoch-tagged).
enum StreamMode : int { kModeStage1 = 0, kModeDown = 1, kModeBlock = 2 };

constexpr int kMaxTp = 8;  // ranks of the fused TP all-reduce

struct StreamArgs {
  // Stage-1 pack ([W_gate|W_up] interleaved): t1 tiles x kb1 K blocks.
  const uint8_t* w1;
  int t1, kb1;
  // Down pack (W_down): t2 tiles x kb2 K blocks (kb2 == t1: one K block of
  // the down projection per stage-1 tile).
  const uint8_t* w2;
  int t2, kb2;
  int B;       // batch rows present
  int n_pad;   // MMA N (tcgen05) / activation box rows (GEMV)
  int xrows;   // rows per activation TMA box (<= n_pad; the smem tile is n_pad rows)
  // x3d: xmap is 3-D (64 K x xrows x K blocks, the K-block dimension 128 B
  // apart), so ONE TMA per ring stage brings the X rows of all its K blocks,
  // packed xrows x 128 B per K block (the MMA's N = 16 operand then reads
  // rows 8..15 of a B <= 8 block from the next block: they only feed
  // discarded accumulator columns).  Stage-1 loads only.
  int x3d;
  int a3d;     // the same for the down pieces' A2 loads (a3map)
  // Stage-1 A2 leaves through a swizzled smem tile and ONE TMA store per tile
  // (amap, box 64 x xrows) instead of per-element stores (tcgen05 family,
  // whole tiles; host sets it when A2 is TMA-addressable).
  int a2_tma;
  int stages;  // ring depth
  // split_k (field below) > 1: stage-1 tiles are split along K over the
  // split_k CTAs of a thread-block cluster; partial gate/up accumulators are
  // reduced into the leader CTA's shared memory through DSMEM
  // (red.shared::cluster) before the SiLU*up epilogue, so partial sums never
  // leave the SMs.  Static plan, tcgen05 family only.
  int split_k;
  int kbs;     // K blocks (16 KiB each) per ring stage
  // Stage-1 output: A2 [B x a2_ld] bf16, columns < cols_valid written.
  __nv_bfloat16* a2;
  int64_t a2_ld;
  int cols_valid;
  // Down output: fp32 accumulation workspace (zero on entry; re-zeroed by
  // the CTA that finalises each tile), per-tile arrival counters (zero on
  // entry, reset on finalise), final Y [B x y_ld] fp32 or bf16.
  float* yacc;
  int yacc_ld;
  int* counters;
  void* y;
  int64_t y_ld;
  int y_bf16;
  int y_vec4;  // fp32 Y, 16-byte aligned rows: float4 stores
  // Direct Y (kModeBlock, dynamic queue, tcgen05, one GPU, fp32 Y in device
  // memory): after griddepcontrol.wait every CTA's epilogue warps zero their
  // 1/G slice of Y and count it on sched[2]; down pieces red.add their
  // partial sums straight into Y once sched[2] == G.  No per-tile counter,
  // no finalize pass and no workspace re-zeroing on the launch's tail.
  int y_direct;
  // tcgen05: independent accumulators per tile (MMA k of a K block goes to
  // accumulator k % nacc), so consecutive MMAs do not serialise on one
  // accumulator; the epilogue sums them.  TMEM = 2 x nacc x n_pad columns.
  int nacc;
  // Host-buffer path (dfk_forward_host_async): X arrives by a copy-engine
  // memcpy on a side stream, which then writes x_seq to *x_ready; the
  // producer waits for it before the first activation load, and the last CTA
  // out stores x_seq to *x_free (the staging slot may be overwritten).
  const unsigned* x_ready;
  unsigned* x_free;
  unsigned* y_done;  // x_seq stored here too: Y complete, the side stream copies it out
  unsigned x_seq;
  int out_cols;
  // kModeBlock: per-stage-1-tile completion flags and this launch's epoch.
  unsigned* flags;
  unsigned epoch;
  // Negative controls (tests only): 1 = SiLU*up per K chunk (stream-K /
  // split-K pieces), 2 = SiLU(A_gate) materialised in mat_scratch
  // [B x cols_valid] fp32 and read back before the multiply.
  int mutant;
  float* mat_scratch;
  // kModeBlock plan (host-computed, block_plan in api.cu).  Stage-1 tiles go
  // round-robin: CTAs c < r own q+1 tiles ("heavy"), the rest own q
  // ("light").  Down units form two groups, each split over all G ranks
  // (light CTA c has rank c - r, heavy CTA c has rank L + c):
  //   A = K blocks [0, kB0) whose stage-1 tile is in an early wave: t-major
  //       segments of nA units; light ranks get al, heavy ah (al - ah = one
  //       stage-1 tile of K blocks), +1 for the first rA ranks;
  //   B = K blocks [kB0, kb2) of the last wave: t-major segments of nB
  //       units, bl per rank, +1 for the first rB ranks.
  // A CTA runs its stage-1 tiles, then its A range, then its B range.
  int bp_r, bp_L, bp_nA, bp_nB, bp_kB0;
  int64_t bp_al, bp_ah, bp_rA, bp_bl, bp_rB;
  // Dynamic scheduling (dynamic != 0): pieces are handed out by an atomic
  // work counter instead of the static plan.  Piece index i: i < t1 (modes
  // Stage1/Block) = stage-1 tile i; then down chunks of chunk_kb K blocks,
  // chunk-major (all t2 tiles of K chunk 0, then chunk 1, ...).  CTA c takes
  // piece c first (prefetched before griddepcontrol.wait), then
  // G + atomicAdd(sched[0], 1); the last CTA to exit resets sched[0..1].
  int dynamic;
  int chunk_kb;
  int* sched;
  // Stage-1 stream-K (dynamic path): a stage-1 piece covers s1_chunk K
  // blocks of one tile (s1_chunk >= kb1 or 0: whole tiles).  Partial
  // gate/up accumulators go to the fp32 workspace s1acc [t1][n_pad][128]
  // with red.global.add; the CTA adding a tile's last piece (s1cnt arrival
  // counter) applies SiLU*up to the FULL sums, writes A2, publishes the
  // tile's flag and re-zeroes its workspace and counter.  Lets every SM
  // stream stage-1 weights when a (TP) shard has fewer tiles than SMs.
  int s1_chunk;
  // Tail split (dynamic path, whole-tile s1_chunk): the first s1_whole
  // stage-1 tiles are whole pieces (one wave over the grid), every later
  // tile is split into s1_tail K parts (stream-K through s1acc), so the
  // last stage-1 wave is spread over all CTAs instead of a fraction of them.
  int s1_tail;
  int s1_whole;
  // Balanced stream-K (dynamic machinery, static pieces): CTA c takes the
  // K-block ranges [c*U/G, (c+1)*U/G) of the flattened stage-1 space
  // (U = t1*kb1) and then of the down space (U = t2*kb2), split at tile
  // boundaries -- every CTA streams the same bytes in both phases.  Tile
  // counters then count K blocks (a tile is complete when kb1 / kb2 of them
  // have arrived).
  int bal;
  float* s1acc;
  int* s1cnt;
  // K blocks of the first piece prefetched into L2 (cp.async.bulk.prefetch)
  // beyond the smem ring BEFORE griddepcontrol.wait: under PDL the HBM
  // stream of this launch starts during the previous launch's tail.
  int pf_kb;
  // Fused tensor-parallel all-reduce (kModeBlock + dynamic, tp_size > 1):
  // down tile t is OWNED by rank t % tp_size.  Every rank red.adds its
  // partial sums of tile t into the owner's fp32 workspace tp_yacc[owner]
  // over NVLink peer memory (system scope, v4) and counts the K blocks it
  // contributed on the owner's tp_cnt[owner][t]; the CTA (on any rank) that
  // completes the tile's tp_total_kb K blocks reads the full sums, stores
  // them into EVERY rank's full-sum slot tp_y[r] (the all-gather, by push),
  // re-zeroes the owner's workspace and counter and raises every rank's
  // tp_done[r][t].  At the end of the launch each rank's CTAs wait for their
  // tiles' done words (local memory), copy the tiles into the caller's Y
  // (y, fp32 or bf16) and re-arm the words: the launch completes with the
  // all-reduced Y in place -- the block's one collective inside its one
  // kernel, overlapped with the down stream.
  int tp_rank, tp_size, tp_total_kb;
  float* tp_yacc[kMaxTp];
  int* tp_cnt[kMaxTp];
  int* tp_done[kMaxTp];  // per down tile
  float* tp_y[kMaxTp];
  // A peer rank shares this GPU: trigger the next PDL launch only after
  // this rank's Y is complete (an early dependent would occupy the SMs the
  // peer's kernel needs to make progress).
  int tp_late_trigger;
  // Error word (host-mapped; dfk_context_sync reports it): set when a wait
  // on another rank (or on the host path's X copy) gives up after 4 s.
  int* tp_error;
  // Optional timeline (tools/trace_block.py): per CTA kTraceSlots globaltimer
  // stamps: [0] start, [1] producer done, [2] consumer done, then per piece
  // i < 8: [3+2i] piece fetched (its first weight copy follows), [4+2i]
  // piece retired, [24+i] descriptor (down << 48 | K blocks << 32 | tile),
  // [32+i] first activation load; ring stages trace_s0 + j, j < 12:
  // [40+j] weight copy issued, [52+j] full barrier passed (MMA lane).
  unsigned long long* trace;
  int trace_s0;
  // trace_rel: slots 40+j / 52+j record when the producer saw ring stage
  // trace_s0+j released / when the MMA lane finished issuing it (instead of
  // weight-copy issue / full-barrier pass).
  int trace_rel;
  // Partial-sum reductions (stage-1 stream-K, down pieces) as
  // red.global.add.v4.f32 after a 4 x 4 lane transpose (small shards).
  int red_v4;
};

constexpr int kTraceSlots = 64;
constexpr int kPieceQueue = 8;  // producer -> consumers piece queue depth

// Smem bytes of one pipeline stage (weights + activation rows).
__host__ __device__ inline int stream_stage_bytes(int n_pad, int kbs) {
  return kbs * (16384 + n_pad * 128);
}

// Stage-1 split-K reduction buffer (leader CTA of a cluster): one fp32
// [128][N + 4] slot per non-leader rank (row-major, padded against bank
// conflicts of the 16-byte accesses).
__host__ __device__ inline int split_row_floats(int n_pad) { return n_pad + 4; }
__host__ __device__ inline int split_red_bytes(int n_pad, int split_k) {
  return split_k > 1 ? (split_k - 1) * 128 * split_row_floats(n_pad) * 4 : 0;
}

cudaError_t launch_stream(int mode, bool tc, int nb_gemv, const CUtensorMap& xmap,
                          const CUtensorMap& amap, const StreamArgs& a, int grid,
                          bool pdl, cudaStream_t stream,
                          const CUtensorMap* a3map = nullptr);  // 3-D A2 loads (a3d)

int stream_smem_bytes(int n_pad, int stages, int kbs, int split_k = 1, int a2_tma = 0);
// Bytes of the A2 staging tile (a2_tma): n_pad rows of 128 B.
__host__ __device__ inline int a2_stage_bytes(int n_pad, int a2_tma) {
  return a2_tma ? n_pad * 128 : 0;
}
int stream_max_clusters(int mode, int split, int smem);
cudaError_t preload_stream_kernels();

}  // namespace dfk
