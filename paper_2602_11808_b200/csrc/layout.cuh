// layout.cuh — the HBM layout of prepacked weights, shared by the pack
// kernels (host-launched, once per weight registration) and the streaming
// kernels.
//
// Every weight matrix is stored as a sequence of 16 KiB "blocks": 128 rows x
// 64 K-elements of bf16, K-major, in exactly the 128B-swizzled image that the
// UMMA shared-memory descriptor (SWIZZLE_128B, K-major, SBO = 1024 B) and the
// GEMV consumers read.  One block is one contiguous 1-D bulk copy
// (cp.async.bulk) from HBM into a pipeline stage, so the weight stream is
// fully sequential per tile: tile t, K-block kb lives at byte offset
// (t * kblocks + kb) * 16384.  Rows / K beyond the matrix are zero-filled,
// which is exact for SwiGLU (silu(0) * 0 = 0, 0 * w = 0).
//
// Stage 1 (W_gate | W_up, reference layout [d_model x d_ff] row-major,
// swiglu.hpp:49-52): tile t covers A2 columns [64t, 64t+64).  Its 128 rows
// interleave gate and up in 16-row groups — row r = 32g + w holds
//   w <  16: W_gate[:, 64t + 16g + w]
//   w >= 16: W_up  [:, 64t + 16g + w - 16]
// so in the TMEM accumulator (row r == TMEM lane r) the gate and up values of
// one A2 column sit in the same warp, 16 lanes apart (one shfl.xor 16).
//
// Down (W_down, reference [d_ff x d_model] row-major): tile t covers Y
// columns [128t, 128t+128); row r holds W_down[:, 128t + r]; K runs over d_ff.
#pragma once

#include <cstdint>

namespace dfk {

constexpr int kBlockRows = 128;            // MMA M / rows per block
constexpr int kBlockK = 64;                // K elements per block row (128 B)
constexpr int kBlockBytes = kBlockRows * kBlockK * 2;  // 16 KiB
constexpr int kS1Cols = 64;                // A2 columns per stage-1 tile
constexpr int kDownCols = 128;             // Y columns per down tile

__host__ __device__ inline int64_t ceil_div64(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

// Element offset of (row r, k) inside one swizzled block: 16-byte chunk
// index (k / 8) is XOR-ed with (r mod 8), matching the hardware's 128B
// swizzle of a 1024-byte-aligned 8-row atom.
__host__ __device__ inline int block_elem_offset(int r, int k) {
  return r * kBlockK + ((((k >> 3) ^ (r & 7)) << 3) | (k & 7));
}

// Stage-1 row -> (is_up, A2 column offset inside the 64-column tile).
__host__ __device__ inline void s1_row_map(int r, int* is_up, int* col) {
  const int g = r >> 5, w = r & 31;
  *is_up = w >= 16 ? 1 : 0;
  *col = g * 16 + (w & 15);
}

}  // namespace dfk
