// stream_kernels.cuh — argument block shared by the host launchers
// (api.cu) and the weight-streaming kernels (stream_kernels.cu).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace dfk {

enum StreamMode : int { kModeStage1 = 0, kModeDown = 1 };

struct StreamArgs {
  const uint8_t* wpack;  // packed weight blocks (layout.cuh)
  int tiles;             // weight tiles (128 rows each)
  int kblocks;           // 64-wide K blocks per tile
  int B;                 // batch rows actually present
  int n_pad;             // MMA N (tcgen05) / X box rows (GEMV)
  int stages;            // pipeline depth
  int split_k;           // stage 1: CTAs of a cluster sharing one tile
  // Stage 1 output: A2 [B x a2_ld] bf16, columns < cols_valid written.
  __nv_bfloat16* a2;
  int64_t a2_ld;
  int cols_valid;
  // Down output: fp32 accumulation workspace (self-cleaning: zero on entry,
  // re-zeroed by the CTA that finalises each tile), per-tile completion
  // counters (zero on entry, reset on finalise), final Y [B x y_ld].
  float* yacc;
  int yacc_ld;
  int* counters;
  void* y;
  int64_t y_ld;
  int y_bf16;
  int out_cols;
  // Debug / negative control: 1 = apply SiLU per K-chunk of a split-K tile
  // (the reference's SiluPerKChunk mutant, verification.cpp:84-124).
  int mutant;
};

// Smem bytes of one pipeline stage (weights + activation rows).
__host__ __device__ inline int stream_stage_bytes(int n_pad) { return 16384 + n_pad * 128; }

// Launchers (stream_kernels.cu). `tc` selects the tcgen05 family, else the
// CUDA-core GEMV family.  grid = CTAs (multiple of split_k).  Returns the
// cudaError of the launch.
cudaError_t launch_stream(int mode, bool tc, int nb_gemv, const CUtensorMap& xmap,
                          const StreamArgs& a, int grid, bool pdl,
                          cudaStream_t stream);

// Max dynamic smem the launcher will request for (tc, n_pad, stages).
int stream_smem_bytes(bool tc, int n_pad, int stages, int split_k);

}  // namespace dfk
