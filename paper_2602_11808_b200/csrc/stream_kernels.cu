// stream_kernels.cu — the hot path: weight-streaming kernels for the fused
// SwiGLU MLP on sm_100a.
//
// One kernel template covers both stages of the block and both consumer
// families:
//
//   mode  kModeStage1  A2 = (X W_up) * silu(X W_gate)     (fused.cpp:74-168,
//                      DeepFusionKernel: gate and up accumulate side by side,
//                      the SiLU*up epilogue runs once per element after the
//                      FULL K reduction, A2 is the only global write)
//   mode  kModeDown    Y = A2 W_down                      (swiglu.cpp:214-226)
//
//   family tcgen05     weights are the MMA M=128 operand, the batch is MMA N
//                      (swap-AB), fp32 accumulators in TMEM, epilogue via
//                      tcgen05.ld ("F2")
//   family GEMV        8 CUDA-core warps dot the same smem stages with fp32
//                      FMAs, warp-shuffle reductions (batch 1-8, "F1")
//
// Common skeleton (warp-specialised, persistent, one CTA per SM):
//   warp 0      producer: 16 KiB weight blocks HBM->smem with 1-D bulk copies
//               (cp.async.bulk, L2 evict_first) + the activation rows of the
//               same K block with a 2-D TMA (128B swizzle) into a ring of
//               `stages` slots, completion counted in bytes on mbarriers.
//               The first ring's weight copies are issued BEFORE
//               griddepcontrol.wait, so under PDL they overlap the previous
//               kernel's tail; activations are only read after the wait.
//   warp 1      tcgen05: one lane issues 4 x (M128 x N x K16) MMAs per block
//               and tcgen05.commit's the slot back to the producer.
//   warps 2-5   tcgen05 epilogue (TMEM lane quarter = warp % 4).
//   warps 1-8   GEMV family: math warps (no TMEM).
//
// Work split: stage 1 hands whole tiles (64 A2 columns x full d_model) to
// CTAs round-robin, so partial gate/up sums never leave the SM.  Down is
// stream-K: the flattened (tile, K-block) space is cut into gridDim equal
// ranges; each CTA reduces its pieces into an fp32 workspace with
// red.global.add, and the CTA that completes a tile's last piece (per-tile
// arrival counter) converts it to the output dtype and re-zeroes the
// workspace, so no memset is ever needed.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "layout.cuh"
#include "ptx.cuh"
#include "stream_kernels.cuh"

namespace dfk {

namespace {

constexpr int kTcThreads = 192;    // producer, MMA, 4 epilogue warps
constexpr int kGemvThreads = 288;  // producer + 8 math warps
constexpr int kGemvWarps = 8;

struct Seg {
  int tile, kb0, kb1;
};

// The i-th (tile, K range) piece of this CTA's work.
__device__ __forceinline__ bool seg_get(const StreamArgs& a, int mode, int i,
                                        Seg& s) {
  const int G = gridDim.x, c = blockIdx.x;
  if (mode == kModeStage1) {
    const int t = c + i * G;
    if (t >= a.tiles) return false;
    s.tile = t;
    s.kb0 = 0;
    s.kb1 = a.kblocks;
    return true;
  }
  const int64_t U = static_cast<int64_t>(a.tiles) * a.kblocks;
  const int64_t u0 = U * c / G, u1 = U * (c + 1) / G;
  const int t = static_cast<int>(u0 / a.kblocks) + i;
  const int64_t ts = static_cast<int64_t>(t) * a.kblocks;
  if (ts >= u1) return false;
  s.tile = t;
  s.kb0 = static_cast<int>(u0 > ts ? u0 - ts : 0);
  s.kb1 = static_cast<int>(u1 - ts < a.kblocks ? u1 - ts : a.kblocks);
  return s.kb0 < s.kb1;
}

__device__ __forceinline__ int64_t cta_work_blocks(const StreamArgs& a,
                                                   int mode) {
  const int G = gridDim.x, c = blockIdx.x;
  if (mode == kModeStage1) {
    const int mine = c < a.tiles ? (a.tiles - 1 - c) / G + 1 : 0;
    return static_cast<int64_t>(mine) * a.kblocks;
  }
  const int64_t U = static_cast<int64_t>(a.tiles) * a.kblocks;
  return U * (c + 1) / G - U * c / G;
}

// Number of CTAs whose stream-K range touches down tile t (all ranges are
// non-empty because the launcher keeps gridDim <= tiles * kblocks).
__device__ __forceinline__ int down_contributors(const StreamArgs& a, int t) {
  const int64_t U = static_cast<int64_t>(a.tiles) * a.kblocks;
  const int64_t G = gridDim.x;
  const int64_t lo = static_cast<int64_t>(t) * a.kblocks;
  const int64_t hi = lo + a.kblocks;
  const int64_t c_first = ((lo + 1) * G + U - 1) / U - 1;
  const int64_t c_last = (hi * G + U - 1) / U - 1;
  return static_cast<int>(c_last - c_first + 1);
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Down epilogue tail: publish this CTA's contribution to tile t; the last
// contributor converts the tile to the output dtype and re-zeroes it.
__device__ __forceinline__ void down_finish_tile(const StreamArgs& a, int t,
                                                 int tid, int nthr,
                                                 int* smem_flag) {
  __threadfence();
  named_bar(1, nthr);
  if (tid == 0) {
    const int old = atomicAdd(&a.counters[t], 1);
    *smem_flag = (old == down_contributors(a, t) - 1) ? 1 : 0;
  }
  named_bar(1, nthr);
  if (*smem_flag) {
    __threadfence();
    const int col0 = t * kDownCols;
    for (int idx = tid; idx < a.B * kDownCols; idx += nthr) {
      const int n = idx / kDownCols, j = col0 + idx % kDownCols;
      if (j < a.out_cols) {
        float* p = a.yacc + static_cast<int64_t>(n) * a.yacc_ld + j;
        const float v = __ldcg(p);
        if (a.y_bf16) {
          reinterpret_cast<__nv_bfloat16*>(a.y)[n * a.y_ld + j] =
              __float2bfloat16_rn(v);
        } else {
          reinterpret_cast<float*>(a.y)[n * a.y_ld + j] = v;
        }
        __stcg(p, 0.0f);
      }
    }
    if (tid == 0) a.counters[t] = 0;
  }
  named_bar(1, nthr);
}

// ---------------------------------------------------------------------------
// Producer (one lane): ring of `stages` slots; the first ring's weight
// copies go out before griddepcontrol.wait (PDL overlap), activations after.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void produce(const StreamArgs& a, int mode,
                                        const CUtensorMap* xmap, uint8_t* smem,
                                        int stage_bytes, uint64_t* full,
                                        uint64_t* empty) {
  const uint64_t policy = policy_evict_first();
  const int64_t total = cta_work_blocks(a, mode);
  const int pre = static_cast<int>(total < a.stages ? total : a.stages);
  const uint32_t x_bytes = static_cast<uint32_t>(a.n_pad) * 128u;
  const uint32_t bytes = static_cast<uint32_t>(kBlockBytes) + x_bytes;
  int pend_kb[32];
  int64_t it = 0;
  Seg s;
  for (int i = 0; seg_get(a, mode, i, s); ++i) {
    for (int kb = s.kb0; kb < s.kb1; ++kb, ++it) {
      const int slot = static_cast<int>(it % a.stages);
      const uint32_t phase = static_cast<uint32_t>((it / a.stages) & 1);
      if (it >= a.stages) mbar_wait(&empty[slot], phase ^ 1u);
      uint8_t* st = smem + static_cast<int64_t>(slot) * stage_bytes;
      mbar_arrive_expect_tx(&full[slot], bytes);
      const uint8_t* src =
          a.wpack + (static_cast<int64_t>(s.tile) * a.kblocks + kb) *
                        static_cast<int64_t>(kBlockBytes);
      bulk_g2s(st, src, kBlockBytes, &full[slot], policy);
      if (it < pre) {
        pend_kb[it] = kb;
        if (it == pre - 1) {
          pdl_wait();
          for (int j = 0; j < pre; ++j) {
            tma_load_2d(smem + static_cast<int64_t>(j) * stage_bytes +
                            kBlockBytes,
                        xmap, pend_kb[j] * kBlockK, 0, &full[j]);
          }
        }
      } else {
        tma_load_2d(st + kBlockBytes, xmap, kb * kBlockK, 0, &full[slot]);
      }
    }
  }
  if (pre == 0) pdl_wait();
}

// ---------------------------------------------------------------------------
// GEMV math warps (batch <= NB). Lane = (q, c): c = 16-byte chunk of the
// 64-wide K block, q = one of 4 rows this warp handles per pass; 4 passes
// cover the 32-row group of each pass p.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int gemv_row(int p, int mw, int q) {
  // q 0,1 -> gate rows 2mw+q, q 2,3 -> matching up rows (16 apart), so the
  // gate/up pair of one A2 column is lane ^ 16 within the warp.
  return p * 32 + (q < 2 ? 2 * mw + q : 16 + 2 * mw + (q - 2));
}

template <int kMode, int NB>
__device__ __forceinline__ void gemv_consume(const StreamArgs& a,
                                             uint8_t* smem, int stage_bytes,
                                             uint64_t* full, uint64_t* empty,
                                             int* smem_flag) {
  const int mw = static_cast<int>(warp_id()) - 1;
  const int lane = static_cast<int>(lane_id());
  const int q = lane >> 3, c = lane & 7;
  const int tid = mw * 32 + lane;
  int64_t it = 0;
  Seg s;
  for (int i = 0; seg_get(a, kMode, i, s); ++i) {
    float acc[4][NB];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int n = 0; n < NB; ++n) acc[p][n] = 0.f;

    for (int kb = s.kb0; kb < s.kb1; ++kb, ++it) {
      const int slot = static_cast<int>(it % a.stages);
      const uint32_t phase = static_cast<uint32_t>((it / a.stages) & 1);
      mbar_wait(&full[slot], phase);
      const uint8_t* st = smem + static_cast<int64_t>(slot) * stage_bytes;
      const uint8_t* xs = st + kBlockBytes;
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
      for (int p = 0; p < 4; ++p) {
        const int r = gemv_row(p, mw, q);
        const uint4 wv = *reinterpret_cast<const uint4*>(
            st + r * 128 + ((c ^ (r & 7)) << 4));
        float wf[8];
        wf[0] = bf16lo(wv.x); wf[1] = bf16hi(wv.x);
        wf[2] = bf16lo(wv.y); wf[3] = bf16hi(wv.y);
        wf[4] = bf16lo(wv.z); wf[5] = bf16hi(wv.z);
        wf[6] = bf16lo(wv.w); wf[7] = bf16hi(wv.w);
#pragma unroll
        for (int n = 0; n < NB; ++n)
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[p][n] = fmaf(wf[e], xf[n][e], acc[p][n]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }

    // Reduce the 8 K-chunks of every row.
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        float v = acc[p][n];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        acc[p][n] = v;
      }

    if constexpr (kMode == kModeStage1) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int col = s.tile * kS1Cols + p * 16 + 2 * mw + q;
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const float up = __shfl_xor_sync(0xffffffffu, acc[p][n], 16);
          if (c == 0 && q < 2 && n < a.B && col < a.cols_valid) {
            a.a2[n * a.a2_ld + col] =
                __float2bfloat16_rn(silu_f(acc[p][n]) * up);
          }
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int j = s.tile * kDownCols + gemv_row(p, mw, q);
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          if (c == 0 && n < a.B && j < a.out_cols) {
            atomicAdd(a.yacc + static_cast<int64_t>(n) * a.yacc_ld + j,
                      acc[p][n]);
          }
        }
      }
      down_finish_tile(a, s.tile, tid, kGemvWarps * 32, smem_flag);
    }
  }
}

// ---------------------------------------------------------------------------
// tcgen05 MMA issuer (one lane of warp 1).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_issue(const StreamArgs& a, int mode,
                                          uint8_t* smem, int stage_bytes,
                                          uint64_t* full, uint64_t* empty,
                                          uint64_t* tfull, uint64_t* tempty,
                                          uint32_t tmem_base) {
  const uint32_t idesc = umma_idesc_bf16(128, static_cast<uint32_t>(a.n_pad));
  int64_t it = 0;
  int acc_it = 0;
  Seg s;
  for (int i = 0; seg_get(a, mode, i, s); ++i, ++acc_it) {
    const int ab = acc_it & 1;
    const uint32_t aph = static_cast<uint32_t>((acc_it >> 1) & 1);
    mbar_wait(&tempty[ab], aph ^ 1u);
    tc_fence_after();
    const uint32_t d = tmem_base + static_cast<uint32_t>(ab * a.n_pad);
    for (int kb = s.kb0; kb < s.kb1; ++kb, ++it) {
      const int slot = static_cast<int>(it % a.stages);
      const uint32_t phase = static_cast<uint32_t>((it / a.stages) & 1);
      mbar_wait(&full[slot], phase);
      tc_fence_after();
      const uint32_t wbase =
          smem_u32(smem + static_cast<int64_t>(slot) * stage_bytes);
      const uint32_t xbase = wbase + kBlockBytes;
#pragma unroll
      for (int k = 0; k < kBlockK / 16; ++k) {
        tc_mma_bf16(d, umma_desc_sw128(wbase + k * 32),
                    umma_desc_sw128(xbase + k * 32), idesc,
                    (kb > s.kb0 || k > 0) ? 1u : 0u);
      }
      tc_commit(&empty[slot]);
    }
    tc_commit(&tfull[ab]);
  }
}

// ---------------------------------------------------------------------------
// tcgen05 epilogue (warps 2-5; TMEM lanes 32*(warp%4) .. +31).
// ---------------------------------------------------------------------------
template <int kMode>
__device__ __forceinline__ void tc_epilogue(const StreamArgs& a,
                                            uint64_t* tfull, uint64_t* tempty,
                                            uint32_t tmem_base,
                                            int* smem_flag) {
  const int w = static_cast<int>(warp_id());
  const int quarter = w & 3;
  const int lane = static_cast<int>(lane_id());
  const int row = quarter * 32 + lane;
  const int tid = (w - 2) * 32 + lane;
  int acc_it = 0;
  Seg s;
  for (int i = 0; seg_get(a, kMode, i, s); ++i, ++acc_it) {
    const int ab = acc_it & 1;
    const uint32_t aph = static_cast<uint32_t>((acc_it >> 1) & 1);
    mbar_wait(&tfull[ab], aph);
    tc_fence_after();
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                           static_cast<uint32_t>(ab * a.n_pad);
    if constexpr (kMode == kModeStage1) {
      int is_up, cofs;
      s1_row_map(row, &is_up, &cofs);
      const int col = s.tile * kS1Cols + cofs;
      for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float up = __shfl_xor_sync(0xffffffffu, v[e], 16);
          const int n = c0 + e;
          if (!is_up && n < a.B && col < a.cols_valid) {
            a.a2[n * a.a2_ld + col] = __float2bfloat16_rn(silu_f(v[e]) * up);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
    } else {
      const int j = s.tile * kDownCols + row;
      for (int c0 = 0; c0 < a.n_pad; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int n = c0 + e;
          if (n < a.B && j < a.out_cols) {
            atomicAdd(a.yacc + static_cast<int64_t>(n) * a.yacc_ld + j, v[e]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      down_finish_tile(a, s.tile, tid, 128, smem_flag);
    }
  }
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(p) + 1023) & ~static_cast<uintptr_t>(1023));
}

// ---------------------------------------------------------------------------
// The kernel.
// ---------------------------------------------------------------------------
template <int kMode, bool kTC, int NB>
__global__ void __launch_bounds__(kTC ? kTcThreads : kGemvThreads, 1)
    stream_kernel(const __grid_constant__ CUtensorMap xmap,
                  const StreamArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int stage_bytes = stream_stage_bytes(a.n_pad);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
  uint64_t* empty = full + a.stages;
  uint64_t* tfull = empty + a.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* smem_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t w = warp_id();
  if (w == 0 && lane_id() == 0) {
    prefetch_tmap(&xmap);
    for (int i = 0; i < a.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTC ? 1 : kGemvWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  uint32_t tmem_cols = 0;
  if constexpr (kTC) {
    tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(2 * a.n_pad)) tmem_cols <<= 1;
    if (w == 1) tmem_alloc(tmem_slot, tmem_cols);
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = kTC ? *tmem_slot : 0u;

  // Let the next kernel in the stream get scheduled as SMs drain; it only
  // touches our outputs after its own griddepcontrol.wait.
  pdl_launch_dependents();

  if (w == 0) {
    if (lane_id() == 0) produce(a, kMode, &xmap, smem, stage_bytes, full, empty);
  } else if constexpr (kTC) {
    if (w == 1) {
      if (lane_id() == 0)
        mma_issue(a, kMode, smem, stage_bytes, full, empty, tfull, tempty,
                  tmem_base);
    } else {
      tc_epilogue<kMode>(a, tfull, tempty, tmem_base, smem_flag);
    }
  } else {
    gemv_consume<kMode, NB>(a, smem, stage_bytes, full, empty, smem_flag);
  }

  __syncthreads();
  if constexpr (kTC) {
    if (w == 1) {
      __syncwarp();
      tc_fence_after();
      tmem_dealloc(tmem_base, tmem_cols);
    }
  }
}

template <int kMode, bool kTC, int NB>
cudaError_t launch_one(const CUtensorMap& xmap, const StreamArgs& a, int grid,
                       int smem, bool pdl, cudaStream_t stream) {
  auto kern = stream_kernel<kMode, kTC, NB>;
  static int configured_smem = -1;  // per instantiation; one device per process
  if (smem > configured_smem) {
    cudaError_t e = cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured_smem = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kTC ? kTcThreads : kGemvThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  int na = 0;
  if (pdl) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, xmap, a);
}

}  // namespace

int stream_smem_bytes(bool tc, int n_pad, int stages, int split_k) {
  (void)tc;
  (void)split_k;
  return 1024 + stages * stream_stage_bytes(n_pad) + (2 * stages + 4) * 8 + 16;
}

cudaError_t launch_stream(int mode, bool tc, int nb_gemv,
                          const CUtensorMap& xmap, const StreamArgs& a,
                          int grid, bool pdl, cudaStream_t stream) {
  const int smem = stream_smem_bytes(tc, a.n_pad, a.stages, a.split_k);
  if (tc) {
    return mode == kModeStage1
               ? launch_one<kModeStage1, true, 0>(xmap, a, grid, smem, pdl, stream)
               : launch_one<kModeDown, true, 0>(xmap, a, grid, smem, pdl, stream);
  }
#define DFK_GEMV_CASE(NBV)                                                    \
  case NBV:                                                                   \
    return mode == kModeStage1                                                \
               ? launch_one<kModeStage1, false, NBV>(xmap, a, grid, smem, pdl, \
                                                     stream)                  \
               : launch_one<kModeDown, false, NBV>(xmap, a, grid, smem, pdl,   \
                                                   stream);
  switch (nb_gemv) {
    DFK_GEMV_CASE(1)
    DFK_GEMV_CASE(2)
    DFK_GEMV_CASE(4)
    DFK_GEMV_CASE(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef DFK_GEMV_CASE
}

}  // namespace dfk
