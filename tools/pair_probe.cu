// pair_probe.cu — does a 2-SM (cta_group::2) UMMA pair stream weights faster
// than single-SM CTAs in the block kernel's regime?  Standalone measurement
// aid (not product code): weights (M operand) and a batch operand (N rows)
// stream HBM -> SMEM by TMA into a ring; one lane issues tcgen05.mma into
// TMEM and commits each slot back; no epilogue.  352 MB of weights per
// launch, 40 PDL-chained launches, CUDA-event timed.
//
//   single: 1 CTA per SM, M=128, each CTA loads its 128 weight rows and all N
//           batch rows per 64-wide K block.
//   pair:   clusters of 2, M=256 (cta_group::2), each CTA loads its 128 weight
//           rows and N/2 batch rows; both CTAs' TMA bytes land on the leader's
//           full barrier (peer bit cleared), the leader issues the MMA and its
//           commit multicasts to both CTAs' empty barriers.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2602_11808_b200/csrc tools/pair_probe.cu -o tools/pair_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace dfk;

namespace {

constexpr int kThreads = 64;

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1,
                                     uint64_t* bar, bool pair) {
  if (pair) {
    const uint32_t b = smem_u32(bar) & 0xFEFFFFFFu;  // the leader's barrier
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
        "bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(b)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
  }
}

template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
    probe(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
          int tiles, int kblocks, int kbs, int stages, int n, unsigned* sink) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) &
                                             ~uintptr_t(1023));
  const int xrows = kPair ? n / 2 : n;
  const int stage_bytes = kbs * (16384 + xrows * 128);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + stages);
  const uint32_t rank = kPair ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  if (w == 1) {
    if (kPair)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n"
                   "tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::"r"(
                       smem_u32(tslot)),
                   "r"(256u)
                   : "memory");
    else
      tmem_alloc(tslot, 256u);
  }
  __syncthreads();
  if (kPair) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_launch_dependents();
  const int units = kPair ? gridDim.x / 2 : gridDim.x;  // work owners
  const int unit = kPair ? blockIdx.x / 2 : blockIdx.x;
  const int per = kPair ? 2 : 1;                         // tiles per unit step
  if (w == 0 && lane == 0) {
    int64_t it = 0;
    bool waited = false;
    for (int t = unit * per; t < tiles; t += units * per) {
      const int tile = t + static_cast<int>(rank);
      for (int kb = 0; kb < kblocks; kb += kbs, ++it) {
        const int slot = static_cast<int>(it % stages);
        const uint32_t ph = static_cast<uint32_t>((it / stages) & 1);
        if (it >= stages) mbar_wait(&empty[slot], ph ^ 1u);
        if (!waited && it >= stages) {
          pdl_wait();
          waited = true;
        }
        uint8_t* st = smem + static_cast<int64_t>(slot) * stage_bytes;
        const uint32_t own = static_cast<uint32_t>(kbs) * (16384u + xrows * 128u);
        if (leader) mbar_arrive_expect_tx(&full[slot], kPair ? 2 * own : own);
        for (int b = 0; b < kbs; b += 2) {  // 2 weight blocks (256 rows) per TMA
          const int rows = (tile * kblocks + kb + b) * 128;
          tma2d(st + b * 16384, &wmap, 0, rows, &full[slot], kPair);
        }
        for (int b = 0; b < kbs; ++b)
          tma2d(st + kbs * 16384 + b * xrows * 128, &xmap, (kb + b) * 64,
                static_cast<int>(rank) * xrows, &full[slot], kPair);
      }
    }
    if (!waited) pdl_wait();
  } else if (w == 1 && lane == 0 && leader) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                           ((static_cast<uint32_t>(n) >> 3) << 17) |
                           ((static_cast<uint32_t>(kPair ? 256 : 128) >> 4) << 24);
    int64_t it = 0;
    for (int t = unit * per; t < tiles; t += units * per) {
      for (int kb = 0; kb < kblocks; kb += kbs, ++it) {
        const int slot = static_cast<int>(it % stages);
        const uint32_t ph = static_cast<uint32_t>((it / stages) & 1);
        mbar_wait(&full[slot], ph);
        tc_fence_after();
        const uint32_t sb = smem_u32(smem + static_cast<int64_t>(slot) * stage_bytes);
        for (int b = 0; b < kbs; ++b)
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = umma_desc_sw128(sb + b * 16384 + k * 32);
            const uint64_t bd = umma_desc_sw128(sb + kbs * 16384 + b * xrows * 128 + k * 32);
            const uint32_t acc = (kb | b | k) ? 1u : 0u;
            if (kPair)
              asm volatile(
                  "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                  " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                  "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
                  : "memory");
            else
              tc_mma_bf16(tmem, ad, bd, idesc, acc);
          }
        if (kPair)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
              "cluster.b64 [%0], %1;" ::"r"(smem_u32(&empty[slot])),
              "h"(static_cast<uint16_t>(3))
              : "memory");
        else
          tc_commit(&empty[slot]);
      }
    }
  }
  __syncthreads();
  if (kPair) cluster_sync();
  if (w == 1) {
    tc_fence_after();
    if (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(256u)
                   : "memory");
    else
      tmem_dealloc(tmem, 256u);
  }
  if (threadIdx.x == 0 && tmem == 0xFFFFFFFFu) sink[0] = 1;
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

CUtensorMap make_map(void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                     uint32_t box_rows, bool swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box,
                         es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::printf("encode failed %d\n", static_cast<int>(r));
    std::exit(1);
  }
  return m;
}

}  // namespace

int main() {
  const int kblocks = 64;                 // d_model 4096
  const int tiles_per_launch = 336;       // 336 x 64 x 16 KiB = 352 MB
  const int nsets = 3;
  const size_t per_launch = size_t(tiles_per_launch) * kblocks * 16384;
  uint8_t* w;
  cudaMalloc(&w, per_launch * nsets);
  cudaMemset(w, 0, per_launch * nsets);
  uint16_t* x;
  cudaMalloc(&x, 256 * 4096 * 2);
  cudaMemset(x, 0, 256 * 4096 * 2);
  unsigned* sink;
  cudaMalloc(&sink, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int n : {16, 32, 64})
    for (int pair : {0, 1})
      for (int grid : {128, 146}) {
        const int xrows = pair ? n / 2 : n;
        const int kbs = 4;
        const int stage = kbs * (16384 + xrows * 128);
        const int stages = std::min(6, (227 * 1024 - 2048) / stage);
        const int smem = stages * stage + 1024 + 16 * stages + 64;
        CUtensorMap wm[nsets];
        for (int s = 0; s < nsets; ++s)
          wm[s] = make_map(w + s * per_launch, 64, uint64_t(tiles_per_launch) * kblocks * 128,
                           64, 256, false);
        CUtensorMap xm = make_map(x, 4096, 256, 64, xrows, true);
        auto launch = [&](int i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(grid);
          cfg.blockDim = dim3(kThreads);
          cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[2];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          at[1].id = cudaLaunchAttributeClusterDimension;
          at[1].val.clusterDim.x = pair ? 2 : 1;
          at[1].val.clusterDim.y = 1;
          at[1].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 2;
          if (pair)
            cudaLaunchKernelEx(&cfg, probe<true>, wm[i % nsets], xm, tiles_per_launch, kblocks,
                               kbs, stages, n, sink);
          else
            cudaLaunchKernelEx(&cfg, probe<false>, wm[i % nsets], xm, tiles_per_launch,
                               kblocks, kbs, stages, n, sink);
        };
        for (int i = 0; i < 6; ++i) launch(i);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          std::printf("n=%d pair=%d grid=%d: %s\n", n, pair, grid, cudaGetErrorString(e));
          return 1;
        }
        cudaEventRecord(a);
        for (int i = 0; i < 40; ++i) launch(i);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("N=%3d %-6s grid=%3d stages=%d : %7.2f us/launch  %7.1f GB/s\n", n,
                    pair ? "pair" : "single", grid, stages, ms * 1e3 / 40,
                    double(per_launch) * 40 / ms / 1e6);
      }
  return 0;
}
