// stream_probe.cu — microbenchmark of HBM->SMEM streaming on B200, used to
// size the weight-streaming pipeline (chunk size, ring depth, CTAs per SM).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2602_11808_b200/csrc tools/stream_probe.cu -o tools/stream_probe
//
// Variants:
//   bulk  : one producer lane issues cp.async.bulk of `chunk` bytes into a ring
//           of `stages` slots; a consumer lane releases each slot on arrival.
//   ldg   : every thread streams 16-byte ld.global.nc.L1::no_allocate loads
//           (unroll 8) and XOR-reduces them (the plain-LDG ceiling).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "ptx.cuh"

using namespace dfk;

__global__ void __launch_bounds__(64, 1)
    bulk_stream(const uint8_t* __restrict__ src, size_t per_cta, int chunk,
                int stages, unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(stages) * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * per_cta;
  const long n = static_cast<long>(per_cta / chunk);
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0) {
    for (long it = 0; it < n; ++it) {
      const int s = static_cast<int>(it % stages);
      const uint32_t ph = static_cast<uint32_t>((it / stages) & 1);
      if (it >= stages) mbar_wait(&empty[s], ph ^ 1u);
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_g2s(smem + size_t(s) * chunk, base + it * chunk, chunk, &full[s], pol);
    }
  } else if (threadIdx.x == 32) {
    unsigned acc = 0;
    for (long it = 0; it < n; ++it) {
      const int s = static_cast<int>(it % stages);
      const uint32_t ph = static_cast<uint32_t>((it / stages) & 1);
      mbar_wait(&full[s], ph);
      acc ^= *reinterpret_cast<volatile unsigned*>(smem + size_t(s) * chunk);
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) sink[blockIdx.x] = acc;
  }
}

// Same as bulk_stream, but PDL-chained: the first ring is issued before
// griddepcontrol.wait (as the block kernel does), dependents launch at once.
__global__ void __launch_bounds__(64, 1)
    bulk_stream_pdl(const uint8_t* __restrict__ src, size_t per_cta, int chunk,
                    int stages, unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(stages) * chunk);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_launch_dependents();
  const uint8_t* base = src + blockIdx.x * per_cta;
  const long n = static_cast<long>(per_cta / chunk);
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0) {
    for (long it = 0; it < n; ++it) {
      const int s = static_cast<int>(it % stages);
      const uint32_t ph = static_cast<uint32_t>((it / stages) & 1);
      if (it == stages) pdl_wait();
      if (it >= stages) mbar_wait(&empty[s], ph ^ 1u);
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_g2s(smem + size_t(s) * chunk, base + it * chunk, chunk, &full[s], pol);
    }
    if (n <= stages) pdl_wait();
  } else if (threadIdx.x == 32) {
    unsigned acc = 0;
    for (long it = 0; it < n; ++it) {
      const int s = static_cast<int>(it % stages);
      const uint32_t ph = static_cast<uint32_t>((it / stages) & 1);
      mbar_wait(&full[s], ph);
      acc ^= *reinterpret_cast<volatile unsigned*>(smem + size_t(s) * chunk);
      mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) sink[blockIdx.x] = acc;
  }
}

__global__ void __launch_bounds__(512) ldg_stream(const uint4* __restrict__ src,
                                                   size_t n16, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(src + i + u * stride));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char** argv) {
  const size_t total = size_t(1) << 30;  // 1 GiB >> L2
  const bool launch_mode = argc > 1 && std::string(argv[1]) == "launch";
  uint8_t* buf;
  unsigned* sink;
  cudaMalloc(&buf, total + (64 << 20));
  cudaMalloc(&sink, 1 << 20);
  cudaMemset(buf, 1, total);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time_it = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    return best;
  };
  if (launch_mode) {
    // Per-launch cost of a 352 MB stream (the Llama-8B block's bytes) over
    // rotating quarter-GiB windows, 40 back-to-back launches, with and
    // without PDL: the floor for a single-launch block of this size.
    cudaFuncSetAttribute(bulk_stream_pdl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    // optional per-launch sizes in MB after "launch" (default: 352 MB)
    std::vector<size_t> sizes;
    for (int i = 2; i < argc; ++i) sizes.push_back(size_t(atof(argv[i]) * 1e6) / 65536 * 65536);
    if (sizes.empty()) sizes.push_back(352321536);
    for (size_t per_launch : sizes)
    for (int pdl : {0, 1})
      for (int grid : {129, 148})
        for (int chunk : {32768, 65536}) {
          const int stages = chunk == 65536 ? 3 : 6;
          const size_t per_cta = per_launch / grid / chunk * chunk;
          const int smem = stages * chunk + 1024 + 16 * stages + 64;
          auto one = [&](int i) {
            const uint8_t* src = buf + (size_t(i % 3) * (size_t(1) << 28));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(64);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at;
            at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at.val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = &at;
            cfg.numAttrs = pdl;
            cudaLaunchKernelEx(&cfg, bulk_stream_pdl, src, per_cta, chunk, stages, sink);
          };
          float ms = time_it([&] { for (int i = 0; i < 40; ++i) one(i); });
          printf("launch %6.1fMB pdl=%d grid=%3d chunk=%6d stages=%d : %7.2f us/launch  %7.1f GB/s\n",
                 per_launch / 1e6, pdl, grid, chunk, stages, ms * 1e3 / 40,
                 double(per_cta) * grid * 40 / ms / 1e6);
        }
    return 0;
  }
  {
    const size_t n16 = total / 16;
    for (int blocks_per_sm : {1, 2, 4}) {
      const int grid = sms * blocks_per_sm;
      float ms = time_it([&] { ldg_stream<<<grid, 512>>>((const uint4*)buf, n16, sink); });
      printf("ldg   grid=%4d x512           : %7.1f GB/s\n", grid, total / ms / 1e6);
    }
  }
  struct Cfg { int chunk, stages, ctas_per_sm, grid_sms; };
  std::vector<Cfg> cfgs;
  for (int chunk : {8192, 16384, 32768, 65536})
    for (int inflight_kb : {32, 64, 96, 128, 192})
      for (int cps : {1, 2}) {
        const int stages = inflight_kb * 1024 / chunk / cps;
        if (stages < 2) continue;
        if (size_t(stages) * chunk * cps > 220 * 1024) continue;
        cfgs.push_back({chunk, stages, cps, sms});
      }
  // Partial-occupancy runs: how fast can a subset of SMs stream?
  for (int g : {76, 112}) cfgs.push_back({16384, 12, 1, g});
  for (int g : {76, 112}) cfgs.push_back({32768, 6, 1, g});
  for (const Cfg& c : cfgs) {
    const int grid = c.grid_sms * c.ctas_per_sm;
    size_t per_cta = (total / grid) / c.chunk * c.chunk;
    const int smem = c.stages * c.chunk + 1024 + 16 * c.stages + 64;
    float ms = time_it([&] {
      bulk_stream<<<grid, 64, smem>>>(buf, per_cta, c.chunk, c.stages, sink);
    });
    cudaError_t e = cudaGetLastError();
    printf("bulk  chunk=%6d stages=%2d ctas/sm=%d grid=%4d inflight/SM=%4dKB : %7.1f GB/s %s\n",
           c.chunk, c.stages, c.ctas_per_sm, grid, c.chunk * c.stages * c.ctas_per_sm / 1024,
           per_cta * grid / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
