// aux_kernels.cu — one-time weight prepack / unpack kernels and the small
// elementwise kernels of the unfused comparators (two-kernel: silu_mul,
// swiglu.cpp:205-211; four-kernel: silu, mul, swiglu.cpp:186-191).
// None of these is on the fused hot path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.h"
#include "layout.cuh"
#include "ptx.cuh"

namespace dfk {

namespace {

template <typename T>
__device__ __forceinline__ float ld_as_float(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ld_as_float<double>(const double* p,
                                                     int64_t i) {
  return static_cast<float>(p[i]);
}
template <>
__device__ __forceinline__ float ld_as_float<float>(const float* p, int64_t i) {
  return p[i];
}
template <>
__device__ __forceinline__ float ld_as_float<__nv_bfloat16>(
    const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

__device__ __forceinline__ int64_t gtid() {
  return static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
}

// One thread per (block, chunk, row): 8 bf16 of row r, K chunk c.  Threads
// of a warp take consecutive rows so source reads along d_ff coalesce.
// fp64 sources are rounded to fp32 (RNE) and then to bf16 (RNE), the same
// two-step rounding as the oracle's dfo_quantize_bf16.
template <typename T>
__global__ void pack_stage1_kernel(const T* __restrict__ wg,
                                   const T* __restrict__ wu, int64_t dm,
                                   int64_t df_total, int64_t ff_begin,
                                   int64_t df, int kblocks, int64_t total,
                                   uint8_t* __restrict__ dst) {
  for (int64_t idx = gtid(); idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx & 127);
    const int c = static_cast<int>((idx >> 7) & 7);
    const int64_t blk = idx >> 10;
    const int t = static_cast<int>(blk / kblocks);
    const int kb = static_cast<int>(blk % kblocks);
    int is_up, cofs;
    s1_row_map(r, &is_up, &cofs);
    const int64_t col = static_cast<int64_t>(t) * kS1Cols + cofs;
    const T* src = is_up ? wu : wg;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t k = static_cast<int64_t>(kb) * kBlockK + c * 8 + e;
      float f = 0.f;
      if (k < dm && col < df) f = ld_as_float(src, k * df_total + ff_begin + col);
      v[e] = __float2bfloat16_rn(f);
    }
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(
        dst + blk * static_cast<int64_t>(kBlockBytes));
    *reinterpret_cast<uint4*>(out + block_elem_offset(r, c * 8)) =
        *reinterpret_cast<const uint4*>(v);
  }
}

template <typename T>
__global__ void pack_down_kernel(const T* __restrict__ wd, int64_t dm,
                                 int64_t ff_begin, int64_t df, int kblocks,
                                 int64_t total, uint8_t* __restrict__ dst) {
  for (int64_t idx = gtid(); idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx & 127);
    const int c = static_cast<int>((idx >> 7) & 7);
    const int64_t blk = idx >> 10;
    const int t = static_cast<int>(blk / kblocks);
    const int kb = static_cast<int>(blk % kblocks);
    const int64_t j = static_cast<int64_t>(t) * kDownCols + r;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t f = static_cast<int64_t>(kb) * kBlockK + c * 8 + e;
      float x = 0.f;
      if (f < df && j < dm) x = ld_as_float(wd, (ff_begin + f) * dm + j);
      v[e] = __float2bfloat16_rn(x);
    }
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(
        dst + blk * static_cast<int64_t>(kBlockBytes));
    *reinterpret_cast<uint4*>(out + block_elem_offset(r, c * 8)) =
        *reinterpret_cast<const uint4*>(v);
  }
}

// Pack -> K-major W_cat^T [2 df x dm] (rows 0..df-1 gate, df..2df-1 up).
__global__ void unpack_stage1_kernel(const uint8_t* __restrict__ pack,
                                     int64_t dm, int64_t df, int kblocks,
                                     int64_t total,
                                     __nv_bfloat16* __restrict__ cat_t) {
  for (int64_t idx = gtid(); idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = idx % dm;
    const int64_t row = idx / dm;  // 0 .. 2df-1
    const int is_up = row >= df ? 1 : 0;
    const int64_t col = is_up ? row - df : row;
    const int t = static_cast<int>(col / kS1Cols);
    const int cin = static_cast<int>(col % kS1Cols);
    const int r = (cin / 16) * 32 + is_up * 16 + (cin % 16);
    const int kb = static_cast<int>(k / kBlockK);
    const __nv_bfloat16* blk = reinterpret_cast<const __nv_bfloat16*>(
        pack + (static_cast<int64_t>(t) * kblocks + kb) * kBlockBytes);
    cat_t[idx] = blk[block_elem_offset(r, static_cast<int>(k % kBlockK))];
  }
}

// Pack -> K-major W_down^T [dm x df].
__global__ void unpack_down_kernel(const uint8_t* __restrict__ pack,
                                   int64_t dm, int64_t df, int kblocks,
                                   int64_t total,
                                   __nv_bfloat16* __restrict__ down_t) {
  for (int64_t idx = gtid(); idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t f = idx % df;
    const int64_t j = idx / df;
    const int t = static_cast<int>(j / kDownCols);
    const int r = static_cast<int>(j % kDownCols);
    const int kb = static_cast<int>(f / kBlockK);
    const __nv_bfloat16* blk = reinterpret_cast<const __nv_bfloat16*>(
        pack + (static_cast<int64_t>(t) * kblocks + kb) * kBlockBytes);
    down_t[idx] = blk[block_elem_offset(r, static_cast<int>(f % kBlockK))];
  }
}

__global__ void pad_rows_kernel(const __nv_bfloat16* __restrict__ src,
                                int64_t rows, int64_t cols, int64_t ld_src,
                                __nv_bfloat16* __restrict__ dst,
                                int64_t ld_dst) {
  const int64_t total = rows * ld_dst;
  for (int64_t idx = gtid(); idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / ld_dst, c = idx % ld_dst;
    dst[idx] = c < cols ? src[r * ld_src + c] : __float2bfloat16_rn(0.f);
  }
}

__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gate,
                                int64_t ld_gate,
                                const __nv_bfloat16* __restrict__ up,
                                int64_t ld_up, __nv_bfloat16* __restrict__ out,
                                int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = gtid(); idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / cols, c = idx % cols;
    const float g = __bfloat162float(gate[r * ld_gate + c]);
    const float u = __bfloat162float(up[r * ld_up + c]);
    out[idx] = __float2bfloat16_rn(silu_f(g) * u);
  }
}

__global__ void silu_kernel(const __nv_bfloat16* __restrict__ in,
                            __nv_bfloat16* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    out[i] = __float2bfloat16_rn(silu_f(__bfloat162float(in[i])));
  }
}

__global__ void mul_kernel(const __nv_bfloat16* __restrict__ a,
                           const __nv_bfloat16* __restrict__ b,
                           __nv_bfloat16* __restrict__ out, int64_t n) {
  for (int64_t i = gtid(); i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    out[i] = __float2bfloat16_rn(__bfloat162float(a[i]) *
                                 __bfloat162float(b[i]));
  }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

__global__ void fill_uniform_kernel(__nv_bfloat16* __restrict__ p, int64_t n,
                                    uint64_t seed, float lo, float hi) {
  for (int64_t i = gtid(); i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = splitmix64(seed ^ splitmix64(static_cast<uint64_t>(i)));
    const float u = static_cast<float>(h >> 40) * (1.0f / 16777216.0f);
    p[i] = __float2bfloat16_rn(lo + u * (hi - lo));
  }
}

__global__ void flush_kernel(uint4* __restrict__ p, int64_t n) {
  for (int64_t i = gtid(); i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    p[i] = make_uint4(static_cast<uint32_t>(i), 1u, 2u, 3u);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in,
                                   __nv_bfloat16* __restrict__ out,
                                   int64_t n) {
  for (int64_t i = gtid(); i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    out[i] = __float2bfloat16_rn(in[i]);
  }
}

// Host-buffer path: copies X (bf16, 16-byte units) from mapped pinned host
// memory into a device staging slot, then joins the programmatic-dependent
// chain: it lets the next block kernel pre-launch immediately and waits for
// the previous kernel only AFTER its copy -- so the PCIe read of call i+1's
// X overlaps call i's block.
__global__ void stage_rows_kernel(const uint4* __restrict__ src,
                                  uint4* __restrict__ dst, int64_t n16) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t i = gtid(); i < n16; i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

unsigned grid_for(int64_t total, int threads) {
  int64_t g = (total + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<unsigned>(g);
}

}  // namespace

// Force-load every kernel of this translation unit (CUDA lazy loading would
// otherwise load a module at its first launch, which can wait for the
// device -- fatal between the launches of ranks that wait for each other).
cudaError_t preload_aux_kernels() {
  const void* fns[] = {
      reinterpret_cast<const void*>(pack_stage1_kernel<double>),
      reinterpret_cast<const void*>(pack_stage1_kernel<float>),
      reinterpret_cast<const void*>(pack_stage1_kernel<__nv_bfloat16>),
      reinterpret_cast<const void*>(pack_down_kernel<double>),
      reinterpret_cast<const void*>(pack_down_kernel<float>),
      reinterpret_cast<const void*>(pack_down_kernel<__nv_bfloat16>),
      reinterpret_cast<const void*>(unpack_stage1_kernel),
      reinterpret_cast<const void*>(unpack_down_kernel),
      reinterpret_cast<const void*>(pad_rows_kernel),
      reinterpret_cast<const void*>(silu_mul_kernel),
      reinterpret_cast<const void*>(silu_kernel),
      reinterpret_cast<const void*>(mul_kernel),
      reinterpret_cast<const void*>(fill_uniform_kernel),
      reinterpret_cast<const void*>(flush_kernel),
      reinterpret_cast<const void*>(f32_to_bf16_kernel),
      reinterpret_cast<const void*>(stage_rows_kernel)};
  for (const void* f : fns) {
    cudaFuncAttributes at;
    const cudaError_t e = cudaFuncGetAttributes(&at, f);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_pack_stage1(const void* w_gate, const void* w_up, int dtype,
                               int64_t d_model, int64_t d_ff_total,
                               int64_t ff_begin, int64_t d_ff, int tiles,
                               int kblocks, uint8_t* dst, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(tiles) * kblocks * 1024;
  const unsigned g = grid_for(total, 256);
  switch (dtype) {
    case DFK_F64:
      pack_stage1_kernel<double><<<g, 256, 0, s>>>(
          static_cast<const double*>(w_gate), static_cast<const double*>(w_up),
          d_model, d_ff_total, ff_begin, d_ff, kblocks, total, dst);
      break;
    case DFK_F32:
      pack_stage1_kernel<float><<<g, 256, 0, s>>>(
          static_cast<const float*>(w_gate), static_cast<const float*>(w_up),
          d_model, d_ff_total, ff_begin, d_ff, kblocks, total, dst);
      break;
    default:
      pack_stage1_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(
          static_cast<const __nv_bfloat16*>(w_gate),
          static_cast<const __nv_bfloat16*>(w_up), d_model, d_ff_total,
          ff_begin, d_ff, kblocks, total, dst);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_down(const void* w_down, int dtype, int64_t d_model,
                             int64_t ff_begin, int64_t d_ff, int tiles,
                             int kblocks, uint8_t* dst, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(tiles) * kblocks * 1024;
  const unsigned g = grid_for(total, 256);
  switch (dtype) {
    case DFK_F64:
      pack_down_kernel<double><<<g, 256, 0, s>>>(
          static_cast<const double*>(w_down), d_model, ff_begin, d_ff, kblocks,
          total, dst);
      break;
    case DFK_F32:
      pack_down_kernel<float><<<g, 256, 0, s>>>(
          static_cast<const float*>(w_down), d_model, ff_begin, d_ff, kblocks,
          total, dst);
      break;
    default:
      pack_down_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(
          static_cast<const __nv_bfloat16*>(w_down), d_model, ff_begin, d_ff,
          kblocks, total, dst);
  }
  return cudaGetLastError();
}

cudaError_t launch_unpack_stage1(const uint8_t* pack, int64_t d_model,
                                 int64_t d_ff, int tiles, int kblocks,
                                 __nv_bfloat16* cat_t, cudaStream_t s) {
  (void)tiles;
  const int64_t total = 2 * d_ff * d_model;
  unpack_stage1_kernel<<<grid_for(total, 256), 256, 0, s>>>(
      pack, d_model, d_ff, kblocks, total, cat_t);
  return cudaGetLastError();
}

cudaError_t launch_unpack_down(const uint8_t* pack, int64_t d_model,
                               int64_t d_ff, int tiles, int kblocks,
                               __nv_bfloat16* down_t, cudaStream_t s) {
  (void)tiles;
  const int64_t total = d_model * d_ff;
  unpack_down_kernel<<<grid_for(total, 256), 256, 0, s>>>(
      pack, d_model, d_ff, kblocks, total, down_t);
  return cudaGetLastError();
}

cudaError_t launch_pad_rows(const __nv_bfloat16* src, int64_t rows,
                            int64_t cols, int64_t ld_src, __nv_bfloat16* dst,
                            int64_t ld_dst, cudaStream_t s) {
  pad_rows_kernel<<<grid_for(rows * ld_dst, 256), 256, 0, s>>>(
      src, rows, cols, ld_src, dst, ld_dst);
  return cudaGetLastError();
}

cudaError_t launch_silu_mul(const __nv_bfloat16* gate, int64_t ld_gate,
                            const __nv_bfloat16* up, int64_t ld_up,
                            __nv_bfloat16* out, int64_t rows, int64_t cols,
                            cudaStream_t s) {
  silu_mul_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(
      gate, ld_gate, up, ld_up, out, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_silu(const __nv_bfloat16* in, __nv_bfloat16* out,
                        int64_t n, cudaStream_t s) {
  silu_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t launch_mul(const __nv_bfloat16* a, const __nv_bfloat16* b,
                       __nv_bfloat16* out, int64_t n, cudaStream_t s) {
  mul_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, b, out, n);
  return cudaGetLastError();
}

cudaError_t launch_fill_uniform_bf16(__nv_bfloat16* p, int64_t n,
                                     uint64_t seed, float lo, float hi,
                                     cudaStream_t s) {
  fill_uniform_kernel<<<grid_for(n, 256), 256, 0, s>>>(p, n, seed, lo, hi);
  return cudaGetLastError();
}

cudaError_t launch_flush(void* p, size_t bytes, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(bytes / 16);
  flush_kernel<<<grid_for(n, 256), 256, 0, s>>>(static_cast<uint4*>(p), n);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_bf16(const float* in, __nv_bfloat16* out, int64_t n,
                               cudaStream_t s) {
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t launch_stage_rows(const void* src, void* dst, int64_t bytes,
                              cudaStream_t s) {
  const int64_t n16 = bytes / 16;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(16, (n16 + 255) / 256 + 1)));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, stage_rows_kernel, static_cast<const uint4*>(src),
                            static_cast<uint4*>(dst), n16);
}

}  // namespace dfk
