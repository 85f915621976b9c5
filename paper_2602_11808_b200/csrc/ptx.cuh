// ptx.cuh — thin inline-PTX wrappers for the sm_100a features the
// weight-streaming kernels use: mbarriers, 1-D bulk copies and 2-D TMA
// (cp.async.bulk[.tensor]), tcgen05 MMA / TMEM, PDL (griddepcontrol) and
// cluster DSMEM.  Written for sm_100a only; there is no fallback path.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

namespace dfk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Warp-uniform warp index (broadcast from lane 0 so the compiler treats the
// role dispatch as uniform).
__device__ __forceinline__ uint32_t warp_id() {
  return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
}

// ----------------------------------------------------------------------------
// mbarrier
// ----------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
}

// Makes mbarrier.init visible to the async proxy and to the other CTAs of the
// cluster.
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar,
                                                      uint32_t bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], "
      "%1;\n}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// Remote arrive on the mbarrier at the same smem offset in CTA `cta_rank` of
// this cluster (release at cluster scope: prior DSMEM stores are visible to a
// waiter that acquires the phase).
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar,
                                                    uint32_t cta_rank) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(
          smem_u32(bar)),
      "r"(cta_rank)
      : "memory");
}

__device__ __forceinline__ uint32_t mbar_try_wait(uint64_t* bar,
                                                  uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], "
      "%2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Cluster-scope acquire variant (for barriers armed by remote CTAs).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar,
                                                  uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::"
        "cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// ----------------------------------------------------------------------------
// L2 cache policies and bulk copies (global -> shared, completion counted on
// an mbarrier in bytes).
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;"
               : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;"
               : "=l"(p));
  return p;
}

// 1-D bulk copy of `bytes` (multiple of 16, 16-byte aligned both sides).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc,
                                         uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::"
      "cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// 2-D TMA tile load: box at (c0 = innermost coordinate, c1 = row).
__device__ __forceinline__ void tma_load_2d(void* smem_dst,
                                            const CUtensorMap* map,
                                            int32_t c0, int32_t c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_"
      "tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
      "r"(smem_u32(bar))
      : "memory");
}

// 3-D TMA tile load: box at (c0, c1, c2) (c0 innermost).
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map,
                                            int32_t c0, int32_t c1, int32_t c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_"
      "tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(
                   reinterpret_cast<uint64_t>(map))
               : "memory");
}

// ----------------------------------------------------------------------------
// Programmatic dependent launch.
// ----------------------------------------------------------------------------
// 2-D TMA store shared::cta -> global (bulk group), its commit and waits.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem_src,
                                             int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Generic-proxy shared-memory writes become visible to the async proxy (TMA).
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Bulk prefetch of global memory into L2 (no shared memory, no barrier).
__device__ __forceinline__ void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gsrc), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ----------------------------------------------------------------------------
// Clusters / DSMEM.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n"
      "barrier.cluster.wait.acquire.aligned;" ::
          : "memory");
}

// Store a float4 into CTA `rank`'s shared memory at the address that `p`
// has in this CTA.
__device__ __forceinline__ void st_dsmem_f4(const void* p, uint32_t rank,
                                            float4 v) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " st.shared::cluster.v4.f32 [ra], {%2, %3, %4, %5};\n}" ::"r"(
          smem_u32(p)),
      "r"(rank), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
      : "memory");
}

// Store one float into CTA `rank`'s shared memory (DSMEM).
__device__ __forceinline__ void st_dsmem_f32(const float* p, uint32_t rank,
                                             float v) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " st.shared::cluster.f32 [ra], %2;\n}" ::"r"(smem_u32(p)),
      "r"(rank), "f"(v)
      : "memory");
}

// Asynchronous 16-byte DSMEM store into CTA `rank` whose completion is
// counted (in bytes) on that CTA's mbarrier `bar` (same smem offset).
__device__ __forceinline__ void st_async_f4(const void* p, uint64_t* bar,
                                            uint32_t rank, float x, float y,
                                            float z, float w) {
  asm volatile(
      "{\n .reg .b32 ra, rb;\n mapa.shared::cluster.u32 ra, %0, %6;\n"
      " mapa.shared::cluster.u32 rb, %1, %6;\n"
      " st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [ra], "
      "{%2, %3, %4, %5}, [rb];\n}" ::"r"(smem_u32(p)),
      "r"(smem_u32(bar)), "f"(x), "f"(y), "f"(z), "f"(w), "r"(rank)
      : "memory");
}

__device__ __forceinline__ float4 ld_shared_f4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// Atomic add into CTA `rank`'s shared memory (DSMEM) at the address `p`
// has in this CTA.
__device__ __forceinline__ void red_add_dsmem(const float* p, uint32_t rank,
                                              float v) {
  asm volatile(
      "{\n .reg .b32 ra;\n mapa.shared::cluster.u32 ra, %0, %1;\n"
      " red.shared::cluster.add.f32 [ra], %2;\n}" ::"r"(smem_u32(p)),
      "r"(rank), "f"(v)
      : "memory");
}

// ----------------------------------------------------------------------------
// tcgen05 / TMEM.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile(
      "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
          smem_u32(smem_dst)),
      "r"(ncols)
      : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
                   taddr),
               "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate.
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc,
                                            uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(
          d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrives (once) on `bar` when every previously issued tcgen05.mma of this
// thread has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 "
      "[%0];" ::"r"(smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns: thread t of the warp receives
// TMEM lane (base lane + t), columns [col, col+16).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, "
      "%7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]),
        "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
        "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Sum of `nacc` accumulators `stride` TMEM columns apart (the independent
// MMA chains of one tile), 16 columns from taddr.
__device__ __forceinline__ void tmem_ld16_sum(uint32_t taddr, int nacc, uint32_t stride,
                                              float (&v)[16]) {
  tmem_ld16(taddr, v);
  for (int j = 1; j < nacc; ++j) {
    float t[16];
    tmem_ld16(taddr + static_cast<uint32_t>(j) * stride, t);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] += t[i];
  }
}

// UMMA shared-memory descriptor for a K-major, 128B-swizzled operand whose
// 8-row groups are 1024 B apart (rows 128 B = 64 bf16 of K).
// Fields (sm100): start>>4 [0,14), LBO>>4 [16,30) (unused for SW128 K-major,
// 1), SBO>>4 [32,46) = 64, version [46,48) = 1, layout [61,64) = 2
// (SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// Instruction descriptor, kind::f16: bf16 A/B, fp32 D, both K-major.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(uint32_t M,
                                                       uint32_t N) {
  return (1u << 4)            // D format: F32
         | (1u << 7)          // A format: BF16
         | (1u << 10)         // B format: BF16
         | ((N >> 3) << 17)   // N >> 3
         | ((M >> 4) << 24);  // M >> 4
}

// ----------------------------------------------------------------------------
// Numerics helpers.
// ----------------------------------------------------------------------------
__device__ __forceinline__ float bf16lo(uint32_t u) {
  return __uint_as_float(u << 16);
}
__device__ __forceinline__ float bf16hi(uint32_t u) {
  return __uint_as_float(u & 0xFFFF0000u);
}

// silu(g) = g * sigmoid(g) (tensor.hpp:155-163) with the MUFU approximations (ex2.approx,
// rcp.approx; ~2 ulp fp32, far below the bf16 rounding of A2).  Stable for
// |g| >> 1: exp(-g) saturates to +inf, rcp(inf) = 0, so large negative g
// gives -0, never NaN.  Five instructions and no branch: the epilogue that
// runs it executes once per tile from a cold instruction cache, and
// __frcp_rn's refinement + slow-path branch tripled its code (and its
// instruction-fetch stalls, profiles/r1c_epilogue.md).
// red.global.add.f32 under a predicate (no branch around it).
__device__ __forceinline__ void red_add_f32_if(float* addr, float v, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p red.global.add.f32 [%0], %1;\n}" ::"l"(addr),
      "f"(v), "r"(static_cast<int>(pred))
      : "memory");
}

// red.global.add.v4.f32 (16-byte aligned) under a predicate.
__device__ __forceinline__ void red_add_v4_f32_if(float* addr, float a, float b, float c,
                                                  float d, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n"
      " @p red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n}" ::"l"(addr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(static_cast<int>(pred))
      : "memory");
}

// System-scope forms for partial sums added into another GPU's memory
// (fused TP all-reduce): every rank's reductions to one address must be
// atomic with respect to each other, i.e. at .sys scope.
__device__ __forceinline__ void red_add_sys_f32_if(float* addr, float v, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p red.relaxed.sys.global.add.f32 [%0], %1;\n}"
      ::"l"(addr), "f"(v), "r"(static_cast<int>(pred))
      : "memory");
}

__device__ __forceinline__ void red_add_sys_v4_f32_if(float* addr, float a, float b, float c,
                                                      float d, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n"
      " @p red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n}" ::"l"(addr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(static_cast<int>(pred))
      : "memory");
}

__device__ __forceinline__ void st_shared_u16(uint32_t addr, unsigned short v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float silu_f(float g) {
  return g * rcp_approx(1.0f + __expf(-g));
}

__device__ __forceinline__ float ld_shared_f32(const float* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
  return v;
}

}  // namespace dfk
