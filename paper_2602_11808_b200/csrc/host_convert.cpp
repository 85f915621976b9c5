// host_convert.cpp — host-side element conversions of the reference-facing
// calls (dfk_forward_host, the C++ drop-in's Matrix in/out: the reference's
// operands are fp64, tensor.hpp:73-128).
//
// Converting B x d_model fp64 activations to bf16 (and the fp32 Y back to
// fp64) touches every host byte once.  The per-element rounding is
// branch-free RNE with NaN kept quiet -- identical to the device's
// __float2bfloat16_rn and to the oracle's quantisation -- so the loops
// vectorise; the branchy scalar version cost 0.65 ms of a 0.75 ms
// dfk_forward_host call at Llama-8B B = 64 (61 us kernel), this one about a
// third of that (profiles/r2_host_convert.md).  Splitting the loops over a
// worker pool was measured too: faster into a warm caller buffer, slower
// into the freshly zeroed Matrix the C++ drop-in returns (the lines live in
// the calling core's cache), so the calls stay on the caller's thread.
#include <cstdint>
#include <cstring>

#include "internal.h"

namespace dfk {
namespace {

inline uint16_t bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
  const bool nan = (u & 0x7FFFFFFFu) > 0x7F800000u;
  return static_cast<uint16_t>(nan ? ((u >> 16) | 0x40u) : r);
}

}  // namespace

void host_to_bf16(const void* src, int dtype, size_t n, uint16_t* dst) {
  if (dtype == DFK_BF16) {
    std::memcpy(dst, src, n * 2);
  } else if (dtype == DFK_F32) {
    const float* s = static_cast<const float*>(src);
    for (size_t i = 0; i < n; ++i) dst[i] = bf16_rne(s[i]);
  } else {
    const double* s = static_cast<const double*>(src);
    for (size_t i = 0; i < n; ++i) dst[i] = bf16_rne(static_cast<float>(s[i]));
  }
}

void host_from_f32(const float* src, size_t n, void* dst, int dtype) {
  if (dtype == DFK_F32) {
    std::memcpy(dst, src, n * 4);
  } else if (dtype == DFK_F64) {
    double* d = static_cast<double*>(dst);
    for (size_t i = 0; i < n; ++i) d[i] = src[i];
  } else {
    uint16_t* d = static_cast<uint16_t*>(dst);
    for (size_t i = 0; i < n; ++i) d[i] = bf16_rne(src[i]);
  }
}

void host_from_bf16(const uint16_t* src, size_t n, void* dst, int dtype) {
  auto widen = [](uint16_t v) {
    const uint32_t u = static_cast<uint32_t>(v) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  };
  if (dtype == DFK_BF16) {
    std::memcpy(dst, src, n * 2);
  } else if (dtype == DFK_F32) {
    float* d = static_cast<float*>(dst);
    for (size_t i = 0; i < n; ++i) d[i] = widen(src[i]);
  } else {
    double* d = static_cast<double*>(dst);
    for (size_t i = 0; i < n; ++i) d[i] = widen(src[i]);
  }
}

}  // namespace dfk

using namespace dfk;

extern "C" {

int dfk_host_to_bf16(const void* src, int32_t src_dtype, size_t n, uint16_t* dst) {
  if ((!src || !dst) && n) return fail(DFK_ERR_INVALID, "null host pointer");
  if (src_dtype != DFK_F64 && src_dtype != DFK_F32 && src_dtype != DFK_BF16)
    return fail(DFK_ERR_INVALID, "unknown source dtype");
  host_to_bf16(src, src_dtype, n, dst);
  return DFK_OK;
}

int dfk_host_from_f32(const float* src, size_t n, void* dst, int32_t dst_dtype) {
  if ((!src || !dst) && n) return fail(DFK_ERR_INVALID, "null host pointer");
  if (dst_dtype != DFK_F64 && dst_dtype != DFK_F32 && dst_dtype != DFK_BF16)
    return fail(DFK_ERR_INVALID, "unknown destination dtype");
  host_from_f32(src, n, dst, dst_dtype);
  return DFK_OK;
}

int dfk_host_from_bf16(const uint16_t* src, size_t n, void* dst, int32_t dst_dtype) {
  if ((!src || !dst) && n) return fail(DFK_ERR_INVALID, "null host pointer");
  if (dst_dtype != DFK_F64 && dst_dtype != DFK_F32 && dst_dtype != DFK_BF16)
    return fail(DFK_ERR_INVALID, "unknown destination dtype");
  host_from_bf16(src, n, dst, dst_dtype);
  return DFK_OK;
}

}  // extern "C"
