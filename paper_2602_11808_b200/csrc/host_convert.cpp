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
// the calling core's cache), so B x d_model sized calls stay on the caller's
// thread.  Only rounding to bf16 of >= kParallelMin elements (into our own
// staging buffer: X at B >= 32, the B x d_ff A2 the drop-in's down_projection
// receives) is split over a small persistent pool.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

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

constexpr size_t kParallelMin = size_t{1} << 17;  // elements
constexpr size_t kChunk = size_t{1} << 16;

// A job lives on the caller's stack: [0, n) split into kChunk pieces taken
// with an atomic cursor by the workers and the caller alike.  Workers pick
// the job up under the lock (counted in `active`) and the caller returns only
// when every piece is done and no worker still holds the job.  One job at a
// time: a caller that finds the pool busy converts serially.
class Pool {
 public:
  static Pool& get() {
    static Pool* p = new Pool();  // never destroyed: no join race at exit
    return *p;
  }
  bool run(size_t n, const std::function<void(size_t, size_t)>& fn) {
    std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
    if (!busy.owns_lock() || workers_ == 0) return false;
    Job job{&fn, n, (n + kChunk - 1) / kChunk};
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      ++gen_;
    }
    cv_.notify_all();
    job.work();
    while (job.done.load(std::memory_order_acquire) < job.chunks) std::this_thread::yield();
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = nullptr;  // no new worker picks it up
    }
    while (active_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
    return true;
  }

 private:
  struct Job {
    const std::function<void(size_t, size_t)>* fn;
    size_t n, chunks;
    std::atomic<size_t> next{0}, done{0};
    Job(const std::function<void(size_t, size_t)>* f, size_t n_, size_t c)
        : fn(f), n(n_), chunks(c) {}
    void work() {
      for (size_t c; (c = next.fetch_add(1)) < chunks;) {
        (*fn)(c * kChunk, std::min(n, (c + 1) * kChunk));
        done.fetch_add(1, std::memory_order_release);
      }
    }
  };
  Pool() {
    const unsigned hw = std::thread::hardware_concurrency();
    workers_ = std::min(7u, hw > 2 ? hw / 2 - 1 : 0u);
    for (unsigned i = 0; i < workers_; ++i) std::thread([this] { loop(); }).detach();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      Job* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        job = job_;
        if (!job) continue;
        active_.fetch_add(1, std::memory_order_relaxed);
      }
      job->work();
      active_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::mutex busy_, mu_;
  std::condition_variable cv_;
  Job* job_ = nullptr;
  uint64_t gen_ = 0;
  std::atomic<int> active_{0};
  unsigned workers_ = 0;
};

// The element loops over [lo, hi), kept as plain functions on restrict
// pointers so that they vectorise (the inline path of small calls runs them
// directly, the pool through a std::function per chunk).
void f64_to_bf16(const double* __restrict s, uint16_t* __restrict d, size_t lo, size_t hi) {
  for (size_t i = lo; i < hi; ++i) d[i] = bf16_rne(static_cast<float>(s[i]));
}
void f32_to_bf16(const float* __restrict s, uint16_t* __restrict d, size_t lo, size_t hi) {
  for (size_t i = lo; i < hi; ++i) d[i] = bf16_rne(s[i]);
}
inline float widen(uint16_t v) {
  const uint32_t u = static_cast<uint32_t>(v) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

}  // namespace

// Rounding into bf16 (our own staging buffer, fp64 / fp32 input of any
// size): inputs of >= 128 K elements on the pool -- the drop-in's
// down_projection A2 at B = 64 (917 K elements) 750 -> 620 us,
// dfk_forward_host's X at B = 32 / 64: 227 -> 190 / 361 -> 339 us per call.  Widening into the caller's fp64
// Matrix stays on the calling thread: the pool was slower there (B = 64
// run_fused_stage1 517 -> 620 us; the destination lines are the caller's).
void host_to_bf16(const void* src, int dtype, size_t n, uint16_t* dst) {
  if (dtype == DFK_BF16) {
    std::memcpy(dst, src, n * 2);
  } else if (dtype == DFK_F32) {
    const float* s = static_cast<const float*>(src);
    if (n < kParallelMin ||
        !Pool::get().run(n, [=](size_t lo, size_t hi) { f32_to_bf16(s, dst, lo, hi); }))
      f32_to_bf16(s, dst, 0, n);
  } else {
    const double* s = static_cast<const double*>(src);
    if (n < kParallelMin ||
        !Pool::get().run(n, [=](size_t lo, size_t hi) { f64_to_bf16(s, dst, lo, hi); }))
      f64_to_bf16(s, dst, 0, n);
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
