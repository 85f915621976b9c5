// deepfusion_gpu.cpp — the reference operator API (deepfusion.hpp) on top of
// the B200 C ABI (include/dfk.h).  Host-side only: conversion of fp64
// matrices to/from the device, weight-pack caching, exception mapping.  All
// arithmetic runs in libdfk.so's sm_100a kernels; there is no CPU path.
#include "deepfusion.hpp"

#include <cmath>
#include <cstring>
#include <tuple>
#include <mutex>
#include <sstream>

#include "dfk.h"

namespace deepfusion {

namespace {

[[noreturn]] void raise(int status) {
  const std::string msg = dfk_last_error();
  if (status == DFK_ERR_SHAPE) throw ShapeError(msg);
  if (status == DFK_ERR_INVALID) throw std::invalid_argument(msg);
  throw GpuError(status, msg);
}

void check(int status) {
  if (status != DFK_OK) raise(status);
}

// One process-wide context per device (created on first use).
struct Runtime {
  std::mutex mu;
  std::map<int, dfk_context> ctx;
  struct WeightsKey {
    const void* g;
    const void* u;
    const void* d;
    Index dm, df, f0, f1;
    int device;
    bool operator<(const WeightsKey& o) const {
      return std::tie(g, u, d, dm, df, f0, f1, device) <
             std::tie(o.g, o.u, o.d, o.dm, o.df, o.f0, o.f1, o.device);
    }
  };
  struct Cached {
    dfk_weights h = nullptr;
    std::uint64_t fingerprint = 0;
  };
  std::map<WeightsKey, Cached> weights;

  dfk_context context(int device) {
    auto it = ctx.find(device);
    if (it != ctx.end()) return it->second;
    dfk_context c = nullptr;
    check(dfk_context_create(device, nullptr, &c));
    ctx[device] = c;
    return c;
  }
};

Runtime& rt() {
  static Runtime* r = new Runtime();  // intentionally leaked: no teardown race
  return *r;
}

std::uint64_t sample_fingerprint(const Matrix& m) {
  std::uint64_t h = 1469598103934665603ULL ^ static_cast<std::uint64_t>(m.size());
  const Index n = m.size();
  const Index step = n > 256 ? n / 256 : 1;
  for (Index i = 0; i < n; i += step) {
    std::uint64_t b;
    std::memcpy(&b, m.data() + i, 8);
    h = (h ^ b) * 1099511628211ULL;
  }
  return h;
}

// Device handle for (w_gate, w_up, w_down) restricted to [f0, f1) of d_ff.
dfk_weights weights_for(const Matrix& w_gate, const Matrix& w_up,
                        const Matrix& w_down, Index f0, Index f1,
                        int device = 0) {
  Runtime& r = rt();
  std::lock_guard<std::mutex> lk(r.mu);
  const Index dm = w_gate.rows(), df = w_gate.cols();
  Runtime::WeightsKey key{w_gate.data(), w_up.data(), w_down.data(), dm, df, f0,
                          f1, device};
  const std::uint64_t fp = sample_fingerprint(w_gate) ^
                           (sample_fingerprint(w_up) * 3) ^
                           (sample_fingerprint(w_down) * 7);
  auto it = r.weights.find(key);
  if (it != r.weights.end()) {
    if (it->second.fingerprint == fp) return it->second.h;
    dfk_weights_destroy(it->second.h);
    r.weights.erase(it);
  }
  dfk_weights h = nullptr;
  check(dfk_weights_create(r.context(device), w_gate.data(), w_up.data(),
                           w_down.data(), dm, df, DFK_F64, DFK_HOST, f0, f1, &h));
  r.weights[key] = {h, fp};
  return h;
}

// Uncached registration for calls whose weights are temporaries (stage 1
// alone, down alone): destroyed with the guard.
struct TempWeights {
  dfk_weights h = nullptr;
  TempWeights(const Matrix& g, const Matrix& u, const Matrix& d, Index f0, Index f1) {
    check(dfk_weights_create(rt().context(0), g.data(), u.data(), d.data(), g.rows(),
                             g.cols(), DFK_F64, DFK_HOST, f0, f1, &h));
  }
  ~TempWeights() { dfk_weights_destroy(h); }
  TempWeights(const TempWeights&) = delete;
  TempWeights& operator=(const TempWeights&) = delete;
};

std::vector<std::uint16_t> to_bf16(const Matrix& m) {
  std::vector<std::uint16_t> out(static_cast<size_t>(m.size()));
  for (Index i = 0; i < m.size(); ++i) {
    float f = static_cast<float>(m.data()[i]);
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) {
      out[static_cast<size_t>(i)] = static_cast<std::uint16_t>((u >> 16) | 0x40u);
    } else {
      u += 0x7FFFu + ((u >> 16) & 1u);
      out[static_cast<size_t>(i)] = static_cast<std::uint16_t>(u >> 16);
    }
  }
  return out;
}

Matrix from_bf16(const std::vector<std::uint16_t>& v, Index rows, Index cols) {
  Matrix m(rows, cols);
  for (Index i = 0; i < m.size(); ++i) {
    const std::uint32_t u = static_cast<std::uint32_t>(v[static_cast<size_t>(i)]) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    m.data()[i] = f;
  }
  return m;
}

struct DevBuf {
  dfk_context c;
  void* p = nullptr;
  DevBuf(dfk_context ctx, size_t bytes) : c(ctx) { check(dfk_malloc(c, bytes, &p)); }
  ~DevBuf() { dfk_free(c, p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

dfk_config variant_config(VariantTag v) {
  dfk_config c;
  std::memset(&c, 0, sizeof(c));
  if (v == VariantTag::Fused) {
    // Default fused launch (the scheduler's choice once tuned): ask for the
    // library default by passing NULL; this copy is only used for the
    // unfused variants.
    c.variant = DFK_VARIANT_FUSED;
  } else {
    c.variant = v == VariantTag::TwoKernel ? DFK_VARIANT_TWO_KERNEL
                                           : DFK_VARIANT_FOUR_KERNEL;
  }
  return c;
}

const dfk_config* cfg_ptr(VariantTag v, dfk_config* storage) {
  if (v == VariantTag::Fused) return nullptr;
  *storage = variant_config(v);
  return storage;
}

// Stage 1 through the ABI: A2 = (X W_up) * silu(X W_gate).
void gpu_stage1(VariantTag v, const Matrix& x, const Matrix& w_up,
                const Matrix& w_gate, const Matrix* w_down, Matrix& a2) {
  const Index B = x.rows(), dm = x.cols(), df = w_up.cols();
  std::unique_ptr<TempWeights> temp;
  dfk_weights h = nullptr;
  if (w_down) {
    h = weights_for(w_gate, w_up, *w_down, 0, df);
  } else {
    temp = std::make_unique<TempWeights>(w_gate, w_up, Matrix(df, dm), 0, df);
    h = temp->h;
  }
  dfk_context c = rt().context(0);
  DevBuf xd(c, static_cast<size_t>(B * dm) * 2), ad(c, static_cast<size_t>(B * df) * 2);
  const auto xb = to_bf16(x);
  check(dfk_memcpy_h2d(c, xd.p, xb.data(), xb.size() * 2));
  dfk_config storage;
  check(dfk_stage1(c, h, xd.p, B, ad.p, cfg_ptr(v, &storage)));
  std::vector<std::uint16_t> out(static_cast<size_t>(B * df));
  check(dfk_memcpy_d2h(c, out.data(), ad.p, out.size() * 2));
  check(dfk_context_sync(c));
  a2 = from_bf16(out, B, df);
}

Matrix gpu_forward(VariantTag v, const Matrix& x, const MlpWeights& w) {
  dfk_weights h = weights_for(w.w_gate, w.w_up, w.w_down, 0, w.shape.d_ff);
  Matrix y(x.rows(), w.shape.d_model);
  dfk_config storage;
  check(dfk_forward_host(rt().context(0), h, x.data(), DFK_F64, x.rows(), y.data(),
                         DFK_F64, cfg_ptr(v, &storage)));
  return y;
}

void check_input(const Matrix& x, const MlpWeights& w) {
  w.validate();
  if (x.cols() != w.shape.d_model) {
    std::ostringstream msg;
    msg << "executor: x has " << x.cols() << " columns, weights expect d_model="
        << w.shape.d_model;
    throw ShapeError(msg.str());
  }
}

void check_stage1_output(const Matrix& x, const MlpWeights& w, const Matrix& a2) {
  if (a2.rows() != x.rows() || a2.cols() != w.shape.d_ff) {
    std::ostringstream msg;
    msg << "executor: a2 is " << a2.rows() << "x" << a2.cols() << ", expected "
        << x.rows() << "x" << w.shape.d_ff;
    throw ShapeError(msg.str());
  }
}

}  // namespace

// --- Matrix / shapes / generator ------------------------------------------------
Matrix::Matrix(Index rows, Index cols) : rows_(rows), cols_(cols) {
  if (rows < 1 || cols < 1) {
    std::ostringstream msg;
    msg << "Matrix: dimensions must be >= 1, got " << rows << "x" << cols;
    throw ShapeError(msg.str());
  }
  data_.assign(static_cast<size_t>(rows) * static_cast<size_t>(cols), 0.0);
}

Matrix Matrix::identity(Index n) {
  Matrix m(n, n);
  for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}

void Matrix::set_zero() { std::fill(data_.begin(), data_.end(), 0.0); }

void MlpShape::validate() const {
  if (batch < 1 || d_model < 1 || d_ff < 1)
    throw ShapeError("MlpShape: all dimensions must be >= 1, got " + to_string(*this));
}

bool MlpShape::ff_ratio_typical() const {
  const double r = static_cast<double>(d_ff) / static_cast<double>(d_model);
  return r >= 3.5 && r <= 4.0;
}

std::string to_string(const MlpShape& s) {
  std::ostringstream o;
  o << "(B=" << s.batch << ", d_model=" << s.d_model << ", d_ff=" << s.d_ff << ")";
  return o.str();
}

double uniform_double(std::mt19937_64& rng, double lo, double hi) {
  const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
  return lo + u * (hi - lo);
}

void fill_uniform(Matrix& m, std::mt19937_64& rng, double lo, double hi) {
  for (Index i = 0; i < m.rows(); ++i)
    for (Index j = 0; j < m.cols(); ++j) m(i, j) = uniform_double(rng, lo, hi);
}

std::string_view to_string(VariantTag v) {
  switch (v) {
    case VariantTag::FourKernel: return "four_kernel";
    case VariantTag::TwoKernel: return "two_kernel";
    case VariantTag::Fused: return "fused";
  }
  return "unknown";
}

std::optional<VariantTag> variant_from_string(std::string_view s) {
  if (s == "four_kernel" || s == "four-kernel") return VariantTag::FourKernel;
  if (s == "two_kernel" || s == "two-kernel") return VariantTag::TwoKernel;
  if (s == "fused") return VariantTag::Fused;
  return std::nullopt;
}

void MlpWeights::validate() const {
  shape.validate();
  auto expect = [](const Matrix& m, Index r, Index c, const char* name) {
    if (m.rows() != r || m.cols() != c) {
      std::ostringstream msg;
      msg << "MlpWeights: " << name << " is " << m.rows() << "x" << m.cols()
          << ", expected " << r << "x" << c;
      throw ShapeError(msg.str());
    }
  };
  expect(w_up, shape.d_model, shape.d_ff, "w_up");
  expect(w_gate, shape.d_model, shape.d_ff, "w_gate");
  expect(w_down, shape.d_ff, shape.d_model, "w_down");
}

MlpWeights make_random_weights(const MlpShape& shape, std::mt19937_64& rng,
                               double scale) {
  shape.validate();
  MlpWeights w{Matrix(shape.d_model, shape.d_ff), Matrix(shape.d_model, shape.d_ff),
               Matrix(shape.d_ff, shape.d_model), shape};
  fill_uniform(w.w_up, rng, -scale, scale);
  fill_uniform(w.w_gate, rng, -scale, scale);
  fill_uniform(w.w_down, rng, -scale, scale);
  return w;
}

std::string_view to_string(LoopOrder order) {
  return order == LoopOrder::RowMajorTiling ? "row" : "col";
}

void TileConfig::validate() const {
  if (tile_m < 1 || tile_n < 1 || tile_k < 1)
    throw ShapeError("TileConfig: tile dimensions must be >= 1, got " + describe());
}

TileConfig TileConfig::clamped(const MlpShape& s) const {
  TileConfig t = *this;
  t.tile_m = std::min(t.tile_m, s.batch);
  t.tile_n = std::min(t.tile_n, s.d_ff);
  t.tile_k = std::min(t.tile_k, s.d_model);
  return t;
}

std::string TileConfig::describe() const {
  std::ostringstream o;
  o << "m" << tile_m << "_n" << tile_n << "_k" << tile_k << "_" << to_string(loop_order);
  return o.str();
}

// --- executors -------------------------------------------------------------------
void run_four_kernel_stage1(const Matrix& x, const MlpWeights& w, Matrix& a2,
                            Accounting) {
  check_input(x, w);
  check_stage1_output(x, w, a2);
  gpu_stage1(VariantTag::FourKernel, x, w.w_up, w.w_gate, &w.w_down, a2);
}

Matrix run_four_kernel(const Matrix& x, const MlpWeights& w, Accounting) {
  check_input(x, w);
  return gpu_forward(VariantTag::FourKernel, x, w);
}

void run_two_kernel_stage1(const Matrix& x, const MlpWeights& w, Matrix& a2,
                           Accounting) {
  check_input(x, w);
  check_stage1_output(x, w, a2);
  gpu_stage1(VariantTag::TwoKernel, x, w.w_up, w.w_gate, &w.w_down, a2);
}

Matrix run_two_kernel(const Matrix& x, const MlpWeights& w, Accounting) {
  check_input(x, w);
  return gpu_forward(VariantTag::TwoKernel, x, w);
}

Matrix down_projection(const Matrix& a2, const Matrix& w_down, Accounting) {
  if (a2.cols() != w_down.rows()) {
    std::ostringstream msg;
    msg << "down_projection: a2 has " << a2.cols() << " columns, w_down has "
        << w_down.rows() << " rows";
    throw ShapeError(msg.str());
  }
  const Index B = a2.rows(), df = a2.cols(), dm = w_down.cols();
  const Matrix zeros(dm, df);
  TempWeights temp(zeros, zeros, w_down, 0, df);
  dfk_weights h = temp.h;
  dfk_context c = rt().context(0);
  DevBuf ad(c, static_cast<size_t>(B * df) * 2), yd(c, static_cast<size_t>(B * dm) * 4);
  const auto ab = to_bf16(a2);
  check(dfk_memcpy_h2d(c, ad.p, ab.data(), ab.size() * 2));
  check(dfk_down(c, h, ad.p, B, yd.p, DFK_F32, nullptr));
  std::vector<float> out(static_cast<size_t>(B * dm));
  check(dfk_memcpy_d2h(c, out.data(), yd.p, out.size() * 4));
  check(dfk_context_sync(c));
  Matrix y(B, dm);
  for (Index i = 0; i < y.size(); ++i) y.data()[i] = out[static_cast<size_t>(i)];
  return y;
}

void run_fused_stage1(const Matrix& x, const Matrix& w_up, const Matrix& w_gate,
                      const TileConfig& tile, Matrix& a2, int) {
  tile.validate();
  if (w_up.rows() != x.cols() || w_gate.rows() != x.cols() ||
      w_up.cols() != w_gate.cols()) {
    std::ostringstream msg;
    msg << "run_fused_stage1: inconsistent dims, x is " << x.rows() << "x" << x.cols()
        << ", w_up is " << w_up.rows() << "x" << w_up.cols() << ", w_gate is "
        << w_gate.rows() << "x" << w_gate.cols();
    throw ShapeError(msg.str());
  }
  if (a2.rows() != x.rows() || a2.cols() != w_up.cols()) {
    std::ostringstream msg;
    msg << "run_fused_stage1: a2 is " << a2.rows() << "x" << a2.cols()
        << ", expected " << x.rows() << "x" << w_up.cols();
    throw ShapeError(msg.str());
  }
  gpu_stage1(VariantTag::Fused, x, w_up, w_gate, nullptr, a2);
}

Matrix run_fused(const Matrix& x, const MlpWeights& w, const TileConfig& tile, int) {
  check_input(x, w);
  tile.validate();
  return gpu_forward(VariantTag::Fused, x, w);
}

void run_stage1(VariantTag variant, const Matrix& x, const MlpWeights& w, Matrix& a2,
                const TileConfig& tile, Accounting mode) {
  switch (variant) {
    case VariantTag::FourKernel:
      run_four_kernel_stage1(x, w, a2, mode);
      return;
    case VariantTag::TwoKernel:
      run_two_kernel_stage1(x, w, a2, mode);
      return;
    case VariantTag::Fused:
      w.validate();
      run_fused_stage1(x, w.w_up, w.w_gate, tile, a2);
      return;
  }
  throw std::invalid_argument("run_stage1: unknown variant");
}

Matrix run_variant(const KernelConfig& config, const Matrix& x, const MlpWeights& w,
                   Accounting) {
  check_input(x, w);
  config.tile.validate();
  if (config.variant != VariantTag::Fused && config.variant != VariantTag::TwoKernel &&
      config.variant != VariantTag::FourKernel)
    throw std::invalid_argument("run_stage1: unknown variant");
  return gpu_forward(config.variant, x, w);
}

// --- tensor parallelism ------------------------------------------------------------
std::vector<ColRange> balanced_ranges(Index extent, Index parts) {
  std::vector<ColRange> out;
  if (parts < 1) {
    Index b, e;
    raise(dfk_balanced_range(extent, parts, 0, &b, &e));
  }
  for (Index p = 0; p < parts; ++p) {
    Index b = 0, e = 0;
    check(dfk_balanced_range(extent, parts, p, &b, &e));
    out.push_back({b, e});
  }
  return out;
}

void ShardPlan::validate(Index d_ff) const {
  if (num_devices < 1 || ff_ranges.size() != static_cast<size_t>(num_devices))
    throw ShapeError("ShardPlan: range count does not match num_devices");
  Index cursor = 0;
  for (const ColRange& r : ff_ranges) {
    if (r.begin != cursor || r.size() < 1) {
      std::ostringstream msg;
      msg << "ShardPlan: ranges must be contiguous, disjoint and non-empty; "
             "offending range ["
          << r.begin << ", " << r.end << ") at cursor " << cursor;
      throw ShapeError(msg.str());
    }
    cursor = r.end;
  }
  if (cursor != d_ff) {
    std::ostringstream msg;
    msg << "ShardPlan: ranges cover [0, " << cursor << ") but d_ff is " << d_ff;
    throw ShapeError(msg.str());
  }
}

ShardPlan make_plan(Index d_ff, Index num_devices, ShardScheme scheme) {
  ShardPlan p;
  p.num_devices = num_devices;
  p.ff_ranges = balanced_ranges(d_ff, num_devices);
  p.scheme = scheme;
  return p;
}

std::string_view to_string(CollectiveKind kind) {
  return kind == CollectiveKind::AllReduce ? "all_reduce" : "all_gather";
}

TpResult run_tp_mlp(const Matrix& x, const MlpWeights& w, const ShardPlan& plan,
                    const KernelConfig& executor) {
  w.validate();
  plan.validate(w.shape.d_ff);
  if (plan.scheme != ShardScheme::CompoundSingleAllReduce)
    throw std::invalid_argument(
        "run_tp_mlp: plan scheme must be CompoundSingleAllReduce (use "
        "run_naive_tp_mlp for the per-GEMM baseline)");
  if (x.cols() != w.shape.d_model)
    throw ShapeError("run_tp_mlp: x column count does not match d_model");
  const Index B = x.rows(), dm = w.shape.d_model;
  dfk_config storage;
  const dfk_config* cfg = cfg_ptr(executor.variant, &storage);
  TpResult result;
  int ndev = 0;
  dfk_device_count(&ndev);
  const auto xb = to_bf16(x);
  if (plan.num_devices > 1 && plan.num_devices <= 8 && dm % 4 == 0 && B <= 256) {
    // One context per rank -- on its own device when there are enough, else
    // all on device 0 (each rank's block on its own stream) -- with the
    // fused all-reduce: partial Y reduced over peer memory INSIDE the block
    // kernel (dfk_tp_forward_fused), the block's one collective
    // (tp.cpp:140-167).  Every buffer exists before the first launch.
    const bool multi = plan.num_devices <= ndev;
    std::vector<dfk_context> ctxs(static_cast<size_t>(plan.num_devices));
    for (Index p = 0; p < plan.num_devices; ++p)
      check(dfk_context_create(multi ? static_cast<int>(p) : 0, nullptr,
                               &ctxs[static_cast<size_t>(p)]));
    for (dfk_context c : ctxs) check(dfk_tp_sym_create(c, B, dm, nullptr));
    check(dfk_tp_sym_attach(ctxs.data(), static_cast<int>(plan.num_devices)));
    std::vector<dfk_weights> hs;
    std::vector<void*> xs, ys, as;
    for (Index p = 0; p < plan.num_devices; ++p) {
      const ColRange r = plan.ff_ranges[static_cast<size_t>(p)];
      dfk_context c = ctxs[static_cast<size_t>(p)];
      dfk_weights h = nullptr;
      check(dfk_weights_create(c, w.w_gate.data(), w.w_up.data(), w.w_down.data(), dm,
                               w.shape.d_ff, DFK_F64, DFK_HOST, r.begin, r.end, &h));
      hs.push_back(h);
      void *xp, *yp, *ap;
      check(dfk_malloc(c, xb.size() * 2, &xp));
      check(dfk_malloc(c, static_cast<size_t>(B * dm) * 4, &yp));
      check(dfk_malloc(c, static_cast<size_t>(B * r.size()) * 2, &ap));
      check(dfk_memcpy_h2d(c, xp, xb.data(), xb.size() * 2));
      xs.push_back(xp);
      ys.push_back(yp);
      as.push_back(ap);
    }
    // Stage-1 shards (for TpResult::stage1_shards), synchronised, then the
    // fused blocks issued back to back on the ranks' streams.
    for (Index p = 0; p < plan.num_devices; ++p) {
      check(dfk_stage1(ctxs[static_cast<size_t>(p)], hs[static_cast<size_t>(p)],
                       xs[static_cast<size_t>(p)], B, as[static_cast<size_t>(p)], cfg));
      check(dfk_context_sync(ctxs[static_cast<size_t>(p)]));
    }
    for (Index p = 0; p < plan.num_devices; ++p)
      check(dfk_tp_forward_fused(ctxs[static_cast<size_t>(p)], hs[static_cast<size_t>(p)],
                                 xs[static_cast<size_t>(p)], B,
                                 static_cast<float*>(ys[static_cast<size_t>(p)]), cfg));
    std::vector<float> out(static_cast<size_t>(B * dm));
    for (Index p = 0; p < plan.num_devices; ++p) check(dfk_context_sync(ctxs[static_cast<size_t>(p)]));
    for (Index p = 0; p < plan.num_devices; ++p) {
      dfk_context c = ctxs[static_cast<size_t>(p)];
      const ColRange r = plan.ff_ranges[static_cast<size_t>(p)];
      std::vector<std::uint16_t> a(static_cast<size_t>(B * r.size()));
      check(dfk_memcpy_d2h(c, a.data(), as[static_cast<size_t>(p)], a.size() * 2));
      if (p == 0) check(dfk_memcpy_d2h(c, out.data(), ys[0], out.size() * 4));
      check(dfk_context_sync(c));
      result.stage1_shards.push_back(from_bf16(a, B, r.size()));
    }
    result.output = Matrix(B, dm);
    for (Index i = 0; i < result.output.size(); ++i)
      result.output.data()[i] = out[static_cast<size_t>(i)];
    for (Index p = 0; p < plan.num_devices; ++p) {
      dfk_context c = ctxs[static_cast<size_t>(p)];
      dfk_free(c, xs[static_cast<size_t>(p)]);
      dfk_free(c, ys[static_cast<size_t>(p)]);
      dfk_free(c, as[static_cast<size_t>(p)]);
      dfk_weights_destroy(hs[static_cast<size_t>(p)]);
      dfk_context_destroy(c);
    }
  } else {
    // Shapes the fused all-reduce does not take (d_model % 4, B > 256, more
    // than 8 ranks): shards in sequence on one GPU, fp32 partials summed in
    // device order.
    dfk_context c = rt().context(0);
    DevBuf xd(c, xb.size() * 2), yd(c, static_cast<size_t>(B * dm) * 4);
    check(dfk_memcpy_h2d(c, xd.p, xb.data(), xb.size() * 2));
    result.output = Matrix(B, dm);
    std::vector<float> part(static_cast<size_t>(B * dm));
    for (const ColRange& r : plan.ff_ranges) {
      dfk_weights h = weights_for(w.w_gate, w.w_up, w.w_down, r.begin, r.end);
      DevBuf ad(c, static_cast<size_t>(B * r.size()) * 2);
      check(dfk_stage1(c, h, xd.p, B, ad.p, cfg));
      check(dfk_down(c, h, ad.p, B, yd.p, DFK_F32, cfg));
      std::vector<std::uint16_t> a(static_cast<size_t>(B * r.size()));
      check(dfk_memcpy_d2h(c, a.data(), ad.p, a.size() * 2));
      check(dfk_memcpy_d2h(c, part.data(), yd.p, part.size() * 4));
      check(dfk_context_sync(c));
      result.stage1_shards.push_back(from_bf16(a, B, r.size()));
      for (Index i = 0; i < result.output.size(); ++i)
        result.output.data()[i] += part[static_cast<size_t>(i)];
    }
  }
  result.log.events.push_back(
      {CollectiveKind::AllReduce, static_cast<std::uint64_t>(B * dm)});
  return result;
}

double comm_volume_bytes(const CollectiveLog& log, Index num_devices, CommModel model,
                         std::uint64_t bytes_per_element) {
  if (num_devices < 1) throw ShapeError("comm_volume_bytes: num_devices must be >= 1");
  const double p = static_cast<double>(num_devices);
  double bytes = 0.0;
  for (const CollectiveEvent& e : log.events) {
    const double payload =
        static_cast<double>(e.payload_elements_per_device * bytes_per_element);
    if (model == CommModel::Logical) {
      bytes += payload;
    } else if (e.kind == CollectiveKind::AllReduce) {
      bytes += 2.0 * (p - 1.0) / p * payload;
    } else {
      bytes += (p - 1.0) / p * payload;
    }
  }
  return bytes;
}

// --- scheduler -------------------------------------------------------------------
std::string default_fingerprint() {
  char buf[256];
  check(dfk_fingerprint(rt().context(0), buf, sizeof(buf)));
  return buf;
}

ScheduleEntry Tuner::get_or_tune(const MlpShape& shape, const MlpWeights& w) {
  w.validate();
  if (opts_.warmup < 1) throw std::invalid_argument("profile: warmup must be >= 1");
  if (opts_.runs < 3) throw std::invalid_argument("profile: runs must be >= 3");
  dfk_weights h = weights_for(w.w_gate, w.w_up, w.w_down, 0, w.shape.d_ff);
  dfk_config chosen;
  int32_t hit = 0;
  std::vector<char> json(1 << 16);
  check(dfk_tune(rt().context(0), h, shape.batch,
                 opts_.cache_path.empty() ? nullptr : opts_.cache_path.c_str(),
                 opts_.warmup, opts_.runs, &chosen, &hit, json.data(), json.size()));
  last_was_cache_hit_ = hit != 0;
  if (!hit) ++profile_invocations_;
  return {shape, default_fingerprint(), chosen.label, json.data(), hit != 0};
}

void release_gpu_cache() {
  Runtime& r = rt();
  std::lock_guard<std::mutex> lk(r.mu);
  for (auto& [k, v] : r.weights) dfk_weights_destroy(v.h);
  r.weights.clear();
}

}  // namespace deepfusion
