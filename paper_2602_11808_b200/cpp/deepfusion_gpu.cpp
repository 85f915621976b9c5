// deepfusion_gpu.cpp — the reference operator API (deepfusion.hpp) on top of
// the B200 C ABI (include/dfk.h).  Host-side only: conversion of fp64
// matrices to/from the device, weight-pack caching, exception mapping, the
// scheduler's reference-facing surface.  All arithmetic runs in libdfk.so's
// sm_100a kernels; there is no CPU path.
#include "deepfusion.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <ctime>
#include <list>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>

#include <json.hpp>

#include "dfk.h"

namespace deepfusion {

namespace {

[[noreturn]] void raise(int status) {
  const std::string msg = dfk_last_error();
  if (status == DFK_ERR_SHAPE) throw ShapeError(msg);
  if (status == DFK_ERR_INVALID) throw std::invalid_argument(msg);
  if (status == DFK_ERR_CACHE) throw CacheError(msg);
  throw GpuError(status, msg);
}

void check(int status) {
  if (status != DFK_OK) raise(status);
}

// Device scratch of one context, grown on demand (never per call).
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(dfk_context c, size_t need) {
    if (need > bytes) {
      if (p) dfk_free(c, p);
      p = nullptr;
      bytes = 0;
      check(dfk_malloc(c, need, &p));
      bytes = need;
    }
    return p;
  }
};

// Pinned host staging for the stage-only calls' copies (pageable std::vector
// buffers made every H2D / D2H a bounce-buffered synchronous copy: ~0.3 ms of
// run_fused_stage1's A2 read-back at Llama-8B B = 64).  Grows geometrically;
// used under Runtime::mu.
struct PinnedScratch {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      const size_t nb = std::max(need, 2 * bytes);
      if (p) dfk_host_free(p);
      p = nullptr;
      bytes = 0;
      check(dfk_host_alloc(nb, &p));
      bytes = nb;
    }
    return p;
  }
};

// One process-wide context per device (created on first use), its scratch,
// and an LRU cache of prepacked weight sets keyed by the matrices' exact
// contents (Matrix id + version, see deepfusion.hpp).
struct Runtime {
  std::mutex mu;
  std::map<int, dfk_context> ctx;
  std::map<int, Scratch> x_buf, a2_buf, y_buf;
  PinnedScratch h_in, h_out;  // host staging of the stage-only calls

  struct Key {
    std::uint64_t g_id, g_ver, u_id, u_ver, d_id, d_ver;
    Index dm, df, f0, f1;
    int device;
    bool operator<(const Key& o) const {
      return std::tie(g_id, g_ver, u_id, u_ver, d_id, d_ver, dm, df, f0, f1, device) <
             std::tie(o.g_id, o.g_ver, o.u_id, o.u_ver, o.d_id, o.d_ver, o.dm, o.df, o.f0,
                      o.f1, o.device);
    }
  };
  // most recently used at the front
  std::list<std::pair<Key, dfk_weights>> lru;

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

std::uint64_t id_of(const Matrix* m) { return m ? m->id() : 0; }
std::uint64_t ver_of(const Matrix* m) { return m ? m->version() : 0; }

// Device handle for (w_gate, w_up, w_down) restricted to [f0, f1) of d_ff;
// w_gate/w_up or w_down may be null (stage-only sets).  Served from the
// cache while the matrices are unchanged; caller holds rt().mu.
dfk_weights weights_for_locked(const Matrix* w_gate, const Matrix* w_up,
                               const Matrix* w_down, Index f0, Index f1, int device = 0) {
  Runtime& r = rt();
  const Index dm = w_gate ? w_gate->rows() : w_down->cols();
  const Index df = w_gate ? w_gate->cols() : w_down->rows();
  const Runtime::Key key{id_of(w_gate), ver_of(w_gate), id_of(w_up), ver_of(w_up),
                         id_of(w_down), ver_of(w_down), dm, df, f0, f1, device};
  for (auto it = r.lru.begin(); it != r.lru.end(); ++it) {
    if (!(it->first < key) && !(key < it->first)) {
      r.lru.splice(r.lru.begin(), r.lru, it);
      return it->second;
    }
  }
  dfk_weights h = nullptr;
  check(dfk_weights_create(r.context(device), w_gate ? w_gate->data() : nullptr,
                           w_up ? w_up->data() : nullptr, w_down ? w_down->data() : nullptr,
                           dm, df, DFK_F64, DFK_HOST, f0, f1, &h));
  r.lru.emplace_front(key, h);
  while (static_cast<int>(r.lru.size()) > kGpuCachedWeightSets) {
    dfk_weights_destroy(r.lru.back().second);
    r.lru.pop_back();
  }
  return h;
}

// Matrix <-> device element conversions on the library's host pool
// (dfk_host_to_bf16 / dfk_host_from_bf16: RNE, as the device rounds).
void to_bf16(const double* src, Index n, std::uint16_t* out) {
  check(dfk_host_to_bf16(src, DFK_F64, static_cast<size_t>(n), out));
}

void from_bf16(const std::uint16_t* v, Matrix& m) {
  check(dfk_host_from_bf16(v, static_cast<size_t>(m.size()), m.data(), DFK_F64));
}

const dfk_config* cfg_ptr(VariantTag v, dfk_config* storage) {
  if (v == VariantTag::Fused) return nullptr;  // the scheduler's / library's pick
  std::memset(storage, 0, sizeof(*storage));
  storage->variant =
      v == VariantTag::TwoKernel ? DFK_VARIANT_TWO_KERNEL : DFK_VARIANT_FOUR_KERNEL;
  return storage;
}

// The GPU launch configuration a KernelConfig names: one of
// dfk_candidates_shape's labels (gpu_candidates), else the variant's default.
bool gpu_config_for(const KernelConfig& k, Index B, Index dm, Index df, dfk_config* out) {
  if (k.label.empty()) return false;
  dfk_context c = rt().context(0);
  std::vector<dfk_config> all(256);
  int32_t n = 0;
  check(dfk_candidates_shape(c, B, dm, df, all.data(), static_cast<int32_t>(all.size()), &n));
  for (int32_t i = 0; i < std::min<int32_t>(n, static_cast<int32_t>(all.size())); ++i) {
    if (k.label == all[static_cast<size_t>(i)].label) {
      *out = all[static_cast<size_t>(i)];
      return true;
    }
  }
  return false;
}

// Stage 1 through the ABI: A2 = (X W_up) * silu(X W_gate).  `w_down` given:
// the full set is cached (and shared with full-block calls).
void gpu_stage1(const dfk_config* cfg, const Matrix& x, const Matrix& w_up,
                const Matrix& w_gate, const Matrix* w_down, Matrix& a2) {
  const Index B = x.rows(), dm = x.cols(), df = w_up.cols();
  Runtime& r = rt();
  std::lock_guard<std::mutex> lk(r.mu);
  dfk_weights h = weights_for_locked(&w_gate, &w_up, w_down, 0, df);
  dfk_context c = r.context(0);
  void* xd = r.x_buf[0].get(c, static_cast<size_t>(B * dm) * 2);
  void* ad = r.a2_buf[0].get(c, static_cast<size_t>(B * df) * 2);
  auto* xb = static_cast<std::uint16_t*>(r.h_in.get(static_cast<size_t>(B * dm) * 2));
  auto* out = static_cast<std::uint16_t*>(r.h_out.get(static_cast<size_t>(B * df) * 2));
  to_bf16(x.data(), B * dm, xb);
  check(dfk_memcpy_h2d(c, xd, xb, static_cast<size_t>(B * dm) * 2));
  check(dfk_stage1(c, h, xd, B, ad, cfg));
  check(dfk_memcpy_d2h(c, out, ad, static_cast<size_t>(B * df) * 2));
  check(dfk_context_sync(c));
  from_bf16(out, a2);
}

Matrix gpu_forward(const dfk_config* cfg, const Matrix& x, const MlpWeights& w) {
  Runtime& r = rt();
  std::lock_guard<std::mutex> lk(r.mu);
  dfk_weights h = weights_for_locked(&w.w_gate, &w.w_up, &w.w_down, 0, w.shape.d_ff);
  Matrix y(x.rows(), w.shape.d_model);
  check(dfk_forward_host(r.context(0), h, x.data(), DFK_F64, x.rows(), y.data(), DFK_F64,
                         cfg));
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

void check_fused_stage1_args(const Matrix& x, const Matrix& w_up, const Matrix& w_gate,
                             const Matrix& a2) {
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
    msg << "run_fused_stage1: a2 is " << a2.rows() << "x" << a2.cols() << ", expected "
        << x.rows() << "x" << w_up.cols();
    throw ShapeError(msg.str());
  }
}

}  // namespace

// --- Matrix / shapes / generator ------------------------------------------------
Matrix::Matrix(Index rows, Index cols) : rows_(rows), cols_(cols), id_(next_id()) {
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

void Matrix::set_zero() {
  ++version_;
  std::fill(data_.begin(), data_.end(), 0.0);
}

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
  dfk_config storage;
  gpu_stage1(cfg_ptr(VariantTag::FourKernel, &storage), x, w.w_up, w.w_gate, &w.w_down, a2);
}

Matrix run_four_kernel(const Matrix& x, const MlpWeights& w, Accounting) {
  check_input(x, w);
  dfk_config storage;
  return gpu_forward(cfg_ptr(VariantTag::FourKernel, &storage), x, w);
}

void run_two_kernel_stage1(const Matrix& x, const MlpWeights& w, Matrix& a2,
                           Accounting) {
  check_input(x, w);
  check_stage1_output(x, w, a2);
  dfk_config storage;
  gpu_stage1(cfg_ptr(VariantTag::TwoKernel, &storage), x, w.w_up, w.w_gate, &w.w_down, a2);
}

Matrix run_two_kernel(const Matrix& x, const MlpWeights& w, Accounting) {
  check_input(x, w);
  dfk_config storage;
  return gpu_forward(cfg_ptr(VariantTag::TwoKernel, &storage), x, w);
}

// Y = A2 W_down with a down-only weight set (cached like every other set).
Matrix down_projection(const Matrix& a2, const Matrix& w_down, Accounting) {
  if (a2.cols() != w_down.rows()) {
    std::ostringstream msg;
    msg << "down_projection: a2 has " << a2.cols() << " columns, w_down has "
        << w_down.rows() << " rows";
    throw ShapeError(msg.str());
  }
  const Index B = a2.rows(), df = a2.cols(), dm = w_down.cols();
  Runtime& r = rt();
  std::lock_guard<std::mutex> lk(r.mu);
  dfk_weights h = weights_for_locked(nullptr, nullptr, &w_down, 0, df);
  dfk_context c = r.context(0);
  void* ad = r.a2_buf[0].get(c, static_cast<size_t>(B * df) * 2);
  void* yd = r.y_buf[0].get(c, static_cast<size_t>(B * dm) * 4);
  auto* ab = static_cast<std::uint16_t*>(r.h_in.get(static_cast<size_t>(B * df) * 2));
  auto* out = static_cast<float*>(r.h_out.get(static_cast<size_t>(B * dm) * 4));
  to_bf16(a2.data(), B * df, ab);
  check(dfk_memcpy_h2d(c, ad, ab, static_cast<size_t>(B * df) * 2));
  check(dfk_down(c, h, ad, B, yd, DFK_F32, nullptr));
  check(dfk_memcpy_d2h(c, out, yd, static_cast<size_t>(B * dm) * 4));
  check(dfk_context_sync(c));
  Matrix y(B, dm);
  check(dfk_host_from_f32(out, static_cast<size_t>(B * dm), y.data(), DFK_F64));
  return y;
}

// Stage 1 with a stage-1-only weight set (W_up, W_gate; cached).
void run_fused_stage1(const Matrix& x, const Matrix& w_up, const Matrix& w_gate,
                      const TileConfig& tile, Matrix& a2, int) {
  tile.validate();
  check_fused_stage1_args(x, w_up, w_gate, a2);
  gpu_stage1(nullptr, x, w_up, w_gate, nullptr, a2);
}

Matrix run_fused(const Matrix& x, const MlpWeights& w, const TileConfig& tile, int) {
  check_input(x, w);
  tile.validate();
  return gpu_forward(nullptr, x, w);
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

// A KernelConfig whose label is one of gpu_candidates() runs that launch
// configuration; any other label runs the variant's default.
Matrix run_variant(const KernelConfig& config, const Matrix& x, const MlpWeights& w,
                   Accounting) {
  check_input(x, w);
  config.tile.validate();
  if (config.variant != VariantTag::Fused && config.variant != VariantTag::TwoKernel &&
      config.variant != VariantTag::FourKernel)
    throw std::invalid_argument("run_stage1: unknown variant");
  dfk_config storage;
  if (gpu_config_for(config, x.rows(), w.shape.d_model, w.shape.d_ff, &storage))
    return gpu_forward(&storage, x, w);
  return gpu_forward(cfg_ptr(config.variant, &storage), x, w);
}

ReuseCounts predicted_reuse_counts(const MlpShape& shape, const TileConfig& tile) {
  shape.validate();
  tile.validate();
  const TileConfig t = tile.clamped(shape);
  const auto B = static_cast<std::uint64_t>(shape.batch);
  const auto dm = static_cast<std::uint64_t>(shape.d_model);
  const auto df = static_cast<std::uint64_t>(shape.d_ff);
  const auto blocks = [](std::uint64_t n, std::uint64_t b) { return (n + b - 1) / b; };
  ReuseCounts r;
  r.a2_writes = B * df;
  if (t.loop_order == LoopOrder::ColumnMajorTiling) {
    // weight strips resident, X re-staged once per column block
    r.x_reads = B * dm * blocks(df, static_cast<std::uint64_t>(t.tile_n));
    r.weight_reads = 2 * dm * df;
  } else {
    // X strips resident, weight strips re-staged once per row block
    r.x_reads = B * dm;
    r.weight_reads = 2 * dm * df * blocks(B, static_cast<std::uint64_t>(t.tile_m));
  }
  return r;
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
  std::vector<std::uint16_t> xb(static_cast<size_t>(x.size()));
  to_bf16(x.data(), x.size(), xb.data());
  // The fused all-reduce needs every rank on its balanced_ranges shard (the
  // tile-completion count is derived from it); other plans run the shards
  // in sequence below.
  const bool balanced = plan.ff_ranges == balanced_ranges(w.shape.d_ff, plan.num_devices);
  if (balanced && plan.num_devices > 1 && plan.num_devices <= 8 && dm % 4 == 0 && B <= 256) {
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
                                 ys[static_cast<size_t>(p)], DFK_F32, cfg));
    std::vector<float> out(static_cast<size_t>(B * dm));
    for (Index p = 0; p < plan.num_devices; ++p) check(dfk_context_sync(ctxs[static_cast<size_t>(p)]));
    for (Index p = 0; p < plan.num_devices; ++p) {
      dfk_context c = ctxs[static_cast<size_t>(p)];
      const ColRange r = plan.ff_ranges[static_cast<size_t>(p)];
      std::vector<std::uint16_t> a(static_cast<size_t>(B * r.size()));
      check(dfk_memcpy_d2h(c, a.data(), as[static_cast<size_t>(p)], a.size() * 2));
      if (p == 0) check(dfk_memcpy_d2h(c, out.data(), ys[0], out.size() * 4));
      check(dfk_context_sync(c));
      Matrix shard(B, r.size());
      from_bf16(a.data(), shard);
      result.stage1_shards.push_back(std::move(shard));
    }
    result.output = Matrix(B, dm);
    check(dfk_host_from_f32(out.data(), static_cast<size_t>(result.output.size()),
                            result.output.data(), DFK_F64));
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
    Runtime& rr = rt();
    std::lock_guard<std::mutex> lk(rr.mu);
    dfk_context c = rr.context(0);
    void* xd = rr.x_buf[0].get(c, xb.size() * 2);
    void* yd = rr.y_buf[0].get(c, static_cast<size_t>(B * dm) * 4);
    check(dfk_memcpy_h2d(c, xd, xb.data(), xb.size() * 2));
    result.output = Matrix(B, dm);
    double* ov = result.output.data();
    std::vector<float> part(static_cast<size_t>(B * dm));
    for (const ColRange& r : plan.ff_ranges) {
      dfk_weights h = weights_for_locked(&w.w_gate, &w.w_up, &w.w_down, r.begin, r.end);
      void* ad = rr.a2_buf[0].get(c, static_cast<size_t>(B * r.size()) * 2);
      check(dfk_stage1(c, h, xd, B, ad, cfg));
      check(dfk_down(c, h, ad, B, yd, DFK_F32, cfg));
      std::vector<std::uint16_t> a(static_cast<size_t>(B * r.size()));
      check(dfk_memcpy_d2h(c, a.data(), ad, a.size() * 2));
      check(dfk_memcpy_d2h(c, part.data(), yd, part.size() * 4));
      check(dfk_context_sync(c));
      Matrix shard(B, r.size());
      from_bf16(a.data(), shard);
      result.stage1_shards.push_back(std::move(shard));
      for (Index i = 0; i < result.output.size(); ++i) ov[i] += part[static_cast<size_t>(i)];
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
namespace {

using nlohmann::json;

int variant_rank(VariantTag v) {  // deeper fusion first on ties (tuner.cpp:23-30)
  return v == VariantTag::Fused ? 0 : v == VariantTag::TwoKernel ? 1 : 2;
}

std::string utc_now() {
  const std::time_t t = std::chrono::system_clock::to_time_t(std::chrono::system_clock::now());
  std::tm u{};
  gmtime_r(&t, &u);
  char b[32];
  std::strftime(b, sizeof(b), "%Y-%m-%dT%H:%M:%SZ", &u);
  return b;
}

// max|a - ref| / max|ref| (max|a - ref| when ref is all zero).
double rel_inf(const Matrix& a, const Matrix& ref) {
  double num = 0.0, den = 0.0;
  for (Index i = 0; i < a.size(); ++i) {
    const double d = std::fabs(a.data()[i] - ref.data()[i]);
    num = std::isnan(d) ? INFINITY : std::max(num, d);
    den = std::max(den, std::fabs(ref.data()[i]));
  }
  return den > 0 ? num / den : num;
}

// ScheduleEntry <-> the cache schema (tuner.cpp:198-266 field names).
json entry_to_json(const ScheduleEntry& e) {
  json results = json::array();
  for (const BenchmarkResult& r : e.all_results) {
    json j = {{"label", r.config_label},
              {"variant", std::string(to_string(r.variant))},
              {"samples_ns", r.samples_ns},
              {"median_ns", r.median_ns},
              {"warmup_runs", r.warmup_runs},
              {"measured_runs", r.measured_runs}};
    if (r.disqualified) j["disqualified"] = *r.disqualified;
    results.push_back(std::move(j));
  }
  return {{"shape", {{"batch", e.shape.batch}, {"d_model", e.shape.d_model},
                     {"d_ff", e.shape.d_ff}}},
          {"fingerprint", e.fingerprint},
          {"chosen", e.chosen},
          {"created_at", e.created_at},
          {"results", std::move(results)}};
}

ScheduleEntry entry_from_json(const json& j, const std::string& where) {
  const auto need = [&](const json& o, const char* k) -> const json& {
    auto it = o.find(k);
    if (it == o.end()) throw CacheError(where + ": entry has no '" + k + "'");
    return *it;
  };
  try {
    ScheduleEntry e;
    const json& sh = need(j, "shape");
    e.shape = {need(sh, "batch").get<Index>(), need(sh, "d_model").get<Index>(),
               need(sh, "d_ff").get<Index>()};
    e.fingerprint = need(j, "fingerprint").get<std::string>();
    e.chosen = need(j, "chosen").get<std::string>();
    e.created_at = need(j, "created_at").get<std::string>();
    for (const json& r : need(j, "results")) {
      BenchmarkResult b;
      b.config_label = need(r, "label").get<std::string>();
      const auto v = variant_from_string(need(r, "variant").get<std::string>());
      if (!v) throw CacheError(where + ": unknown variant name in a result");
      b.variant = *v;
      b.samples_ns = need(r, "samples_ns").get<std::vector<std::int64_t>>();
      b.median_ns = need(r, "median_ns").get<std::int64_t>();
      b.warmup_runs = need(r, "warmup_runs").get<int>();
      b.measured_runs = need(r, "measured_runs").get<int>();
      if (auto d = r.find("disqualified"); d != r.end()) b.disqualified = d->get<std::string>();
      e.all_results.push_back(std::move(b));
    }
    return e;
  } catch (const json::exception& ex) {
    throw CacheError(where + ": malformed entry (" + ex.what() + ")");
  }
}

}  // namespace

std::vector<KernelConfig> default_candidates(const MlpShape& shape) {
  shape.validate();
  std::vector<KernelConfig> out = {{VariantTag::FourKernel, {}, "four_kernel"},
                                   {VariantTag::TwoKernel, {}, "two_kernel"}};
  std::set<std::tuple<Index, Index, Index, LoopOrder>> seen;
  for (Index tm : {Index{1}, shape.batch})
    for (Index tn : {Index{32}, Index{128}, shape.d_ff})
      for (Index tk : {Index{32}, shape.d_model})
        for (LoopOrder o : {LoopOrder::RowMajorTiling, LoopOrder::ColumnMajorTiling}) {
          const TileConfig t = TileConfig{tm, tn, tk, o}.clamped(shape);
          if (seen.emplace(t.tile_m, t.tile_n, t.tile_k, o).second)
            out.push_back({VariantTag::Fused, t, "fused_" + t.describe()});
        }
  return out;
}

std::vector<KernelConfig> gpu_candidates(const MlpShape& shape) {
  shape.validate();
  std::vector<dfk_config> all(256);
  int32_t n = 0;
  {
    std::lock_guard<std::mutex> lk(rt().mu);
    check(dfk_candidates_shape(rt().context(0), shape.batch, shape.d_model, shape.d_ff,
                               all.data(), static_cast<int32_t>(all.size()), &n));
  }
  std::vector<KernelConfig> out;
  for (int32_t i = 0; i < std::min<int32_t>(n, static_cast<int32_t>(all.size())); ++i) {
    const dfk_config& c = all[static_cast<size_t>(i)];
    const VariantTag v = c.variant == DFK_VARIANT_TWO_KERNEL    ? VariantTag::TwoKernel
                         : c.variant == DFK_VARIANT_FOUR_KERNEL ? VariantTag::FourKernel
                                                                : VariantTag::Fused;
    out.push_back({v, TileConfig{shape.batch, shape.d_ff, shape.d_model}, c.label});
  }
  return out;
}

CandidateRunner make_runner(const KernelConfig& config) {
  return {config, [config](const Matrix& x, const MlpWeights& w, Matrix& a2) {
            check_input(x, w);
            check_stage1_output(x, w, a2);
            dfk_config c;
            if (gpu_config_for(config, x.rows(), w.shape.d_model, w.shape.d_ff, &c)) {
              gpu_stage1(&c, x, w.w_up, w.w_gate, &w.w_down, a2);
            } else {
              run_stage1(config.variant, x, w, a2, config.tile);
            }
          }};
}

std::vector<CandidateRunner> make_runners(const std::vector<KernelConfig>& configs) {
  std::vector<CandidateRunner> out;
  out.reserve(configs.size());
  for (const KernelConfig& c : configs) out.push_back(make_runner(c));
  return out;
}

std::vector<BenchmarkResult> profile(const std::vector<CandidateRunner>& cands,
                                     const MlpShape& shape, const ProfileOptions& opts) {
  if (opts.warmup < 1) throw std::invalid_argument("profile: warmup must be >= 1");
  if (opts.runs < 3) throw std::invalid_argument("profile: runs must be >= 3");
  shape.validate();
  // Seeded data, identical across candidates: X first, then the weights
  // (tuner.cpp:117-120 fill order).
  std::mt19937_64 rng(opts.seed);
  Matrix x(shape.batch, shape.d_model);
  fill_uniform(x, rng);
  const MlpWeights w = make_random_weights(shape, rng);
  Matrix ref(shape.batch, shape.d_ff);
  run_four_kernel_stage1(x, w, ref);  // the gate's reference (tuner.cpp:122-123)

  std::vector<BenchmarkResult> results;
  results.reserve(cands.size());
  for (const CandidateRunner& cand : cands) {
    BenchmarkResult res;
    res.config_label = cand.config.label;
    res.variant = cand.config.variant;
    res.warmup_runs = opts.warmup;
    Matrix a2(shape.batch, shape.d_ff);
    cand.stage1(x, w, a2);  // gate, unmeasured
    const double dev = rel_inf(a2, ref);
    if (!(dev <= kCorrectnessGateTolerance)) {
      std::ostringstream why;
      why << "output deviates from the four-kernel reference by " << dev
          << " relative (gate " << kCorrectnessGateTolerance << ")";
      res.disqualified = why.str();
      results.push_back(std::move(res));
      continue;
    }
    for (int i = 0; i < opts.warmup; ++i) cand.stage1(x, w, a2);
    for (int i = 0; i < opts.runs; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      cand.stage1(x, w, a2);
      const auto t1 = std::chrono::steady_clock::now();
      res.samples_ns.push_back(
          std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
    }
    res.measured_runs = opts.runs;
    std::vector<std::int64_t> s = res.samples_ns;
    std::sort(s.begin(), s.end());
    res.median_ns = s[(s.size() - 1) / 2];  // lower median (tuner.cpp:32-35)
    results.push_back(std::move(res));
  }
  return results;
}

std::vector<BenchmarkResult> profile(const std::vector<KernelConfig>& configs,
                                     const MlpShape& shape, const ProfileOptions& opts) {
  return profile(make_runners(configs), shape, opts);
}

ScheduleEntry select(const MlpShape& shape, const std::string& fingerprint,
                     const std::vector<BenchmarkResult>& results) {
  const BenchmarkResult* best = nullptr;
  const auto rank = [](const BenchmarkResult& r) {
    return std::make_tuple(r.median_ns, variant_rank(r.variant), std::cref(r.config_label));
  };
  for (const BenchmarkResult& r : results)
    if (!r.disqualified && (!best || rank(r) < rank(*best))) best = &r;
  if (!best)
    throw std::runtime_error("select: no candidate passed the correctness gate");
  return {shape, fingerprint, best->config_label, results, utc_now()};
}

void cache_store(const ScheduleEntry& entry, const std::filesystem::path& path) {
  const std::string text = entry_to_json(entry).dump();
  check(dfk_cache_store(path.c_str(), text.c_str()));
}

std::optional<ScheduleEntry> cache_lookup(const MlpShape& shape,
                                          const std::string& fingerprint,
                                          const std::filesystem::path& path) {
  size_t need = 0;
  int32_t found = 0;
  check(dfk_cache_lookup(path.c_str(), shape.batch, shape.d_model, shape.d_ff,
                         fingerprint.c_str(), nullptr, 0, &need, &found));
  if (!found) return std::nullopt;
  std::string buf(need, '\0');
  check(dfk_cache_lookup(path.c_str(), shape.batch, shape.d_model, shape.d_ff,
                         fingerprint.c_str(), buf.data(), buf.size(), &need, &found));
  if (!found) return std::nullopt;  // replaced between the two reads: a miss
  buf.resize(std::strlen(buf.c_str()));
  const json j = json::parse(buf, nullptr, false);
  if (j.is_discarded()) throw CacheError("tuning cache " + path.string() + ": bad entry");
  return entry_from_json(j, "tuning cache " + path.string());
}

std::string default_fingerprint() {
  char buf[256];
  std::lock_guard<std::mutex> lk(rt().mu);
  check(dfk_fingerprint(rt().context(0), buf, sizeof(buf)));
  return buf;
}

ScheduleEntry Tuner::get_or_tune(const MlpShape& shape,
                                 const std::vector<KernelConfig>& candidates) {
  if (!opts_.cache_path.empty()) {
    if (auto hit = cache_lookup(shape, opts_.fingerprint, opts_.cache_path)) {
      last_was_cache_hit_ = true;
      return *hit;
    }
  }
  last_was_cache_hit_ = false;
  ++profile_invocations_;
  ScheduleEntry e = select(shape, opts_.fingerprint, profile(candidates, shape, opts_.profile));
  if (!opts_.cache_path.empty()) cache_store(e, opts_.cache_path);
  return e;
}

ScheduleEntry tune_on_device(const MlpShape& shape, const MlpWeights& w,
                             const std::filesystem::path& cache_path, int warmup, int runs) {
  w.validate();
  if (shape.d_model != w.shape.d_model || shape.d_ff != w.shape.d_ff)
    throw ShapeError("tune_on_device: shape and weights disagree");
  if (warmup < 1) throw std::invalid_argument("profile: warmup must be >= 1");
  if (runs < 3) throw std::invalid_argument("profile: runs must be >= 3");
  Runtime& r = rt();
  std::lock_guard<std::mutex> lk(r.mu);
  dfk_weights h = weights_for_locked(&w.w_gate, &w.w_up, &w.w_down, 0, w.shape.d_ff);
  dfk_config chosen;
  int32_t hit = 0;
  std::string out(1 << 20, '\0');
  check(dfk_tune(r.context(0), h, shape.batch,
                 cache_path.empty() ? nullptr : cache_path.c_str(), warmup, runs, &chosen,
                 &hit, out.data(), out.size()));
  out.resize(std::strlen(out.c_str()));
  const json j = json::parse(out, nullptr, false);
  ScheduleEntry e;
  e.shape = shape;
  e.chosen = chosen.label;
  if (!j.is_discarded()) {
    e.fingerprint = j.value("fingerprint", std::string());
    e.created_at = j.value("created_at", std::string());
    for (const json& rj : j.value("results", json::array())) {
      BenchmarkResult b;
      b.config_label = rj.value("label", std::string());
      b.variant = variant_from_string(rj.value("variant", std::string("fused")))
                      .value_or(VariantTag::Fused);
      b.samples_ns = rj.value("samples_ns", std::vector<std::int64_t>{});
      b.median_ns = rj.value("median_ns", std::int64_t{0});
      b.warmup_runs = rj.value("warmup_runs", 0);
      b.measured_runs = rj.value("measured_runs", 0);
      if (rj.contains("disqualified")) b.disqualified = rj["disqualified"].get<std::string>();
      e.all_results.push_back(std::move(b));
    }
  }
  return e;
}

void release_gpu_cache() {
  Runtime& r = rt();
  std::lock_guard<std::mutex> lk(r.mu);
  for (auto& kv : r.lru) dfk_weights_destroy(kv.second);
  r.lru.clear();
}

// --- verification seam (verification.hpp:27-53) -----------------------------------
namespace verification {

std::optional<Mutant> mutant_from_string(std::string_view s) {
  if (s == "none") return Mutant::None;
  if (s == "silu-per-k-chunk") return Mutant::SiluPerKChunk;
  if (s == "materialize-intermediate") return Mutant::MaterializeIntermediate;
  return std::nullopt;
}

FusedStage1Fn fused_stage1_for(Mutant mutant) {
  switch (mutant) {
    case Mutant::None:
      return [](const Matrix& x, const Matrix& w_up, const Matrix& w_gate,
                const TileConfig& tile, Matrix& a2) {
        run_fused_stage1(x, w_up, w_gate, tile, a2);
      };
    case Mutant::SiluPerKChunk:
      return &fused_stage1_silu_per_k_chunk;
    case Mutant::MaterializeIntermediate:
      return &fused_stage1_materializing;
  }
  throw std::invalid_argument("unknown mutant");
}

void fused_stage1_silu_per_k_chunk(const Matrix& x, const Matrix& w_up,
                                   const Matrix& w_gate, const TileConfig& tile,
                                   Matrix& a2) {
  tile.validate();
  check_fused_stage1_args(x, w_up, w_gate, a2);
  const TileConfig t = tile.clamped({x.rows(), x.cols(), w_up.cols()});
  dfk_config c;
  std::memset(&c, 0, sizeof(c));
  c.variant = DFK_VARIANT_FUSED;
  c.s1_family = DFK_FAMILY_TC;
  c.down_family = DFK_FAMILY_TC;
  c.s1_split_k = 1;
  c.dynamic_sched = 1;
  c.s1_chunk_kb = static_cast<int32_t>(std::max<Index>(1, (t.tile_k + 63) / 64));
  c.mutant = 1;
  gpu_stage1(&c, x, w_up, w_gate, nullptr, a2);
}

void fused_stage1_materializing(const Matrix& x, const Matrix& w_up, const Matrix& w_gate,
                                const TileConfig& tile, Matrix& a2) {
  tile.validate();
  check_fused_stage1_args(x, w_up, w_gate, a2);
  dfk_config c;
  std::memset(&c, 0, sizeof(c));
  c.variant = DFK_VARIANT_FUSED;
  c.s1_family = DFK_FAMILY_TC;
  c.down_family = DFK_FAMILY_TC;
  c.s1_split_k = 1;
  c.mutant = 2;
  gpu_stage1(&c, x, w_up, w_gate, nullptr, a2);
}

double max_abs_diff(const Matrix& a, const Matrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols())
    throw ShapeError("max_abs_diff: shapes differ");
  double m = 0.0;
  for (Index i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a.data()[i] - b.data()[i]));
  return m;
}

}  // namespace verification

}  // namespace deepfusion
