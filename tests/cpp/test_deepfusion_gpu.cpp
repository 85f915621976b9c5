// test_deepfusion_gpu.cpp — the reference's own unit tests for the operator
// API, restated against the drop-in C++ shim (deepfusion.hpp ->
// libdeepfusion_b200.so -> libdfk.so).  Exact checks stay exact where bf16
// represents the values; numeric checks use the bf16 gate
// max|dY| / max|Y_ref| <= 1e-2 against an independent fp64 triple loop
// (the reference oracle, verification.cpp:171-202).  Run by
// tests/test_cpp_shim.py (-m gpu).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "deepfusion.hpp"

using namespace deepfusion;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, \
                   #cond);                                                 \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, T)   \
  do {                             \
    bool thrown = false;           \
    try {                          \
      (void)(expr);                \
    } catch (const T&) {           \
      thrown = true;               \
    }                              \
    CHECK(thrown && #T);           \
  } while (0)

static std::vector<std::pair<const char*, std::function<void()>>>& registry() {
  static std::vector<std::pair<const char*, std::function<void()>>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, f}); }
};
#define TEST_CASE(name, fn) static void fn(); static Reg reg_##fn(name, fn); static void fn()

// Independent fp64 oracle (verification.cpp:171-202).
static Matrix oracle_forward(const Matrix& x, const MlpWeights& w) {
  const Index B = x.rows(), dm = w.shape.d_model, df = w.shape.d_ff;
  Matrix a2(B, df), y(B, dm);
  for (Index i = 0; i < B; ++i)
    for (Index j = 0; j < df; ++j) {
      double g = 0, u = 0;
      for (Index p = 0; p < dm; ++p) {
        g += x(i, p) * w.w_gate(p, j);
        u += x(i, p) * w.w_up(p, j);
      }
      a2(i, j) = u * (g / (1.0 + std::exp(-g)));
    }
  for (Index i = 0; i < B; ++i)
    for (Index j = 0; j < dm; ++j) {
      double acc = 0;
      for (Index f = 0; f < df; ++f) acc += a2(i, f) * w.w_down(f, j);
      y(i, j) = acc;
    }
  return y;
}

static double rel_err(const Matrix& a, const Matrix& ref) {
  double num = 0, den = 0;
  for (Index i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a.data()[i] - ref.data()[i]));
    den = std::max(den, std::abs(ref.data()[i]));
  }
  return den > 0 ? num / den : num;
}

static void round_bf16(Matrix& m) {  // inputs exactly representable on GPU
  for (Index i = 0; i < m.size(); ++i) {
    float f = static_cast<float>(m.data()[i]);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    std::memcpy(&f, &u, 4);
    m.data()[i] = f;
  }
}

struct Instance {
  Matrix x;
  MlpWeights w;
};

static Instance random_instance(const MlpShape& shape, std::uint64_t seed,
                                double scale = 1.0) {
  std::mt19937_64 rng(seed);
  Instance inst{Matrix(shape.batch, shape.d_model),
                make_random_weights(shape, rng, scale)};
  fill_uniform(inst.x, rng);
  round_bf16(inst.x);
  round_bf16(inst.w.w_up);
  round_bf16(inst.w.w_gate);
  round_bf16(inst.w.w_down);
  return inst;
}

static MlpWeights weights_from(const MlpShape& s, std::vector<double> up,
                               std::vector<double> gate, std::vector<double> down) {
  MlpWeights w{Matrix(s.d_model, s.d_ff), Matrix(s.d_model, s.d_ff),
               Matrix(s.d_ff, s.d_model), s};
  for (Index i = 0; i < w.w_up.size(); ++i) w.w_up.data()[i] = up[static_cast<size_t>(i)];
  for (Index i = 0; i < w.w_gate.size(); ++i) w.w_gate.data()[i] = gate[static_cast<size_t>(i)];
  for (Index i = 0; i < w.w_down.size(); ++i) w.w_down.data()[i] = down[static_cast<size_t>(i)];
  return w;
}

// test_swiglu.cpp:65-76 / test_fused.cpp:179-189
TEST_CASE("scalar brute-force case: 6 * silu(2)", t_scalar) {
  const MlpShape shape{1, 1, 1};
  MlpWeights w = weights_from(shape, {3}, {1}, {1});
  Matrix x(1, 1);
  x(0, 0) = 2.0;
  const double expected = 6.0 * silu(2.0);
  CHECK(std::abs(expected - 10.5696) < 1e-4);
  for (const Matrix& y : {run_four_kernel(x, w), run_two_kernel(x, w),
                          run_fused(x, w, {1, 1, 1, LoopOrder::ColumnMajorTiling})}) {
    CHECK(std::abs(y(0, 0) - expected) / expected < 2e-3);  // A2 rounds to bf16
  }
}

// test_swiglu.cpp:46-63
TEST_CASE("zero input and zero gate give exact zeros", t_zero) {
  const MlpShape shape{1, 3, 4};
  std::mt19937_64 rng(3);
  MlpWeights w = make_random_weights(shape, rng);
  Matrix x(1, 3);
  for (const Matrix& y : {run_four_kernel(x, w), run_two_kernel(x, w), run_fused(x, w, {})})
    for (Index j = 0; j < 3; ++j) CHECK(y(0, j) == 0.0);
  MlpWeights g0 = weights_from({1, 2, 2}, {1, 1, 1, 1}, {0, 0, 0, 0}, {1, 0, 0, 1});
  Matrix x2(1, 2);
  x2(0, 0) = 1.0;
  const Matrix y = run_fused(x2, g0, {});
  CHECK(y(0, 0) == 0.0 && y(0, 1) == 0.0);
}

// test_swiglu.cpp:94-113
TEST_CASE("down_projection basics", t_down) {
  Matrix a2(1, 2);
  a2(0, 0) = 2.0;
  a2(0, 1) = 3.0;
  Matrix w_down(2, 1);
  w_down(0, 0) = 4.0;
  w_down(1, 0) = 5.0;
  CHECK(down_projection(a2, w_down)(0, 0) == 23.0);
  const Matrix same = down_projection(a2, Matrix::identity(2));
  CHECK(same(0, 0) == 2.0 && same(0, 1) == 3.0);
  Matrix zeros(3, 2);
  const Matrix z = down_projection(zeros, w_down);
  CHECK(z(0, 0) == 0.0 && z(2, 0) == 0.0);
  Matrix bad(3, 1);
  CHECK_THROWS_AS(down_projection(a2, bad), ShapeError);
}

// verification.cpp:217-254 (criterion 1), bf16 gate.
TEST_CASE("variant equivalence vs oracle on randomized instances", t_variants) {
  std::mt19937_64 rng(20260809);
  double worst = 0;
  for (int trial = 0; trial < 40; ++trial) {
    const MlpShape shape{1 + static_cast<Index>(rng() % 8), 2 + static_cast<Index>(rng() % 63),
                         2 + static_cast<Index>(rng() % 63)};
    Instance inst = random_instance(shape, rng());
    const Matrix expected = oracle_forward(inst.x, inst.w);
    worst = std::max(worst, rel_err(run_four_kernel(inst.x, inst.w), expected));
    worst = std::max(worst, rel_err(run_two_kernel(inst.x, inst.w), expected));
    worst = std::max(worst, rel_err(run_fused(inst.x, inst.w, {2, 3, 4, LoopOrder::RowMajorTiling}), expected));
    Matrix a2(shape.batch, shape.d_ff);
    run_fused_stage1(inst.x, inst.w.w_up, inst.w.w_gate, {1, 32, 32}, a2);
    worst = std::max(worst, rel_err(down_projection(a2, inst.w.w_down), expected));
  }
  std::printf("  variant equivalence: worst rel err %.3e\n", worst);
  CHECK(worst <= 1e-2);
}

// verification.cpp:278-308 (criterion 2): tiling invariance.
TEST_CASE("tiling invariance (tile is a hint)", t_tiling) {
  Instance inst = random_instance({5, 13, 17}, 20260809);
  const Matrix base = run_fused(inst.x, inst.w, {5, 17, 13});
  for (const TileConfig& t : {TileConfig{1, 1, 1}, TileConfig{2, 4, 3, LoopOrder::RowMajorTiling},
                              TileConfig{5, 7, 13}}) {
    const Matrix y = run_fused(inst.x, inst.w, t);
    for (Index i = 0; i < y.size(); ++i) CHECK(y.data()[i] == base.data()[i]);
  }
}

// test_tp.cpp:74-112
TEST_CASE("TP equivalence across device counts, one all-reduce", t_tp) {
  Instance inst = random_instance({3, 6, 12}, 71);
  const Matrix expected = oracle_forward(inst.x, inst.w);
  for (Index p : {1, 2, 3, 4, 8}) {
    for (VariantTag v : {VariantTag::FourKernel, VariantTag::TwoKernel, VariantTag::Fused}) {
      const TpResult r = run_tp_mlp(inst.x, inst.w, make_plan(12, p), {v, {}, "tp"});
      CHECK(rel_err(r.output, expected) <= 1e-2);
      CHECK(r.log.events.size() == 1);
      CHECK(r.log.events[0].payload_elements_per_device == 3 * 6);
    }
  }
  Instance u = random_instance({2, 4, 7}, 73);
  const TpResult r = run_tp_mlp(u.x, u.w, make_plan(7, 3), {VariantTag::TwoKernel, {}, ""});
  Matrix a2(2, 7);
  run_two_kernel_stage1(u.x, u.w, a2);
  Index col = 0;
  for (const Matrix& shard : r.stage1_shards) {
    for (Index i = 0; i < 2; ++i)
      for (Index j = 0; j < shard.cols(); ++j)
        CHECK(std::abs(shard(i, j) - a2(i, col + j)) <= 1e-2 * (1 + std::abs(a2(i, col + j))));
    col += shard.cols();
  }
  CHECK(col == 7);
}

// The same equivalence on a shape the fused all-reduce takes (d_model % 4
// == 0): run_tp_mlp's ranks reduce partial Y over peer memory inside the
// block kernel (P contexts on one GPU when fewer devices are visible).
TEST_CASE("TP equivalence with the in-kernel all-reduce", t_tp_fused) {
  Instance inst = random_instance({5, 256, 900}, 79);
  const Matrix expected = oracle_forward(inst.x, inst.w);
  for (Index p : {2, 3, 4, 8}) {
    const TpResult r = run_tp_mlp(inst.x, inst.w, make_plan(900, p), {VariantTag::Fused, {}, "tp"});
    CHECK(rel_err(r.output, expected) <= 1e-2);
    CHECK(r.log.events.size() == 1);
    CHECK(static_cast<Index>(r.stage1_shards.size()) == p);
  }
}

// test_tp.cpp:39-58, tp.cpp:8-29
TEST_CASE("make_plan splits evenly and spreads the remainder", t_plan) {
  const ShardPlan even = make_plan(8, 4);
  CHECK(even.ff_ranges.size() == 4 && even.ff_ranges[1] == (ColRange{2, 4}));
  const ShardPlan odd = make_plan(7, 3);
  CHECK(odd.ff_ranges[0] == (ColRange{0, 3}) && odd.ff_ranges[2] == (ColRange{5, 7}));
  CHECK_THROWS_AS(make_plan(3, 4), ShapeError);
  CHECK_THROWS_AS(make_plan(3, 0), ShapeError);
  ShardPlan bad{2, {{0, 3}, {4, 8}}};
  CHECK_THROWS_AS(bad.validate(8), ShapeError);
}

// fused.cpp:16-68 validation
TEST_CASE("shape errors mirror the reference", t_errors) {
  Instance inst = random_instance({2, 3, 4}, 5);
  Matrix a2(2, 4);
  CHECK_THROWS_AS(run_fused_stage1(inst.x, inst.w.w_up, inst.w.w_gate, {0, 1, 1}, a2), ShapeError);
  Matrix wrong(3, 4);
  CHECK_THROWS_AS(run_fused_stage1(inst.x, inst.w.w_up, inst.w.w_gate, {1, 1, 1}, wrong), ShapeError);
  CHECK_THROWS_AS(Matrix(0, 3), ShapeError);
  MlpWeights w = inst.w;
  w.shape.d_ff = 5;
  CHECK_THROWS_AS(run_fused(inst.x, w, {}), ShapeError);
  CHECK_THROWS_AS(MlpShape({0, 1, 1}).validate(), ShapeError);
}

// tensor.cpp:151-163: generator is bit-stable
TEST_CASE("fill_uniform is deterministic and in range", t_fill) {
  std::mt19937_64 a(9), b(9);
  Matrix m1(4, 5), m2(4, 5);
  fill_uniform(m1, a);
  fill_uniform(m2, b);
  for (Index i = 0; i < m1.size(); ++i) {
    CHECK(m1.data()[i] == m2.data()[i]);
    CHECK(m1.data()[i] >= -1.0 && m1.data()[i] < 1.0);
  }
}

// The library's on-device scheduler through the shim (dfk_tune): a second
// call with the same shape and cache file is a cache hit.
TEST_CASE("tune_on_device: warm cache skips profiling", t_tuner) {
  Instance inst = random_instance({4, 256, 512}, 7, 1.0 / 16);
  const std::string path = std::string(std::getenv("DFK_TEST_TMP") ? std::getenv("DFK_TEST_TMP") : "/tmp") +
                           "/dfk_cpp_tuner_cache.json";
  std::remove(path.c_str());
  const ScheduleEntry e1 = tune_on_device({4, 256, 512}, inst.w, path, 1, 3);
  CHECK(!e1.chosen.empty() && e1.all_results.size() > 3);
  for (const BenchmarkResult& r : e1.all_results)
    if (!r.disqualified) CHECK(r.samples_ns.size() == 3 && r.median_ns > 0);
  const ScheduleEntry e2 = tune_on_device({4, 256, 512}, inst.w, path, 1, 3);
  CHECK(e2.chosen == e1.chosen);
  CHECK(!default_fingerprint().empty());
  // the chosen configuration runs through the reference entry point
  const Matrix y = run_variant({VariantTag::Fused, {}, e1.chosen}, inst.x, inst.w);
  CHECK(rel_err(y, oracle_forward(inst.x, inst.w)) <= 1e-2);
  std::remove(path.c_str());
}

// The weight-pack cache keys on the matrices' exact contents: an in-place
// edit (same storage, same shape) is seen by the next call.
TEST_CASE("in-place weight edits are never served a stale GPU pack", t_stale) {
  Instance inst = random_instance({3, 128, 384}, 11, 1.0 / 8);
  const Matrix y0 = run_fused(inst.x, inst.w, {});
  CHECK(rel_err(y0, oracle_forward(inst.x, inst.w)) <= 1e-2);
  for (Index i = 0; i < inst.w.w_down.size(); ++i) inst.w.w_down.data()[i] *= -0.5;
  const Matrix y1 = run_fused(inst.x, inst.w, {});
  CHECK(rel_err(y1, oracle_forward(inst.x, inst.w)) <= 1e-2);
  inst.w.w_up(5, 7) = 3.0;  // one element, through operator()
  Matrix a2(3, 384), a2b(3, 384);
  run_fused_stage1(inst.x, inst.w.w_up, inst.w.w_gate, {}, a2);
  run_two_kernel_stage1(inst.x, inst.w, a2b);
  CHECK(rel_err(a2, a2b) <= 1e-2);
  // stage-only sets: the down projection alone, same matrix reused
  const Matrix y2 = down_projection(a2b, inst.w.w_down);
  CHECK(rel_err(y2, oracle_forward(inst.x, inst.w)) <= 2e-2);
}

// fused.cpp:218-239
TEST_CASE("predicted_reuse_counts: weights once in column-major order", t_reuse) {
  const ReuseCounts col = predicted_reuse_counts({4, 8, 16}, {4, 4, 8, LoopOrder::ColumnMajorTiling});
  CHECK(col.x_reads == 4u * 8u * 4u && col.weight_reads == 2u * 8u * 16u && col.a2_writes == 64u);
  const ReuseCounts row = predicted_reuse_counts({4, 8, 16}, {2, 16, 8, LoopOrder::RowMajorTiling});
  CHECK(row.x_reads == 32u && row.weight_reads == 2u * 8u * 16u * 2u);
}

// verification.hpp:27-53: the injectable fused stage 1 and its mutants.
TEST_CASE("verification seam: mutants deviate, the product does not", t_mutants) {
  Instance inst = random_instance({4, 512, 384}, 13, 1.0 / 16);
  Matrix ref(4, 384);
  run_two_kernel_stage1(inst.x, inst.w, ref);
  using namespace verification;
  CHECK(mutant_from_string("silu-per-k-chunk") == Mutant::SiluPerKChunk);
  CHECK(!mutant_from_string("bogus").has_value());
  const TileConfig tile{4, 64, 128};
  Matrix a(4, 384), b(4, 384), c(4, 384);
  fused_stage1_for(Mutant::None)(inst.x, inst.w.w_up, inst.w.w_gate, tile, a);
  fused_stage1_for(Mutant::SiluPerKChunk)(inst.x, inst.w.w_up, inst.w.w_gate, tile, b);
  fused_stage1_for(Mutant::MaterializeIntermediate)(inst.x, inst.w.w_up, inst.w.w_gate, tile, c);
  CHECK(rel_err(a, ref) <= 1e-2);
  CHECK(rel_err(b, ref) > 5e-2);   // SiLU per K chunk: numerics break
  CHECK(rel_err(c, ref) <= 1e-2);  // materialising: numerics intact (traffic trips)
  CHECK(max_abs_diff(a, a) == 0.0);
}

int main() {
  for (auto& [name, fn] : registry()) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "%s: unexpected exception: %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
