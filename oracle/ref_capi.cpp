// ref_capi.cpp — extern "C" wrapper over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// /root/reference/proj/src/*.cpp (in place, never copied) into
// oracle/_ref/libdeepfusion_ref.so.  It lets Python drive the reference's own
// code path for (a) pinning the C restatement in oracle/dfk_oracle.c, (b) the
// golden vectors in tests/golden/, and (c) bench.py --impl reference (the
// reference CPU path timed on the GPU box's host cores).
//
// Every entry point returns 0 on success, 2 on deepfusion::ShapeError /
// std::invalid_argument (the reference CLI's exit-2 class, tools/main.cpp:
// 377-389) and 1 on any other exception; the message is kept in
// dfr_last_error().
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "deepfusion/fused.hpp"
#include "deepfusion/swiglu.hpp"
#include "deepfusion/tensor.hpp"
#include "deepfusion/tp.hpp"
#include "deepfusion/traffic.hpp"
#include "deepfusion/tuner.hpp"
#include "deepfusion/verification.hpp"

using namespace deepfusion;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {  // includes ShapeError
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

Matrix from_ptr(const double* p, std::int64_t r, std::int64_t c) {
  Matrix m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

void to_ptr(const Matrix& m, double* p) {
  std::memcpy(p, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
}

struct Instance {
  Matrix x;
  MlpWeights w;
};

TileConfig tile_of(std::int64_t tm, std::int64_t tn, std::int64_t tk,
                   int col_major) {
  return TileConfig{tm, tn, tk,
                    col_major ? LoopOrder::ColumnMajorTiling
                              : LoopOrder::RowMajorTiling};
}

}  // namespace

extern "C" {

const char* dfr_last_error() { return g_err.c_str(); }

double dfr_silu(double x) { return silu(x); }
double dfr_sigmoid(double x) { return sigmoid(x); }

// The reference's own generator (make_random_weights then fill_uniform(x)).
int dfr_make_instance(std::uint64_t seed, std::int64_t B, std::int64_t dm,
                      std::int64_t df, double scale, double* x, double* w_up,
                      double* w_gate, double* w_down) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    MlpWeights w = make_random_weights({B, dm, df}, rng, scale);
    Matrix xm(B, dm);
    fill_uniform(xm, rng);
    to_ptr(xm, x);
    to_ptr(w.w_up, w_up);
    to_ptr(w.w_gate, w_gate);
    to_ptr(w.w_down, w_down);
  });
}

// Instance handle: Matrices built once, so timed calls exclude the copy-in.
void* dfr_instance_create(std::int64_t B, std::int64_t dm, std::int64_t df,
                          const double* x, const double* w_up,
                          const double* w_gate, const double* w_down) {
  try {
    auto* inst = new Instance{from_ptr(x, B, dm),
                              MlpWeights{from_ptr(w_up, dm, df),
                                         from_ptr(w_gate, dm, df),
                                         from_ptr(w_down, df, dm),
                                         MlpShape{B, dm, df}}};
    return inst;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void dfr_instance_destroy(void* h) { delete static_cast<Instance*>(h); }

// run_fused (fused.cpp:209-216) with an explicit tile and worker count.
int dfr_run_fused(void* h, std::int64_t tm, std::int64_t tn, std::int64_t tk,
                  int col_major, int num_workers, double* y) {
  return guarded([&] {
    auto* inst = static_cast<Instance*>(h);
    to_ptr(run_fused(inst->x, inst->w, tile_of(tm, tn, tk, col_major),
                     num_workers),
           y);
  });
}

// run_fused_stage1 (fused.cpp:172-207).
int dfr_run_fused_stage1(void* h, std::int64_t tm, std::int64_t tn,
                         std::int64_t tk, int col_major, int num_workers,
                         double* a2) {
  return guarded([&] {
    auto* inst = static_cast<Instance*>(h);
    Matrix out(inst->w.shape.batch, inst->w.shape.d_ff);
    run_fused_stage1(inst->x, inst->w.w_up, inst->w.w_gate,
                     tile_of(tm, tn, tk, col_major), out, num_workers);
    to_ptr(out, a2);
  });
}

// run_variant (fused.cpp:258-264): variant 0=four, 1=two, 2=fused.
int dfr_run_variant(void* h, int variant, std::int64_t tm, std::int64_t tn,
                    std::int64_t tk, int col_major, double* y) {
  return guarded([&] {
    auto* inst = static_cast<Instance*>(h);
    KernelConfig cfg{static_cast<VariantTag>(variant),
                     tile_of(tm, tn, tk, col_major), "capi"};
    to_ptr(run_variant(cfg, inst->x, inst->w), y);
  });
}

// down_projection (swiglu.cpp:214-226).
int dfr_down_projection(const double* a2, std::int64_t B, std::int64_t df,
                        const double* w_down, std::int64_t dm, double* y) {
  return guarded([&] {
    to_ptr(down_projection(from_ptr(a2, B, df), from_ptr(w_down, df, dm)), y);
  });
}

// oracle_stage1 / oracle_forward (verification.cpp:171-202).
int dfr_oracle_forward(void* h, double* a2, double* y) {
  return guarded([&] {
    auto* inst = static_cast<Instance*>(h);
    if (a2) to_ptr(verification::oracle_stage1(inst->x, inst->w), a2);
    if (y) to_ptr(verification::oracle_forward(inst->x, inst->w), y);
  });
}

// run_tp_mlp (tp.cpp:140-167) with the compound scheme; returns the number
// of collective events and the payload of the first in *events/*payload.
int dfr_run_tp_mlp(void* h, std::int64_t devices, int variant, double* y,
                   std::int64_t* events, std::int64_t* payload) {
  return guarded([&] {
    auto* inst = static_cast<Instance*>(h);
    const MlpShape& s = inst->w.shape;
    KernelConfig cfg{static_cast<VariantTag>(variant),
                     TileConfig{s.batch, s.d_ff, s.d_model,
                                LoopOrder::ColumnMajorTiling},
                     "capi"};
    TpResult r = run_tp_mlp(inst->x, inst->w, make_plan(s.d_ff, devices), cfg);
    to_ptr(r.output, y);
    *events = static_cast<std::int64_t>(r.log.events.size());
    *payload = r.log.events.empty()
                   ? 0
                   : static_cast<std::int64_t>(
                         r.log.events.front().payload_elements_per_device);
  });
}

int dfr_balanced_ranges(std::int64_t extent, std::int64_t parts,
                        std::int64_t* begins, std::int64_t* ends) {
  return guarded([&] {
    const auto rs = balanced_ranges(extent, parts);
    for (size_t i = 0; i < rs.size(); ++i) {
      begins[i] = rs[i].begin;
      ends[i] = rs[i].end;
    }
  });
}

// predict_traffic total bytes (traffic.cpp:96-103) for the fused variant
// with a single covering column-major tile.
std::uint64_t dfr_fused_block_bytes(std::int64_t B, std::int64_t dm,
                                    std::int64_t df, std::uint64_t bpe) {
  const MlpShape s{B, dm, df};
  return predict_traffic(VariantTag::Fused, s,
                         TileConfig{B, df, dm, LoopOrder::ColumnMajorTiling},
                         bpe)
      .total_bytes();
}

// Reference candidate grid size (tuner.cpp:59-88), for scheduler parity.
std::int64_t dfr_default_candidate_count(std::int64_t B, std::int64_t dm,
                                         std::int64_t df) {
  return static_cast<std::int64_t>(default_candidates({B, dm, df}).size());
}

}  // extern "C"
