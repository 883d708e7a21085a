// persyn_gpu.hpp — C++ binding of the B200 hot path for code built against
// the reference's own headers (proj/core/include/persyn): the drop-in a
// maintainer adds to the reference.
//
//  * persyn::gpu::GpuSearchIndex IS a persyn::SearchIndex (optimizer.hpp:
//    111-119): the reference's optimize_level / search_step / compare code
//    accepts it unchanged; nearest() answers one query on the device (the
//    reference's per-query plug-in granularity — correct, but slow).
//  * persyn::gpu::search_step / update_step / optimize_level take and return
//    the reference's types and run the batched device path (the fast path).
//  * psg_status codes are rethrown as the reference's exceptions
//    (errors.hpp:8-36, std::logic_error for invariants).
//
// Header-only over the C ABI (persyn_b200.h); link libpersyn_b200.so.
#pragma once

#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "persyn/errors.hpp"
#include "persyn/neighborhood.hpp"
#include "persyn/optimizer.hpp"
#include "persyn_b200.h"

namespace persyn::gpu {

inline void check(psg_status s) {
  if (s == PSG_OK) return;
  const std::string m = psg_last_error();
  switch (s) {
    case PSG_E_DOMAIN: throw persyn::DomainError(m);
    case PSG_E_SHAPE: throw persyn::ShapeError(m);
    case PSG_E_LOGIC: throw std::logic_error(m);
    case PSG_E_IO: throw persyn::IoError(m);
    case PSG_E_FORMAT: throw persyn::FormatError(m);
    default: throw persyn::Error(m);
  }
}

// One device + stream; owns cuBLAS/cuSOLVER handles and the memory pool.
class Context {
 public:
  explicit Context(int device = 0) { check(psg_ctx_create(device, nullptr, &ctx_)); }
  ~Context() { psg_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  psg_ctx* get() const { return ctx_; }

 private:
  psg_ctx* ctx_ = nullptr;
};

// RgbsImage (image.hpp:68-95) <-> planar [4][H][W] fp64, row 0 = bottom.
inline std::vector<double> planes_of(const RgbsImage& img) {
  const std::size_t P = static_cast<std::size_t>(img.width()) * img.height();
  std::vector<double> out(4 * P);
  for (int c = 0; c < 3; ++c) {
    const auto pl = img.base().plane(c);
    std::copy(pl.begin(), pl.end(), out.begin() + c * P);
  }
  const auto s = img.scale_plane();
  std::copy(s.begin(), s.end(), out.begin() + 3 * P);
  return out;
}

inline RgbsImage image_of(const double* planes, int W, int H) {
  const std::size_t P = static_cast<std::size_t>(W) * H;
  RasterImage base(W, H);
  for (int c = 0; c < 3; ++c) std::copy(planes + c * P, planes + (c + 1) * P, base.plane(c).begin());
  return RgbsImage(std::move(base), std::vector<double>(planes + 3 * P, planes + 4 * P));
}

inline psg_budget to_budget(const QueryBudget& b) {
  psg_budget r{};
  r.mode = b.mode == QueryBudget::Mode::kGreedy   ? PSG_GREEDY
           : b.mode == QueryBudget::Mode::kExact ? PSG_EXACT
                                                 : PSG_BACKTRACK;
  r.max_leaves = b.max_leaves;
  return r;
}

// HistogramSet (optimizer.hpp:55-75) -> [slots][bins] masses.
inline std::vector<double> masses_of(const HistogramSet& h) {
  std::vector<double> m;
  for (std::size_t s = 0; s < h.channel_ids().size(); ++s)
    for (int b = 0; b < h.bins(); ++b) m.push_back(h.mass(s, b));
  return m;
}

class GpuSearchIndex final : public SearchIndex {
 public:
  // make_pca_tree_index(extract_all(exemplar, {w, 1, ..}), variance,
  // branching, seed) (optimizer.cpp:256-262): PCA fit and projection on the
  // device, and the reference's own KmTree::build (km_tree.cpp:141-195,
  // replayed with the same mt19937_64 stream: greedy / backtrack answers are
  // the reference's for the same PCA model); d_cap > 0 caps the retained
  // dimension; tree_kind = PSG_TREE_DEVICE builds the device tree instead.
  static std::unique_ptr<GpuSearchIndex> pca_tree(Context& ctx, const RgbsImage& exemplar, int w,
                                                  double variance_target = 0.95,
                                                  int branching = 4, std::uint64_t seed = 0,
                                                  int d_cap = 0, int hist_bins = 16,
                                                  int tree_kind = PSG_TREE_REFERENCE) {
    psg_index_cfg cfg{};
    cfg.variance_target = variance_target;
    cfg.d_cap = d_cap;
    cfg.branching = branching;
    cfg.seed = seed;
    cfg.hist_bins = hist_bins;
    cfg.tree_kind = tree_kind;
    const auto planes = planes_of(exemplar);
    psg_index* h = nullptr;
    check(psg_index_create(ctx.get(), planes.data(), 4, exemplar.width(), exemplar.height(), w,
                           nullptr, nullptr, 0, &cfg, &h));
    return std::unique_ptr<GpuSearchIndex>(new GpuSearchIndex(ctx, h, exemplar, w, "pca-tree"));
  }

  // make_brute_force_index(extract_all(exemplar, {w, 1, ..})) (optimizer.cpp:168-212).
  static std::unique_ptr<GpuSearchIndex> brute_force(Context& ctx, const RgbsImage& exemplar,
                                                     int w, int hist_bins = 16) {
    const auto planes = planes_of(exemplar);
    psg_index* h = nullptr;
    check(psg_index_create_brute(ctx.get(), planes.data(), 4, exemplar.width(),
                                 exemplar.height(), w, hist_bins, 0, &h));
    return std::unique_ptr<GpuSearchIndex>(new GpuSearchIndex(ctx, h, exemplar, w, "brute-force"));
  }

  ~GpuSearchIndex() override { psg_index_destroy(index_); }

  QueryResult nearest(std::span<const float> query, const QueryBudget& budget) const override {
    QueryResult r;
    std::int32_t idx = -1;
    double dist = 0.0;
    std::int64_t scanned = 0;
    check(psg_index_query(ctx_->get(), index_, query.data(), 1, to_budget(budget), &idx, &dist,
                          nullptr, &scanned));
    r.index = idx;
    r.distance = dist;
    r.stats.points_scanned = scanned;
    return r;
  }

  // The dense window matrix the reference keeps (materialised on first use:
  // the device index never needs it).
  const NeighborhoodMatrix& candidates() const override {
    if (!cand_) cand_ = std::make_unique<NeighborhoodMatrix>(
                     extract_all(exemplar_, GridSpec{w_, 1, exemplar_.width(), exemplar_.height()}));
    return *cand_;
  }

  std::string describe() const override { return kind_ + " (B200)"; }
  psg_index* handle() const { return index_; }
  psg_ctx* ctx() const { return ctx_->get(); }
  int window() const { return w_; }

 private:
  GpuSearchIndex(Context& ctx, psg_index* h, const RgbsImage& ex, int w, std::string kind)
      : ctx_(&ctx), index_(h), exemplar_(ex), w_(w), kind_(std::move(kind)) {}
  Context* ctx_;
  psg_index* index_;
  RgbsImage exemplar_;
  int w_;
  std::string kind_;
  mutable std::unique_ptr<NeighborhoodMatrix> cand_;
};

inline psg_opt_cfg to_cfg(const OptimizerConfig& c) {
  psg_opt_cfg r{};
  r.robust_exponent = c.robust_exponent;
  r.distance_epsilon = c.distance_epsilon;
  r.max_iterations = c.max_iterations;
  r.min_iterations = c.min_iterations;
  r.convergence_fraction = c.convergence_fraction;
  r.histogram_bins = c.histogram_bins;
  r.histogram_matching = c.histogram_matching;
  r.histogram_include_scale = c.histogram_include_scale;
  r.spacing = c.grid.spacing;
  r.patch_width = c.patch.patch_width;
  r.budget = to_budget(c.budget);
  return r;
}

// search_step (optimizer.hpp:141-143), batched on the device.
inline SearchOutcome search_step(const RgbsImage& out, const GpuSearchIndex& index,
                                 const SparseGrid& grid, const PatchSpec& patch,
                                 const QueryBudget& budget) {
  if (grid.spec.image_width != out.width() || grid.spec.image_height != out.height())
    throw ShapeError("grid does not match the output image");
  if (grid.spec.nbhd_width != index.window())
    throw ShapeError("candidate dim does not match the grid window");
  const auto planes = planes_of(out);
  SearchOutcome o;
  o.assignments.input_index.resize(static_cast<std::size_t>(grid.count()));
  o.assignments.distance.resize(static_cast<std::size_t>(grid.count()));
  check(psg_search_step(index.ctx(), index.handle(), planes.data(), out.width(), out.height(),
                        grid.spec.spacing, patch.patch_width, to_budget(budget),
                        o.assignments.input_index.data(), o.assignments.distance.data(),
                        &o.nn_calls, &o.points_scanned));
  return o;
}

// update_step (optimizer.hpp:149-151).
inline RgbsImage update_step(const AssignmentMap& assignments, const WeightMap& weights,
                             const SparseGrid& grid, const GpuSearchIndex& index,
                             const RgbsImage& out) {
  const std::size_t A = static_cast<std::size_t>(grid.count());
  if (assignments.size() != A || weights.size() != A)
    throw ShapeError("assignments/weights do not cover the grid");
  std::vector<double> planes(4 * static_cast<std::size_t>(out.width()) * out.height());
  check(psg_update_step(index.ctx(), index.handle(), assignments.input_index.data(),
                        weights.irls.data(), weights.hist_penalty.data(), out.width(), out.height(),
                        grid.spec.spacing, planes.data()));
  return image_of(planes.data(), out.width(), out.height());
}

// optimize_level (optimizer.hpp:181-183): the whole EM loop on the device.
inline LevelResult optimize_level(const RgbsImage& init, const GpuSearchIndex& index,
                                  const OptimizerConfig& cfg,
                                  const HistogramSet* exemplar_hist = nullptr) {
  cfg.validate();
  if (cfg.grid.image_width != init.width() || cfg.grid.image_height != init.height())
    throw ShapeError("grid does not match the initial image");
  const psg_opt_cfg c = to_cfg(cfg);
  const auto planes = planes_of(init);
  std::vector<double> masses;
  if (exemplar_hist && cfg.histogram_matching) {
    // HistogramSet::compatible (optimizer.cpp:65-67, thrown at :93-95): the
    // library reads bins x (3 or 4) masses in the output set's channel order
    std::vector<int> ids{0, 1, 2};
    if (cfg.histogram_include_scale) ids.push_back(3);
    if (exemplar_hist->bins() != cfg.histogram_bins || exemplar_hist->channel_ids() != ids)
      throw ShapeError("output/exemplar histograms disagree on bins or channels");
  }
  if (exemplar_hist) masses = masses_of(*exemplar_hist);
  std::vector<psg_iter_stats> st(static_cast<std::size_t>(cfg.max_iterations));
  std::vector<double> out(planes.size());
  int n = 0;
  // the reference applies histogram matching only with an exemplar histogram
  psg_opt_cfg cc = c;
  cc.histogram_matching = c.histogram_matching && exemplar_hist != nullptr;
  check(psg_optimize_level(index.ctx(), index.handle(), planes.data(), init.width(), init.height(),
                           &cc, exemplar_hist ? masses.data() : nullptr, out.data(), st.data(),
                           &n));
  LevelResult r{image_of(out.data(), init.width(), init.height()), {}};
  for (int i = 0; i < n; ++i) {
    IterationStats it;
    it.iteration = st[i].iteration;
    it.energy = st[i].energy;
    it.changed = st[i].changed;
    it.nn_calls = st[i].nn_calls;
    it.millis = st[i].millis;
    it.lsq_energy_before = st[i].lsq_energy_before;
    it.lsq_energy_after = st[i].lsq_energy_after;
    it.points_scanned = st[i].points_scanned;
    r.trace.iterations.push_back(it);
  }
  return r;
}

}  // namespace persyn::gpu
