// Drop-in check built against the reference's own headers and library
// (oracle/_ref): persyn::gpu::GpuSearchIndex plugged into the REFERENCE's
// optimize_level / search_step (per-query plug-in path, optimizer.hpp:111-119)
// must give the same result as the batched device path
// (persyn::gpu::optimize_level / search_step).  Prints one JSON line.
// Test infrastructure: built by oracle/Makefile (needs /root/reference), run
// by tests/test_dropin.py on a GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>

#include "persyn_gpu.hpp"

using namespace persyn;

static RgbsImage pattern(int W, int H, int seed) {
  RasterImage base(W, H);
  std::vector<double> s(static_cast<std::size_t>(W) * H);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      for (int c = 0; c < 3; ++c) {
        const double v = 0.5 + 0.25 * std::sin(0.37 * x * (c + 1) + 0.23 * y + seed) +
                         0.2 * std::cos(0.11 * (x + 2 * y) * (c + 2) - seed);
        base.at(c, x, y) = std::round(std::clamp(v, 0.0, 1.0) * 255.0) / 255.0;
      }
      s[static_cast<std::size_t>(y) * W + x] = double(float(y) / float(H - 1));
    }
  return RgbsImage(std::move(base), std::move(s));
}

int main() {
  gpu::Context ctx(0);
  const RgbsImage ex = pattern(40, 40, 1);
  const RgbsImage init = pattern(56, 56, 5);
  auto ix = gpu::GpuSearchIndex::pca_tree(ctx, ex, 8, 0.95, 4, 7);
  OptimizerConfig cfg;
  cfg.grid = GridSpec{8, 4, init.width(), init.height()};
  cfg.patch = PatchSpec{2};
  cfg.budget = QueryBudget::exact();
  cfg.max_iterations = 3;
  cfg.min_iterations = 3;
  cfg.convergence_fraction = 1e-9;
  const HistogramSet eh = build_histograms(ex, 16);
  // search_step: reference loop over the plug-in vs batched device search
  const SparseGrid grid = make_sparse_grid(cfg.grid);
  const SearchOutcome so_ref = persyn::search_step(init, *ix, grid, cfg.patch, cfg.budget, 1);
  const SearchOutcome so_gpu = gpu::search_step(init, *ix, grid, cfg.patch, cfg.budget);
  const bool search_equal = so_ref.assignments.input_index == so_gpu.assignments.input_index &&
                            so_ref.assignments.distance == so_gpu.assignments.distance &&
                            so_ref.nn_calls == so_gpu.nn_calls;
  // optimize_level: the reference's EM loop with the device index plugged in
  const LevelResult a = persyn::optimize_level(init, *ix, cfg, &eh);
  const LevelResult b = gpu::optimize_level(init, *ix, cfg, &eh);
  double maxdiff = 0.0;
  for (int c = 0; c < 4; ++c)
    for (int y = 0; y < init.height(); ++y)
      for (int x = 0; x < init.width(); ++x)
        maxdiff = std::max(maxdiff, std::fabs(a.image.value(c, x, y) - b.image.value(c, x, y)));
  bool stats_equal = a.trace.iterations.size() == b.trace.iterations.size();
  double energy_rel = 0.0;
  for (std::size_t i = 0; stats_equal && i < a.trace.iterations.size(); ++i) {
    const auto& p = a.trace.iterations[i];
    const auto& q = b.trace.iterations[i];
    stats_equal = p.iteration == q.iteration && p.changed == q.changed && p.nn_calls == q.nn_calls;
    energy_rel = std::max(energy_rel, std::fabs(p.energy - q.energy) / std::fabs(p.energy));
  }
  // the error mapping: an odd window is a persyn::DomainError
  bool domain_error = false;
  try {
    gpu::GpuSearchIndex::pca_tree(ctx, ex, 7);
  } catch (const persyn::DomainError&) {
    domain_error = true;
  }
  std::printf("{\"describe\": \"%s\", \"search_equal\": %s, \"optimize_max_abs_diff\": %.3e, "
              "\"optimize_stats_equal\": %s, \"energy_rel_diff\": %.3e, \"iterations\": %zu, "
              "\"domain_error_mapped\": %s}\n",
              ix->describe().c_str(), search_equal ? "true" : "false", maxdiff,
              stats_equal ? "true" : "false", energy_rel, a.trace.iterations.size(),
              domain_error ? "true" : "false");
  return 0;
}
