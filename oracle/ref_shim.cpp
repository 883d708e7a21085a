// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// C-ABI harness over the reference's OWN hot-path translation units
// (/root/reference/proj/core/src/{image,neighborhood,km_tree,optimizer}.cpp),
// compiled unmodified from where they lie by oracle/Makefile into
// oracle/_ref/libpersyn_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg / --impl reference) may load it.
//
// The one reference TU that does not build here is pca.cpp (needs Eigen3,
// absent).  PcaModel's projection is a five-line loop; it is RESTATED below
// from pca.cpp:27-41 / :103-113 so the reference's optimizer can run with a
// PCA basis injected through the public PcaModel ctor (pca.hpp:18-19).
// fit_pca (pca.cpp:49-101) is NOT restated: it throws, parity of the fit is
// unpinned and every basis is injected.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "persyn/image.hpp"
#include "persyn/km_tree.hpp"
#include "persyn/neighborhood.hpp"
#include "persyn/optimizer.hpp"
#include "persyn/pca.hpp"
#include "persyn/pipeline.hpp"
#include "persyn/scale_map.hpp"

// ---- PcaModel restatement (pca.cpp:11-47, :103-113), fp64, j ascending -----
namespace persyn {

PcaModel::PcaModel(std::vector<double> mean, std::vector<double> basis,
                   std::vector<double> variances, std::size_t retained_dim)
    : mean_(std::move(mean)), basis_(std::move(basis)),
      variances_(std::move(variances)), retained_dim_(retained_dim) {}

double PcaModel::retained_variance_ratio() const {
  double total = 0.0, kept = 0.0;
  for (std::size_t i = 0; i < variances_.size(); ++i) {
    total += variances_[i];
    if (i < retained_dim_) kept += variances_[i];
  }
  return total > 0.0 ? kept / total : 1.0;
}

void PcaModel::project(std::span<const float> v, std::span<double> out) const {
  if (v.size() != input_dim()) throw ShapeError("projection dim mismatch");
  for (std::size_t k = 0; k < retained_dim_; ++k) {
    const double* row = basis_.data() + k * input_dim();
    double acc = 0.0;
    for (std::size_t j = 0; j < input_dim(); ++j) {
      const double c = static_cast<double>(v[j]) - mean_[j];
      const double p = c * row[j];
      acc = acc + p;
    }
    out[k] = acc;
  }
}

std::vector<double> PcaModel::project(std::span<const float> v) const {
  std::vector<double> out(retained_dim_);
  project(v, out);
  return out;
}

PcaModel fit_pca(const NeighborhoodMatrix&, double) {
  throw DomainError("fit_pca unavailable in the oracle build (Eigen3 absent); inject a basis");
}

ProjectedMatrix project_all(const PcaModel& model, const NeighborhoodMatrix& points) {
  ProjectedMatrix out;
  out.dim = model.retained_dim();
  out.count = points.count();
  out.data.resize(out.dim * out.count);
  for (std::size_t i = 0; i < out.count; ++i) {
    model.project(points.vec(static_cast<std::int32_t>(i)),
                  {out.data.data() + i * out.dim, out.dim});
  }
  return out;
}

}  // namespace persyn

using namespace persyn;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

// status codes mirror include/persyn_b200.h
enum { OK = 0, E_DOMAIN = 1, E_SHAPE = 2, E_LOGIC = 3, E_OTHER = 9 };

template <class F>
int guard(F&& f) {
  try {
    f();
    return OK;
  } catch (const DomainError& e) {
    return fail(e, E_DOMAIN);
  } catch (const ShapeError& e) {
    return fail(e, E_SHAPE);
  } catch (const std::logic_error& e) {
    return fail(e, E_LOGIC);
  } catch (const std::exception& e) {
    return fail(e, E_OTHER);
  }
}

// planes: [4][H][W] fp64, row 0 = bottom (image.hpp:11-12)
RgbsImage make_rgbs(const double* planes, int W, int H) {
  RasterImage base(W, H);
  const std::size_t P = static_cast<std::size_t>(W) * H;
  for (int c = 0; c < 3; ++c) std::memcpy(base.plane(c).data(), planes + c * P, P * 8);
  std::vector<double> s(planes + 3 * P, planes + 4 * P);
  return RgbsImage(std::move(base), std::move(s));
}

void store_rgbs(const RgbsImage& img, double* planes) {
  const std::size_t P = static_cast<std::size_t>(img.width()) * img.height();
  for (int c = 0; c < 3; ++c) std::memcpy(planes + c * P, img.base().plane(c).data(), P * 8);
  std::memcpy(planes + 3 * P, img.scale_plane().data(), P * 8);
}

QueryBudget make_budget(int mode, int max_leaves) {
  if (mode == 0) return QueryBudget::greedy();
  if (mode == 1) return QueryBudget::backtrack(max_leaves);
  return QueryBudget::exact();
}

// A SearchIndex over reference-extracted candidates with an injected PCA
// model.  kind 0: PCA + the reference's own KmTree (mirrors PcaTreeIndex,
// optimizer.cpp:214-248); kind 1: PCA + brute_force_nearest in PCA space
// (km_tree.cpp:320-340; equals KmTree exact, ann_test.cpp:225-245).
class InjectedIndex final : public SearchIndex {
 public:
  InjectedIndex(NeighborhoodMatrix cand, PcaModel pca, int kind, int branching,
                std::uint64_t seed)
      : cand_(std::move(cand)), pca_(std::move(pca)), kind_(kind) {
    ProjectedMatrix pm = project_all(pca_, cand_);
    proj_ = pm.data;
    if (kind_ == 0) {
      tree_.emplace(KmTree::build(std::move(pm.data), pm.dim, pm.count, branching,
                                  static_cast<std::size_t>(branching), seed));
    }
  }

  QueryResult nearest(std::span<const float> query, const QueryBudget& budget) const override {
    thread_local std::vector<double> q;
    q.resize(pca_.retained_dim());
    pca_.project(query, q);
    QueryResult r;
    if (kind_ == 0) {
      r = tree_->query(q, budget);
    } else {
      double d = 0.0;
      r.index = brute_force_nearest(proj_, pca_.retained_dim(), q, &d);
      r.stats.points_scanned = static_cast<std::int64_t>(cand_.count());
    }
    r.distance = full_distance(query, cand_.vec(r.index));
    return r;
  }
  const NeighborhoodMatrix& candidates() const override { return cand_; }
  const PcaModel* pca_model() const override { return &pca_; }
  std::string describe() const override { return "injected"; }

  const KmTree* tree() const { return tree_ ? &*tree_ : nullptr; }
  const std::vector<double>& projected() const { return proj_; }

 private:
  NeighborhoodMatrix cand_;
  PcaModel pca_;
  int kind_;
  std::vector<double> proj_;
  std::optional<KmTree> tree_;
};

struct RefIndex {
  RgbsImage exemplar;
  std::unique_ptr<SearchIndex> index;
  InjectedIndex* injected = nullptr;
};

OptimizerConfig make_cfg(int W, int H, int w, int sp, int patch, double r, double eps,
                         int max_it, int min_it, double frac, int bins, int hist_on,
                         int include_scale, int mode, int max_leaves) {
  OptimizerConfig cfg;
  cfg.robust_exponent = r;
  cfg.distance_epsilon = eps;
  cfg.max_iterations = max_it;
  cfg.min_iterations = min_it;
  cfg.convergence_fraction = frac;
  cfg.histogram_bins = bins;
  cfg.histogram_matching = hist_on != 0;
  cfg.histogram_include_scale = include_scale != 0;
  cfg.grid = GridSpec{w, sp, W, H};
  cfg.patch = PatchSpec{patch};
  cfg.budget = make_budget(mode, max_leaves);
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- L1 geometry (neighborhood.cpp) ------------------------------------------
int ref_grid_axes(int W, int H, int w, int sp, int* xs, int* nx, int* ys, int* ny) {
  return guard([&] {
    const SparseGrid g = make_sparse_grid(GridSpec{w, sp, W, H});
    *nx = static_cast<int>(g.xs.size());
    *ny = static_cast<int>(g.ys.size());
    if (xs) std::copy(g.xs.begin(), g.xs.end(), xs);
    if (ys) std::copy(g.ys.begin(), g.ys.end(), ys);
  });
}

int ref_containing_anchors(int W, int H, int w, int sp, int ox, int oy, int region,
                           int32_t* out, int* n) {
  return guard([&] {
    const SparseGrid g = make_sparse_grid(GridSpec{w, sp, W, H});
    const auto ids = containing_anchors(g, PixelCoord{ox, oy}, region);
    *n = static_cast<int>(ids.size());
    if (out) std::copy(ids.begin(), ids.end(), out);
  });
}

int ref_patch_tiles(int W, int H, int p, int32_t* xy, int64_t* n) {
  return guard([&] {
    const auto t = patch_tiles(W, H, PatchSpec{p});
    *n = static_cast<int64_t>(t.size());
    if (xy) {
      for (std::size_t i = 0; i < t.size(); ++i) {
        xy[2 * i] = t[i].x;
        xy[2 * i + 1] = t[i].y;
      }
    }
  });
}

// Dense/sparse extraction, rows in ascending anchor order (neighborhood.cpp:103-118).
int ref_extract_all(const double* planes, int W, int H, int w, int sp, float* out,
                    int64_t* count) {
  return guard([&] {
    const RgbsImage img = make_rgbs(planes, W, H);
    const NeighborhoodMatrix m = extract_all(img, GridSpec{w, sp, W, H});
    *count = static_cast<int64_t>(m.count());
    if (out) std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
  });
}

// ---- L2 km_tree ----------------------------------------------------------------
void* ref_kmtree_build(const double* pts, int64_t count, int dim, int branching,
                       int64_t leaf_threshold, uint64_t seed) {
  KmTree* out = nullptr;
  const int st = guard([&] {
    std::vector<double> p(pts, pts + (dim > 0 ? count * dim : 0));
    out = new KmTree(KmTree::build(std::move(p), static_cast<std::size_t>(dim),
                                   static_cast<std::size_t>(count), branching,
                                   static_cast<std::size_t>(leaf_threshold), seed));
  });
  return st == OK ? out : nullptr;
}

void ref_kmtree_destroy(void* t) { delete static_cast<KmTree*>(t); }

int ref_kmtree_query(void* t, const double* q, int dim, int mode, int max_leaves,
                     int32_t* idx, double* dist, int64_t* scanned, int64_t* visited) {
  return guard([&] {
    const QueryResult r = static_cast<KmTree*>(t)->query(
        std::span<const double>(q, static_cast<std::size_t>(dim)), make_budget(mode, max_leaves));
    *idx = r.index;
    *dist = r.distance;
    if (scanned) *scanned = r.stats.points_scanned;
    if (visited) *visited = r.stats.nodes_visited;
  });
}

// Leaves in DFS order (km_tree.cpp:286-298): concatenated ids + per-leaf sizes.
int ref_kmtree_leaves(void* t, int32_t* ids, int32_t* sizes, int64_t* n_leaves) {
  return guard([&] {
    const auto lv = static_cast<KmTree*>(t)->leaves();
    *n_leaves = static_cast<int64_t>(lv.size());
    std::size_t o = 0;
    for (std::size_t i = 0; i < lv.size(); ++i) {
      if (sizes) sizes[i] = static_cast<int32_t>(lv[i].size());
      if (ids) std::copy(lv[i].begin(), lv[i].end(), ids + o);
      o += lv[i].size();
    }
  });
}

int ref_kmtree_structure_json(void* t, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    const std::string s = static_cast<KmTree*>(t)->structure_json();
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > 0) {
      const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

int ref_brute_force_nearest(const double* pts, int64_t count, int dim, const double* q,
                            int32_t* idx, double* dist) {
  return guard([&] {
    *idx = brute_force_nearest(std::span<const double>(pts, count * dim), dim,
                               std::span<const double>(q, dim), dist);
  });
}

// ---- L3 search index ---------------------------------------------------------------
// kind 0: injected PCA + reference KmTree; 1: injected PCA + PCA-space brute
// force; 2: the reference's own BruteForceIndex (full-D, optimizer.cpp:168-212).
void* ref_index_create(const double* ex_planes, int EW, int EH, int w, const double* mean,
                       const double* basis, int d, int kind, int branching, uint64_t seed) {
  RefIndex* out = nullptr;
  const int st = guard([&] {
    auto ri = std::make_unique<RefIndex>();
    ri->exemplar = make_rgbs(ex_planes, EW, EH);
    NeighborhoodMatrix cand = extract_all(ri->exemplar, GridSpec{w, 1, EW, EH});
    if (kind == 2) {
      ri->index = make_brute_force_index(std::move(cand));
    } else {
      const std::size_t D = cand.dim;
      PcaModel pca(std::vector<double>(mean, mean + D),
                   std::vector<double>(basis, basis + static_cast<std::size_t>(d) * D),
                   std::vector<double>(D, 0.0), static_cast<std::size_t>(d));
      auto inj = std::make_unique<InjectedIndex>(std::move(cand), std::move(pca), kind,
                                                 branching, seed);
      ri->injected = inj.get();
      ri->index = std::move(inj);
    }
    out = ri.release();
  });
  return st == OK ? out : nullptr;
}

void ref_index_destroy(void* h) { delete static_cast<RefIndex*>(h); }

int64_t ref_index_count(void* h) {
  return static_cast<int64_t>(static_cast<RefIndex*>(h)->index->candidates().count());
}

// Projected database (N x d, row-major) of an injected index.
int ref_index_projected(void* h, double* out) {
  return guard([&] {
    auto* ri = static_cast<RefIndex*>(h);
    if (!ri->injected) throw DomainError("not an injected PCA index");
    const auto& p = ri->injected->projected();
    std::memcpy(out, p.data(), p.size() * 8);
  });
}

void* ref_index_tree(void* h) {
  auto* ri = static_cast<RefIndex*>(h);
  return ri->injected ? const_cast<KmTree*>(ri->injected->tree()) : nullptr;
}

int ref_index_nearest(void* h, const float* q, int D, int mode, int max_leaves, int32_t* idx,
                      double* dist, int64_t* scanned) {
  return guard([&] {
    const QueryResult r = static_cast<RefIndex*>(h)->index->nearest(
        std::span<const float>(q, static_cast<std::size_t>(D)), make_budget(mode, max_leaves));
    *idx = r.index;
    *dist = r.distance;
    if (scanned) *scanned = r.stats.points_scanned;
  });
}

// ---- L4 optimizer --------------------------------------------------------------------
int ref_search_step(void* h, const double* planes, int W, int H, int w, int sp, int patch,
                    int mode, int max_leaves, int workers, int32_t* idx, double* dist,
                    int64_t* nn_calls, int64_t* scanned) {
  return guard([&] {
    auto* ri = static_cast<RefIndex*>(h);
    const RgbsImage img = make_rgbs(planes, W, H);
    const SparseGrid g = make_sparse_grid(GridSpec{w, sp, W, H});
    const SearchOutcome o =
        search_step(img, *ri->index, g, PatchSpec{patch}, make_budget(mode, max_leaves), workers);
    std::copy(o.assignments.input_index.begin(), o.assignments.input_index.end(), idx);
    std::copy(o.assignments.distance.begin(), o.assignments.distance.end(), dist);
    *nn_calls = o.nn_calls;
    *scanned = o.points_scanned;
  });
}

int ref_update_step(void* h, int W, int H, int w, int sp, const int32_t* idx,
                    const double* irls, const double* pen, const double* in_planes,
                    double* out_planes) {
  return guard([&] {
    auto* ri = static_cast<RefIndex*>(h);
    const SparseGrid g = make_sparse_grid(GridSpec{w, sp, W, H});
    const std::size_t A = static_cast<std::size_t>(g.count());
    AssignmentMap am{std::vector<int32_t>(idx, idx + A), std::vector<double>(A, 0.0)};
    WeightMap wm{std::vector<double>(irls, irls + A), std::vector<double>(pen, pen + A)};
    const RgbsImage x = make_rgbs(in_planes, W, H);
    const RgbsImage y = update_step(am, wm, g, ri->index->candidates(), x);
    store_rgbs(y, out_planes);
  });
}

int ref_assignment_distances(void* h, const double* planes, int W, int H, int w, int sp,
                             const int32_t* idx, double* out) {
  return guard([&] {
    auto* ri = static_cast<RefIndex*>(h);
    const SparseGrid g = make_sparse_grid(GridSpec{w, sp, W, H});
    const RgbsImage x = make_rgbs(planes, W, H);
    const auto d = assignment_distances(
        x, g, ri->index->candidates(),
        std::span<const int32_t>(idx, static_cast<std::size_t>(g.count())));
    std::copy(d.begin(), d.end(), out);
  });
}

// Exemplar histogram of the index's exemplar (pipeline.cpp:286-292 equivalent).
int ref_index_histograms(void* h, int bins, int include_scale, double* mass) {
  return guard([&] {
    const HistogramSet hs =
        build_histograms(static_cast<RefIndex*>(h)->exemplar, bins, include_scale != 0);
    for (std::size_t s = 0; s < hs.channel_ids().size(); ++s)
      for (int b = 0; b < bins; ++b) mass[s * bins + b] = hs.mass(s, b);
  });
}

// stats: per iteration 7 doubles {iter, energy, changed, nn_calls, lsq_before,
// lsq_after, points_scanned} + millis in a separate array.
int ref_optimize_level(void* h, const double* init, int W, int H, int w, int sp, int patch,
                       double r, double eps, int max_it, int min_it, double frac, int bins,
                       int hist_on, int include_scale, int mode, int max_leaves,
                       double* out_planes, double* stats, double* millis, int* n_iters) {
  return guard([&] {
    auto* ri = static_cast<RefIndex*>(h);
    const OptimizerConfig cfg = make_cfg(W, H, w, sp, patch, r, eps, max_it, min_it, frac, bins,
                                         hist_on, include_scale, mode, max_leaves);
    const RgbsImage x = make_rgbs(init, W, H);
    std::optional<HistogramSet> eh;
    if (hist_on) eh = build_histograms(ri->exemplar, bins, include_scale != 0);
    const LevelResult res = optimize_level(x, *ri->index, cfg, eh ? &*eh : nullptr);
    store_rgbs(res.image, out_planes);
    *n_iters = static_cast<int>(res.trace.iterations.size());
    for (std::size_t i = 0; i < res.trace.iterations.size(); ++i) {
      const auto& it = res.trace.iterations[i];
      double* s = stats + 7 * i;
      s[0] = it.iteration;
      s[1] = it.energy;
      s[2] = static_cast<double>(it.changed);
      s[3] = static_cast<double>(it.nn_calls);
      s[4] = it.lsq_energy_before;
      s[5] = it.lsq_energy_after;
      s[6] = static_cast<double>(it.points_scanned);
      if (millis) millis[i] = it.millis;
    }
  });
}

// EnergyTrace::to_jsonl (optimizer.cpp:411-424) over given iteration records
// (stats7: iteration, energy, changed, nn_calls, ... as ref_optimize_level),
// to pin the JSONL trace format of the device path.
int ref_trace_jsonl(const double* stats7, const double* millis, int n, char* buf, int64_t cap,
                    int64_t* len) {
  return guard([&] {
    EnergyTrace tr;
    for (int i = 0; i < n; ++i) {
      IterationStats it;
      it.iteration = static_cast<int>(stats7[7 * i]);
      it.energy = stats7[7 * i + 1];
      it.changed = static_cast<std::int64_t>(stats7[7 * i + 2]);
      it.nn_calls = static_cast<std::int64_t>(stats7[7 * i + 3]);
      it.millis = millis[i];
      tr.iterations.push_back(it);
    }
    const std::string out = tr.to_jsonl();
    *len = static_cast<int64_t>(out.size());
    if (buf && cap > 0) {
      const size_t k = std::min<size_t>(out.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, out.data(), k);
      buf[k] = 0;
    }
  });
}

// One pass of optimize_level's loop body (optimizer.cpp:453-497) driven
// through the reference's own public functions (irls_weight, build_histograms,
// histogram_penalty, update_step, assignment_distances, search_step,
// energy_from_distances) on caller-held state: used to time bounded samples of
// an EM iteration (bench.py --impl reference).  When *primed == 0 the priming
// search (optimizer.cpp:445) runs first and *primed is set.
int ref_em_iteration(void* h, double* planes, int W, int H, int w, int sp, int patch, double r,
                     double eps, int bins, int hist_on, int mode, int max_leaves, int workers,
                     int32_t* idx, double* dist, int* primed, double* energy, int64_t* changed) {
  return guard([&] {
    auto* ri = static_cast<RefIndex*>(h);
    const SparseGrid g = make_sparse_grid(GridSpec{w, sp, W, H});
    const std::size_t A = static_cast<std::size_t>(g.count());
    const QueryBudget budget = make_budget(mode, max_leaves);
    RgbsImage x = make_rgbs(planes, W, H);
    if (!*primed) {
      const SearchOutcome o = search_step(x, *ri->index, g, PatchSpec{patch}, budget, workers);
      std::copy(o.assignments.input_index.begin(), o.assignments.input_index.end(), idx);
      std::copy(o.assignments.distance.begin(), o.assignments.distance.end(), dist);
      *primed = 1;
    }
    const NeighborhoodMatrix& cand = ri->index->candidates();
    WeightMap wm;
    wm.irls.resize(A);
    wm.hist_penalty.assign(A, 0.0);
    for (std::size_t i = 0; i < A; ++i) wm.irls[i] = irls_weight(dist[i], r, eps);
    if (hist_on) {
      const HistogramSet eh = build_histograms(ri->exemplar, bins, false);
      const HistogramSet oh = build_histograms(x, bins, false);
      for (std::size_t i = 0; i < A; ++i)
        wm.hist_penalty[i] = histogram_penalty(cand.vec(idx[i]), oh, eh);
    }
    AssignmentMap am{std::vector<int32_t>(idx, idx + A), std::vector<double>(dist, dist + A)};
    x = update_step(am, wm, g, cand, x);
    const auto after = assignment_distances(x, g, cand, am.input_index);
    double lsq = 0.0;
    for (std::size_t i = 0; i < A; ++i) lsq += wm.effective(i) * after[i] * after[i];
    const SearchOutcome o = search_step(x, *ri->index, g, PatchSpec{patch}, budget, workers);
    int64_t ch = 0;
    for (std::size_t i = 0; i < A; ++i) ch += o.assignments.input_index[i] != idx[i];
    std::copy(o.assignments.input_index.begin(), o.assignments.input_index.end(), idx);
    std::copy(o.assignments.distance.begin(), o.assignments.distance.end(), dist);
    if (energy) *energy = energy_from_distances(o.assignments.distance, r) + 0.0 * lsq;
    if (changed) *changed = ch;
    store_rgbs(x, planes);
  });
}

// ---- weights, histograms, energies (optimizer.cpp:44-131) ------------------------
int ref_build_histograms(const double* planes, int W, int H, int bins, int include_scale,
                         double* mass) {
  return guard([&] {
    const HistogramSet hs = build_histograms(make_rgbs(planes, W, H), bins, include_scale != 0);
    for (std::size_t s = 0; s < hs.channel_ids().size(); ++s)
      for (int b = 0; b < bins; ++b) mass[s * bins + b] = hs.mass(s, b);
  });
}

int ref_histogram_penalty(const float* nb, int64_t D, int bins, int include_scale,
                          const double* out_mass, const double* ex_mass, double* pen) {
  return guard([&] {
    std::vector<int> ch{0, 1, 2};
    if (include_scale) ch.push_back(3);
    std::vector<std::vector<double>> om(ch.size()), em(ch.size());
    for (std::size_t s = 0; s < ch.size(); ++s) {
      om[s].assign(out_mass + s * bins, out_mass + (s + 1) * bins);
      em[s].assign(ex_mass + s * bins, ex_mass + (s + 1) * bins);
    }
    const HistogramSet ho(bins, ch, om), he(bins, ch, em);
    *pen = histogram_penalty(std::span<const float>(nb, static_cast<std::size_t>(D)), ho, he);
  });
}

int ref_irls_weights(const double* d, int64_t n, double r, double eps, double* out) {
  return guard([&] {
    for (int64_t i = 0; i < n; ++i) out[i] = irls_weight(d[i], r, eps);
  });
}

int ref_energy_from_distances(const double* d, int64_t n, double r, double* out) {
  return guard([&] {
    *out = energy_from_distances(std::span<const double>(d, static_cast<std::size_t>(n)), r);
  });
}

int ref_full_distance(const float* a, const float* b, int64_t D, double* out) {
  return guard([&] {
    *out = full_distance(std::span<const float>(a, static_cast<std::size_t>(D)),
                         std::span<const float>(b, static_cast<std::size_t>(D)));
  });
}

// ---- L0 resampling (image.cpp:38-109) ----------------------------------------------
int ref_downsample(const double* rgb, int W, int H, int factor, double* out, int* ow, int* oh) {
  return guard([&] {
    RasterImage img(W, H);
    const std::size_t P = static_cast<std::size_t>(W) * H;
    for (int c = 0; c < 3; ++c) std::memcpy(img.plane(c).data(), rgb + c * P, P * 8);
    const RasterImage o = downsample(img, factor);
    *ow = o.width();
    *oh = o.height();
    const std::size_t Q = static_cast<std::size_t>(o.width()) * o.height();
    if (out)
      for (int c = 0; c < 3; ++c) std::memcpy(out + c * Q, o.plane(c).data(), Q * 8);
  });
}

int ref_upsample_bilinear(const double* rgb, int W, int H, int factor, double* out) {
  return guard([&] {
    RasterImage img(W, H);
    const std::size_t P = static_cast<std::size_t>(W) * H;
    for (int c = 0; c < 3; ++c) std::memcpy(img.plane(c).data(), rgb + c * P, P * 8);
    const RasterImage o = upsample_bilinear(img, factor);
    const std::size_t Q = static_cast<std::size_t>(o.width()) * o.height();
    for (int c = 0; c < 3; ++c) std::memcpy(out + c * Q, o.plane(c).data(), Q * 8);
  });
}

int ref_worker_count(void) { return worker_count(); }

// ---- part 1 (scale_map.cpp, pipeline.cpp:96-175) ----------------------------------
// compute_scale_map: raw float values + bounds {s_max, s_min, s_delta}.
int ref_scale_map(int W, int H, double slant, double tilt, float* values, double* bounds) {
  return guard([&] {
    const ScaleMap m = compute_scale_map(W, H, ViewAngles{slant, tilt});
    std::copy(m.values().begin(), m.values().end(), values);
    bounds[0] = m.bounds().s_max;
    bounds[1] = m.bounds().s_min;
    bounds[2] = m.bounds().s_delta;
  });
}

// attach_scale_channel(rgb, compute_scale_map(W, H, view)) -> 4 planes.
int ref_attach_scale(const double* rgb, int W, int H, double slant, double tilt, double* out4) {
  return guard([&] {
    RasterImage img(W, H);
    const std::size_t P = static_cast<std::size_t>(W) * H;
    for (int c = 0; c < 3; ++c) std::memcpy(img.plane(c).data(), rgb + c * P, P * 8);
    store_rgbs(attach_scale_channel(img, compute_scale_map(W, H, ViewAngles{slant, tilt})), out4);
  });
}

// ---- report / bench formats (pipeline.cpp:182-214, :336-357) -------------------------
static void put_text(const std::string& out, char* buf, int64_t cap, int64_t* len) {
  *len = static_cast<int64_t>(out.size());
  if (buf && cap > 0) {
    const size_t k = std::min<size_t>(out.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, out.data(), k);
    buf[k] = 0;
  }
}

static std::vector<std::string> split_lines(const char* s) {
  std::vector<std::string> v;
  std::string cur;
  for (const char* p = s; *p; ++p) {
    if (*p == '\n') {
      v.push_back(cur);
      cur.clear();
    } else {
      cur += *p;
    }
  }
  v.push_back(cur);
  return v;
}

// SynthesisReport::to_json over given levels; stats5 per iteration:
// iter, energy, changed, nn_calls, millis.
int ref_report_json(const char* config_echo, double part1, double part2, int64_t total_calls,
                    int n_levels, const int* widths, const int* heights, const char* index_names,
                    const int* n_iters, const double* stats5, char* buf, int64_t cap,
                    int64_t* len) {
  return guard([&] {
    SynthesisReport r;
    r.config_echo = config_echo;
    r.part1_millis = part1;
    r.part2_millis = part2;
    r.total_nn_calls = total_calls;
    const auto names = split_lines(index_names);
    const double* s = stats5;
    for (int l = 0; l < n_levels; ++l) {
      LevelReport lr;
      lr.width = widths[l];
      lr.height = heights[l];
      lr.index = names[static_cast<size_t>(l)];
      for (int i = 0; i < n_iters[l]; ++i, s += 5) {
        IterationStats it;
        it.iteration = static_cast<int>(s[0]);
        it.energy = s[1];
        it.changed = static_cast<std::int64_t>(s[2]);
        it.nn_calls = static_cast<std::int64_t>(s[3]);
        it.millis = s[4];
        lr.trace.iterations.push_back(it);
      }
      r.levels.push_back(std::move(lr));
    }
    put_text(r.to_json(), buf, cap, len);
  });
}

// save_scale_map / load_scale_map (scale_map.cpp:125-201, the PSM1 container).
int ref_save_scale_map(const float* values, int W, int H, double slant, double tilt, double s_min,
                       double s_max, const char* path) {
  return guard([&] {
    ScaleBounds b;
    b.s_min = s_min;
    b.s_max = s_max;
    b.s_delta = s_max - s_min;
    save_scale_map(ScaleMap(W, H, std::vector<float>(values, values + (size_t)W * H),
                            ViewAngles{slant, tilt}, b),
                   path);
  });
}

int ref_load_scale_map(const char* path, int* wh, double* view_bounds, float* values) {
  return guard([&] {
    const ScaleMap m = load_scale_map(path);
    wh[0] = m.width();
    wh[1] = m.height();
    view_bounds[0] = m.view().slant_deg;
    view_bounds[1] = m.view().tilt_deg;
    view_bounds[2] = m.bounds().s_min;
    view_bounds[3] = m.bounds().s_max;
    if (values) std::copy(m.values().begin(), m.values().end(), values);
  });
}

// modes_to_json (which = 0) / modes_to_csv (which = 1).
int ref_modes_format(const char* names, const double* wall, const double* part2,
                     const int64_t* calls, const double* energy, int n, int which, char* buf,
                     int64_t cap, int64_t* len) {
  return guard([&] {
    const auto nm = split_lines(names);
    std::vector<ModeRun> runs;
    for (int i = 0; i < n; ++i)
      runs.push_back({nm[static_cast<size_t>(i)], wall[i], part2[i], calls[i], energy[i]});
    put_text(which == 0 ? modes_to_json(runs) : modes_to_csv(runs), buf, cap, len);
  });
}

// initialize_output(exemplar_rgbs, ScaleMap(values, bounds), mt19937_64(seed)).
int ref_initialize_output(const double* ex4, int ew, int eh, const float* out_vals, int ow,
                          int oh, double s_min, double s_max, uint64_t seed, double* out4) {
  return guard([&] {
    const RgbsImage ex = make_rgbs(ex4, ew, eh);
    std::vector<float> v(out_vals, out_vals + static_cast<std::size_t>(ow) * oh);
    ScaleBounds b;
    b.s_max = s_max;
    b.s_min = s_min;
    b.s_delta = s_max - s_min;
    const ScaleMap map(ow, oh, std::move(v), ViewAngles{}, b);
    std::mt19937_64 rng(seed);
    store_rgbs(initialize_output(ex, map, rng), out4);
  });
}

}  // extern "C"
