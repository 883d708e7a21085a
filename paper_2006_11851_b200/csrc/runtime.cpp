// Native host runtime + C ABI (include/persyn_b200.h).
//
// Owns device memory, the stream, the per-stage index build, the EM loop
// (optimize_level, optimizer.cpp:426-516), the pyramid driver
// (synthesize, pipeline.cpp:216-315) and the status/last-error convention.
// All arithmetic on the hot path runs in the sm_100a kernels; the host only
// orchestrates, validates arguments the way the reference does, and reads
// back one small telemetry record per EM iteration (the reference's
// convergence rule needs `changed` on the host).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "numerics.cuh"
#include "psg_internal.h"

namespace psg {

thread_local std::string g_last_error;
thread_local cudaStream_t t_stream = nullptr;
void set_last_error(const std::string& m) { g_last_error = m; }

namespace {
template <class T>
T* dalloc(size_t count) {  // long-lived (index) buffers, from the stream-ordered pool
  T* p = nullptr;
  if (count) PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, t_stream));
  return p;
}

void check_flags(psg_ctx* ctx) {
  int f = 0;
  PSG_CUDA(cudaMemcpyAsync(&f, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  prof_flush(ctx);
  if (!f) return;
  PSG_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), ctx->stream));
  if (f & FLAG_BAD_DISTANCE) fail(PSG_E_DOMAIN, "distance must be non-negative");
  if (f & FLAG_BAD_WEIGHT) fail(PSG_E_DOMAIN, "non-positive or non-finite update weight");
  if (f & FLAG_UNCOVERED) fail(PSG_E_LOGIC, "output pixel not covered by any window");
  if (f & FLAG_STACK_OVERFLOW) fail(PSG_E_LOGIC, "tree traversal stack overflow");
}

void validate_grid(int w, int sp, int W, int H) {  // neighborhood.cpp:22-35
  if (w < 2) fail(PSG_E_DOMAIN, "neighborhood width must be >= 2");
  if (w % 2 != 0) fail(PSG_E_DOMAIN, "neighborhood width must be even");
  if (sp < 1) fail(PSG_E_DOMAIN, "grid spacing must be >= 1");
  if (sp > w) fail(PSG_E_DOMAIN, "grid spacing larger than the neighborhood width");
  if (W < w || H < w)
    fail(PSG_E_DOMAIN, "image " + std::to_string(W) + "x" + std::to_string(H) +
                           " smaller than the neighborhood window " + std::to_string(w));
}

void validate_cfg(const psg_opt_cfg& c, int w, int W, int H) {  // optimizer.cpp:24-42
  if (!(c.robust_exponent > 0.0 && c.robust_exponent < 2.0))
    fail(PSG_E_DOMAIN, "robust exponent must be in (0, 2)");
  if (!(c.distance_epsilon > 0.0)) fail(PSG_E_DOMAIN, "epsilon must be positive");
  if (c.max_iterations < 1) fail(PSG_E_DOMAIN, "max iterations must be >= 1");
  if (c.min_iterations < 1 || c.min_iterations > c.max_iterations)
    fail(PSG_E_DOMAIN, "min iterations must be in [1, max_iterations]");
  if (!(c.convergence_fraction > 0.0 && c.convergence_fraction < 1.0))
    fail(PSG_E_DOMAIN, "convergence fraction must be in (0, 1)");
  if (c.histogram_bins < 2) fail(PSG_E_DOMAIN, "histogram bins must be >= 2");
  validate_grid(w, c.spacing, W, H);
  if (c.patch_width < 1) fail(PSG_E_DOMAIN, "patch width must be >= 1");
  if (c.patch_width > c.spacing) fail(PSG_E_DOMAIN, "patch width must not exceed the grid spacing");
  if (c.budget.mode < 0 || c.budget.mode > 2) fail(PSG_E_DOMAIN, "unknown query budget mode");
  if (c.budget.mode == PSG_BACKTRACK && c.budget.max_leaves < 1)
    fail(PSG_E_DOMAIN, "backtrack budget must be >= 1");
}

void validate_budget(const psg_budget& b) {
  if (b.mode < 0 || b.mode > 2) fail(PSG_E_DOMAIN, "unknown query budget mode");
  if (b.mode == PSG_BACKTRACK && b.max_leaves < 1) fail(PSG_E_DOMAIN, "backtrack budget must be >= 1");
}

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}
}  // namespace

const char* const kKernelNames[K_COUNT] = {
    "make_mirror", "project_kernel", "search_kernel", "rescore_kernel", "weights_kernel",
    "hist_kernels", "penalty_kernel", "mstep_kernel", "stats_kernel", "build_kernels",
    "pyramid_kernels", "tile_schedule", "exact_fallback"};

ProfScope::ProfScope(psg_ctx* c, int k) : ctx(c), kind(k) {
  if (!ctx->profile) return;
  if (ctx->ev_pool.empty()) {
    cudaEvent_t e;
    PSG_CUDA(cudaEventCreate(&e));
    ctx->ev_pool.push_back(e);
  }
  a = ctx->ev_pool.back();
  ctx->ev_pool.pop_back();
  PSG_CUDA(cudaEventRecord(a, ctx->stream));
}

ProfScope::~ProfScope() {
  if (!a) return;
  cudaEvent_t b;
  if (ctx->ev_pool.empty()) {
    if (cudaEventCreate(&b) != cudaSuccess) return;
  } else {
    b = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
  }
  cudaEventRecord(b, ctx->stream);
  ctx->pending.push_back({kind, a, b});
}

void prof_flush(psg_ctx* ctx) {
  if (ctx->pending.empty()) return;
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (const auto& p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      ctx->kernel_ms[p.kind] += ms;
      ctx->kernel_launches[p.kind] += 1;
    }
    ctx->ev_pool.push_back(p.a);
    ctx->ev_pool.push_back(p.b);
  }
  ctx->pending.clear();
}

std::vector<int32_t> axis_positions(int extent, int window, int step) {  // neighborhood.cpp:12-18
  std::vector<int32_t> xs;
  for (int p = 0; p + window <= extent; p += step) xs.push_back(p);
  const int last = extent - window;
  if (xs.empty() || xs.back() != last) xs.push_back(last);
  return xs;
}

int64_t plan_host(int W, int H, int w, int sp, int p, int32_t* mult) {
  const auto xs = axis_positions(W, w, sp), ys = axis_positions(H, w, sp);
  const auto tx = axis_positions(W, p, p), ty = axis_positions(H, p, p);
  auto count_in = [](const std::vector<int32_t>& v, int lo, int hi) {
    return (int64_t)(std::upper_bound(v.begin(), v.end(), hi) -
                     std::lower_bound(v.begin(), v.end(), lo));
  };
  int64_t cx = 0, cy = 0;
  for (int t : tx) cx += count_in(xs, t + p - w, t);
  for (int t : ty) cy += count_in(ys, t + p - w, t);
  bool uncovered = false;
  std::vector<int64_t> mx(xs.size()), my(ys.size());
  for (size_t i = 0; i < xs.size(); ++i) mx[i] = count_in(tx, xs[i], xs[i] + w - p);
  for (size_t i = 0; i < ys.size(); ++i) my[i] = count_in(ty, ys[i], ys[i] + w - p);
  for (size_t iy = 0; iy < ys.size(); ++iy)
    for (size_t ix = 0; ix < xs.size(); ++ix) {
      const int64_t m = mx[ix] * my[iy];
      if (mult) mult[iy * xs.size() + ix] = (int32_t)m;
      if (m == 0) uncovered = true;
    }
  return uncovered ? -1 : cx * cy;
}

double pow_cr_host(double x, double y) { return pow_cr(x, y); }

Index::~Index() {
  // stream-ordered frees (the allocations come from the context's pool)
  cudaStream_t st = ctx ? ctx->stream : nullptr;
  for (void* p : {(void*)ex_mirror, (void*)ex_mirror8, (void*)vectors, (void*)mean, (void*)basis, (void*)proj, (void*)proj_soa, (void*)perm, (void*)tree.centroid, (void*)tree.radius, (void*)tree.first_child, (void*)tree.n_children, (void*)tree.leaf_start, (void*)tree.leaf_count, (void*)tree.centroid32, (void*)tree.radius32, (void*)tree.cnorm32, (void*)proj32_q4, (void*)tree.centroid32T, (void*)tree.boxlo, (void*)tree.boxhi, (void*)tree.box2, (void*)tree.meta, (void*)tree.tie, (void*)pnorm32, (void*)ex_hist, (void*)brute_op, (void*)brute_n2, (void*)brute_nup, (void*)brute_mu, (void*)brute_tmax, (void*)tc_b, (void*)tc_bmu, (void*)pp32, (void*)proj_leaf, (void*)proj_leaf_il, (void*)tree.centroid_il})
    if (p) cudaFreeAsync(p, st);
}

// ---------------------------------------------------------------------------
// Index build (PcaTreeIndex ctor, optimizer.cpp:216-224, per stage
// pipeline.cpp:276-292).
namespace {

// Device copies of ix.htree (replacing any previous tree): exact fp64 tree
// and leaf-ordered projected points, plus the conservative fp32 filter/bound
// copies of the fast search kernels.
void free_tree(Index& ix) {
  cudaStream_t ctx_stream = ix.ctx ? ix.ctx->stream : nullptr;
  DevTree& T = ix.tree;
  for (void* p : {(void*)T.centroid, (void*)T.radius, (void*)T.first_child, (void*)T.n_children,
                  (void*)T.leaf_start, (void*)T.leaf_count, (void*)T.centroid32,
                  (void*)T.centroid32T, (void*)T.radius32, (void*)T.cnorm32, (void*)T.boxlo,
                  (void*)T.boxhi, (void*)T.box2, (void*)T.meta, (void*)T.tie, (void*)ix.perm, (void*)ix.proj_soa,
                  (void*)ix.proj32_q4, (void*)ix.pnorm32, (void*)ix.pp32, (void*)ix.proj_leaf,
                  (void*)ix.proj_leaf_il, (void*)T.centroid_il})
    if (p) cudaFreeAsync(p, ctx_stream);
  T = DevTree{};
  ix.perm = nullptr;
  ix.proj_soa = nullptr;
  ix.proj32_q4 = nullptr;
  ix.pnorm32 = nullptr;
  ix.pp32 = nullptr;
  ix.proj_leaf = nullptr;
  ix.proj_leaf_il = nullptr;
}

void upload_tree(psg_ctx* ctx, Index& ix) {
  free_tree(ix);
  const int d = ix.d;
  const HostTree& t = ix.htree;
  const int nn = (int)t.radius.size();
  ix.tree.n_nodes = nn;
  ix.tree.max_depth = t.max_depth;
  ix.tree.max_children = t.n_children.empty() ? 0 : *std::max_element(t.n_children.begin(), t.n_children.end());
  ix.tree.centroid = dalloc<double>((size_t)nn * (d > 0 ? d : 1));
  ix.tree.radius = dalloc<double>(nn);
  ix.tree.first_child = dalloc<int32_t>(nn);
  ix.tree.n_children = dalloc<int32_t>(nn);
  ix.tree.leaf_start = dalloc<int32_t>(nn);
  ix.tree.leaf_count = dalloc<int32_t>(nn);
  auto up = [&](auto* dst, const auto& v) {
    if (!v.empty())
      PSG_CUDA(cudaMemcpyAsync(dst, v.data(), sizeof(v[0]) * v.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
  };
  up(ix.tree.centroid, t.centroid);
  up(ix.tree.radius, t.radius);
  up(ix.tree.first_child, t.first_child);
  up(ix.tree.n_children, t.n_children);
  up(ix.tree.leaf_start, t.leaf_start);
  up(ix.tree.leaf_count, t.leaf_count);
  ix.perm = dalloc<int32_t>(ix.N);
  up(ix.perm, t.perm);
  ix.proj_soa = dalloc<double>((size_t)ix.N * (d > 0 ? d : 1));
  launch_gather_soa(ctx, ix.proj, ix.N, d, ix.perm, ix.proj_soa);
  ix.proj_leaf = dalloc<double>((size_t)ix.N * (d > 0 ? d : 1));
  if (d > 0) launch_gather_rows_f64(ctx, ix.proj, ix.perm, ix.N, d, ix.proj_leaf);
  // fp32 bound/filter copies (conservative rounding, see search_exact_kernel)
  // fp32 layout width = the tile kernel's DP (24, 32, 48, 64; kMaxDP above)
  ix.dp = d <= 24 ? 24 : (d <= 32 ? 32 : (d <= 48 ? 48 : (d <= 64 ? 64 : kMaxDP)));
  ix.proj32_q4 = dalloc<float>((size_t)ix.N * ix.dp);
  ix.pnorm32 = dalloc<float>(ix.N);
  ix.pp32 = dalloc<float2>(ix.N);
  launch_make_fp32_copies(ctx, ix.proj_soa, ix.N, d, ix.dp, ix.proj32_q4, ix.pnorm32, ix.pp32);
  {
    std::vector<float> pn(ix.N);
    PSG_CUDA(cudaMemcpyAsync(pn.data(), ix.pnorm32, sizeof(float) * ix.N, cudaMemcpyDeviceToHost,
                             ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    float mx = 0.f;
    for (float v : pn) mx = std::max(mx, v);
    ix.pnorm_max = std::nextafter(mx, INFINITY);
  }
  {
    std::vector<float> c32(t.centroid.size()), c32t(t.centroid.size()), r32(nn), n32(nn);
    std::vector<float> blo((size_t)kBoxDims * nn, 0.f), bhi((size_t)kBoxDims * nn, 0.f);
    for (int i = 0; i < nn; ++i)
      for (int j = 0; j < d; ++j) {
        c32[(size_t)i * d + j] = (float)t.centroid[(size_t)i * d + j];
        c32t[(size_t)j * nn + i] = (float)t.centroid[(size_t)i * d + j];
      }
    for (int i = 0; i < nn; ++i)
      for (int j = 0; j < std::min(d, kBoxDims); ++j) {
        blo[(size_t)j * nn + i] = std::nextafter((float)t.boxlo[(size_t)i * kBoxDims + j], -INFINITY);
        bhi[(size_t)j * nn + i] = std::nextafter((float)t.boxhi[(size_t)i * kBoxDims + j], INFINITY);
      }
    std::vector<float> box2((size_t)nn * 2 * kBoxDims);
    for (int i = 0; i < nn; ++i)
      for (int j = 0; j < kBoxDims; ++j) {
        box2[((size_t)i * kBoxDims + j) * 2] = blo[(size_t)j * nn + i];
        box2[((size_t)i * kBoxDims + j) * 2 + 1] = -bhi[(size_t)j * nn + i];
      }
    ix.tree.box2 = dalloc<float>(box2.size());
    up(ix.tree.box2, box2);
    ix.tree.centroid32T = dalloc<float>(c32t.empty() ? 1 : c32t.size());
    ix.tree.boxlo = dalloc<float>(blo.size());
    ix.tree.boxhi = dalloc<float>(bhi.size());
    up(ix.tree.centroid32T, c32t);
    up(ix.tree.boxlo, blo);
    up(ix.tree.boxhi, bhi);
    std::vector<int2> meta(nn);
    for (int i = 0; i < nn; ++i)
      meta[i] = t.n_children[i] > 0 ? make_int2(t.first_child[i], -t.n_children[i])
                                    : make_int2(t.leaf_start[i], t.leaf_count[i]);
    ix.tree.meta = dalloc<int2>(nn);
    up(ix.tree.meta, meta);
    for (int i = 0; i < nn; ++i) {
      r32[i] = std::nextafter((float)t.radius[i], INFINITY);
      double n2 = 0.0;
      for (int j = 0; j < d; ++j) n2 += t.centroid[(size_t)i * d + j] * t.centroid[(size_t)i * d + j];
      n32[i] = std::nextafter((float)(std::sqrt(n2) * (1.0 + 1e-12)), INFINITY);
    }
    ix.tree.centroid32 = dalloc<float>(c32.empty() ? 1 : c32.size());
    ix.tree.radius32 = dalloc<float>(nn);
    ix.tree.cnorm32 = dalloc<float>(nn);
    up(ix.tree.centroid32, c32);
    up(ix.tree.radius32, r32);
    up(ix.tree.cnorm32, n32);
  }
  if (!t.tie.empty()) {
    ix.tree.tie = dalloc<int32_t>(nn);
    up(ix.tree.tie, t.tie);
  }
  // pair-interleaved row blocks of the lane-group backtrack kernel
  if (d > 0 && d <= 64 && ix.tree.max_children <= 16) {
    const int dE = ix.dp;  // blocks padded to the fp32 layouts' width class
    ix.tree.centroid_il = dalloc<double>((size_t)nn * dE);
    launch_interleave_blocks(ctx, ix.tree.centroid, ix.tree.meta, nn, d, dE, false, nn,
                             ix.tree.centroid_il);
    ix.proj_leaf_il = dalloc<double>((size_t)ix.N * dE);
    launch_interleave_blocks(ctx, ix.proj_leaf, ix.tree.meta, nn, d, dE, true, ix.N,
                             ix.proj_leaf_il);
  }
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void finish_index(psg_ctx* ctx, Index& ix, const double* mean, const double* basis, int d,
                  const psg_index_cfg& cfg) {
  const int D = ix.D;
  const bool verbose = ctx->knobs.verbose;
  double t_phase = now_ms();
  auto phase = [&](const char* what) {
    if (!verbose) return;
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    const double t = now_ms();
    fprintf(stderr, "[persyn] index N=%lld D=%d: %s %.2f ms\n", (long long)ix.N, D, what, t - t_phase);
    t_phase = t;
  };
  if (basis) {
    if (d < 0 || d > kMaxDP) fail(PSG_E_DOMAIN, "injected PCA dimension must be in [0, 128]");
    ix.h_mean.assign(mean, mean + D);
    ix.h_basis.assign(basis, basis + (size_t)d * D);
    ix.h_var.assign(D, 0.0);
    ix.d = d;
  } else {
    fit_pca_device(ctx, ix, cfg);
  }
  d = ix.d;
  phase("pca fit");
  ix.mean = dalloc<double>(D);
  PSG_CUDA(cudaMemcpyAsync(ix.mean, ix.h_mean.data(), sizeof(double) * D, cudaMemcpyHostToDevice,
                           ctx->stream));
  // transposed, zero-padded basis [D][KP] for the projection kernel
  const int KP = d <= 32 ? 32 : (d <= 64 ? 64 : kMaxDP);
  std::vector<double> bt((size_t)D * KP, 0.0);
  for (int k = 0; k < d; ++k)
    for (int j = 0; j < D; ++j) bt[(size_t)j * KP + k] = ix.h_basis[(size_t)k * D + j];
  ix.basis = dalloc<double>(bt.size());
  PSG_CUDA(cudaMemcpyAsync(ix.basis, bt.data(), sizeof(double) * bt.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
  // the E-step's tensor-core projection operand (window indexes)
  if (!ix.from_vectors && d > 0) tc_prepare(ctx, ix);
  // project the database (pca.cpp:103-113)
  ix.proj = dalloc<double>((size_t)ix.N * (d > 0 ? d : 1));
  if (d > 0) {
    if (ix.from_vectors) {
      launch_project_vectors(ctx, ix.vectors, ix.N, D, ix.mean, ix.basis, d, ix.proj);
    } else {
      DBuf<int32_t> xs(ix.nxe), ys(ix.eh - ix.w + 1);
      std::vector<int32_t> hx(ix.nxe), hy(ix.eh - ix.w + 1);
      for (int i = 0; i < ix.nxe; ++i) hx[i] = i;
      for (int i = 0; i < ix.eh - ix.w + 1; ++i) hy[i] = i;
      xs.upload(ctx, hx.data(), hx.size());
      ys.upload(ctx, hy.data(), hy.size());
      AnchorSet as{xs.p, ys.p, ix.nxe, ix.N};
      launch_project_windows(ctx, ix.ex_mirror, ix.ew, ix.C, ix.w, as, ix.mean, ix.basis, d,
                             ix.proj);
      PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  }
  phase("db projection");
  // k-means tree over the device-projected points: the device tree, or the
  // reference's own KmTree::build replica (tree_kind, persyn_b200.h)
  const int lt = cfg.leaf_threshold > 0 ? cfg.leaf_threshold : cfg.branching;
  if (cfg.tree_kind == PSG_TREE_REFERENCE) {
    if (cfg.max_depth != 0) fail(PSG_E_DOMAIN, "the reference tree has no depth cap (max_depth 0)");
    std::vector<double> hp((size_t)ix.N * d);
    if (d > 0)
      PSG_CUDA(cudaMemcpyAsync(hp.data(), ix.proj, sizeof(double) * hp.size(),
                               cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    ix.htree = build_reference_tree_host(hp.data(), ix.N, d, cfg.branching, lt, cfg.seed);
    phase("tree build (reference replica)");
  } else if (cfg.tree_kind != PSG_TREE_DEVICE) {
    fail(PSG_E_DOMAIN, "unknown tree_kind");
  } else {
    ix.htree = build_tree_device(ctx, ix.proj, ix.N, d, cfg.branching, cfg.max_depth, lt, cfg.seed);
    phase("tree build (device)");
  }
  upload_tree(ctx, ix);
  phase("tree upload + search copies");
}

void build_exemplar_hist(psg_ctx* ctx, Index& ix, const double* ex_planes_dev, int bins,
                         int include_scale) {
  if (bins <= 0 || ix.from_vectors) return;
  if (bins < 2) fail(PSG_E_DOMAIN, "histogram bins must be >= 2");
  ix.hist_bins = bins;
  ix.hist_slots = include_scale ? ix.C : 3;
  const int n = bins * ix.hist_slots;
  DBuf<unsigned long long> counts(n);
  ix.ex_hist = dalloc<double>(n);
  const int64_t P = (int64_t)ix.ew * ix.eh;
  launch_hist_count(ctx, ex_planes_dev, P, P, bins, ix.hist_slots, counts.p);
  launch_hist_fold(ctx, counts.p, bins, ix.hist_slots, P, nullptr, ix.ex_hist, nullptr);
  ix.h_ex_hist.resize(n);
  PSG_CUDA(cudaMemcpyAsync(ix.h_ex_hist.data(), ix.ex_hist, sizeof(double) * n,
                           cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
}

std::unique_ptr<psg_index> create_index_from_device_planes(psg_ctx* ctx, const double* ex_dev,
                                                           int C, int ew, int eh, int w,
                                                           const double* mean,
                                                           const double* basis, int d,
                                                           const psg_index_cfg& cfg) {
  if (C < 4 || C > 8) fail(PSG_E_SHAPE, "channels must be 3 + G with G in [1, 5]");
  if (w < 2 || w % 2) fail(PSG_E_DOMAIN, "neighborhood width must be even and >= 2");
  if (ew < w || eh < w) fail(PSG_E_DOMAIN, "exemplar smaller than the neighborhood window");
  if (cfg.branching < 2) fail(PSG_E_DOMAIN, "tree branching must be >= 2");
  auto h = std::make_unique<psg_index>();
  Index& ix = h->impl;
  ix.ctx = ctx;
  ix.C = C;
  ix.w = w;
  ix.ew = ew;
  ix.eh = eh;
  ix.D = w * w * C;
  ix.nxe = ew - w + 1;
  ix.N = (int64_t)ix.nxe * (eh - w + 1);
  ix.ex_mirror = dalloc<float>((size_t)ew * eh * C);
  launch_make_mirror(ctx, ex_dev, C, ew, eh, ix.ex_mirror);
  if (C <= 8) {
    ix.ex_mirror8 = dalloc<float>((size_t)ew * eh * 8);
    launch_make_mirror8(ctx, ex_dev, C, ew, eh, ix.ex_mirror8);
  }
  build_exemplar_hist(ctx, ix, ex_dev, cfg.hist_bins, cfg.hist_include_scale);
  finish_index(ctx, ix, mean, basis, d, cfg);
  return h;
}

}  // namespace

// ---------------------------------------------------------------------------
// Level: device-resident EM state for one stage (optimize_level).
}  // namespace psg

struct psg_level {
  psg_ctx* ctx = nullptr;
  const psg::Index* ix = nullptr;
  int W = 0, H = 0, C = 0, w = 0;  // H: global image height
  psg_opt_cfg cfg{};
  psg_band band{};                 // owned rows / anchors (world = 1: everything)
  int Hl = 0, Hu = 0;              // local rows [p0, e1) allocated, owned rows [p0, p1)
  int nx = 0, ny = 0, nh = 0;      // local anchor rows (halo rows first), halo rows
  int64_t A = 0, Ao = 0, off = 0;  // local anchors, owned anchors, first owned anchor
  int64_t P = 0, nn_calls = 0;     // plane stride W*Hl, reference plan calls of owned anchors
  psg::DBuf<int32_t> xs, ys, col_lo, col_hi, row_lo, row_hi, mult;
  psg::DBuf<double> planes;
  psg::DBuf<float> mirror;
  psg::DBuf<double> qproj, d2, cur_dist, next_dist, irls, pen, eff, after;
  psg::DBuf<int32_t> cur_idx, next_idx;
  psg::DBuf<int64_t> scanned, exact_evals;
  psg::DBuf<int32_t> visited;
  psg::DBuf<unsigned long long> counts;
  psg::DBuf<double> out_mass, excess, ex_hist, stats_dev, pen_table;
  psg::DBuf<int32_t> tile_order;
  psg::DBuf<int32_t> resc_list;  // changed-only rescoring: the changed anchors
  psg::DBuf<int> resc_n;
  psg::DBuf<int32_t> ovf_list;   // backtrack(m > 2): queries re-run by the deep-stack kernel
  psg::DBuf<int> ovf_n;
  psg::DBuf<int32_t> ovf2_list;  // ... and the second (large-pool) pass's overflows
  psg::DBuf<int> ovf2_n;
  // tensor-core projection (kernels_project_tc.cu): digit mirror, per-query
  // error bands, ambiguous-query list and the exact fallback's compact buffers
  psg::DBuf<uint8_t> q8;
  psg::DBuf<int> q8_bad, amb_n;
  psg::DBuf<float> qdelta;
  psg::DBuf<int32_t> amb, amb_c0, amb_c1, full_anchor, seed_c;
  psg::DBuf<int> full_n;
  psg::DBuf<double> q_ex;
  // one EM iteration captured as a CUDA graph per cur/next parity (level_step)
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  double* stats_host = nullptr;  // pinned [8]
  bool hist_on = false;
  bool counts_fresh = false;  // L.counts = histogram of the current owned rows (fused M-step)
  int slots = 3;
  bool primed = false;
  bool scanned_valid = false;  // L.scanned holds a search of these anchors (tile order)
  bool stride2 = false;        // anchor columns 0, 2, 4, ... (tensor-core strip mode)
  int iter = 0;
  int64_t pending_calls = 0, pending_scanned = 0;
  double pending_ms = 0.0;
  int64_t unique_queries = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // psg_optimize_level with a pinned result buffer: the image is final after
  // the LAST iteration's M-step, so its download starts there, on the copy
  // stream, under that iteration's E-step
  double* early_host = nullptr;
  cudaEvent_t ev_early = nullptr;
  bool early_done = false;
  ~psg_level() {
    if (early_done && ctx) cudaStreamSynchronize(ctx->copy);  // the copy reads `planes`
    if (ev_early) cudaEventDestroy(ev_early);
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    if (stats_host && ctx) ctx->pinned_free.push_back(stats_host);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }
};

namespace psg {

// Row-band partition of the output.  Rank g owns anchor rows
// [a0, a1) and pixel rows [p0, p1); its windows read rows up to e1 (halo rows
// [p1, e1) come from rank g+1), and its pixels are also covered by anchor rows
// [hlo, a0) of rank g-1.  Accumulating those in ascending anchor id keeps the
// M-step bit-identical to one device.
psg_band shard_plan(int W, int H, int w, int sp, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) fail(PSG_E_DOMAIN, "bad rank / world size");
  validate_grid(w, sp, W, H);
  const auto ys = axis_positions(H, w, sp);
  const int ny = (int)ys.size();
  if (world > ny) fail(PSG_E_DOMAIN, "more ranks than anchor rows");
  auto a0_of = [&](int g) { return (int)((int64_t)g * ny / world); };
  auto p0_of = [&](int g) { return g == 0 ? 0 : ys[a0_of(g)]; };
  psg_band b{};
  b.W = W;
  b.H = H;
  b.w = w;
  b.spacing = sp;
  b.rank = rank;
  b.world = world;
  b.a0 = a0_of(rank);
  b.a1 = a0_of(rank + 1);
  b.p0 = p0_of(rank);
  b.p1 = rank == world - 1 ? H : p0_of(rank + 1);
  b.e1 = std::min(H, ys[b.a1 - 1] + w);
  b.hlo = (int)(std::lower_bound(ys.begin(), ys.end(), b.p0 - w + 1) - ys.begin());
  b.nx = (int)axis_positions(W, w, sp).size();
  b.ny = ny;
  if (rank > 0 && b.hlo < a0_of(rank - 1))
    fail(PSG_E_DOMAIN, "row band thinner than the window: halo anchors span two ranks");
  if (rank < world - 1 && b.e1 > (rank + 2 == world ? H : p0_of(rank + 2)))
    fail(PSG_E_DOMAIN, "row band thinner than the window: halo rows span two ranks");
  return b;
}

namespace {

void level_setup_band(psg_level& L, psg_ctx* ctx, const Index& ix, const psg_band& b,
                      const psg_opt_cfg& cfg, bool full) {
  L.ctx = ctx;
  L.ix = &ix;
  L.W = b.W;
  L.H = b.H;
  L.C = ix.C;
  L.w = ix.w;
  L.cfg = cfg;
  L.band = b;
  const int W = b.W, w = ix.w, sp = cfg.spacing;
  if (sp != b.spacing || w != b.w) fail(PSG_E_SHAPE, "band plan does not match the level");
  L.Hl = b.e1 - b.p0;
  L.Hu = b.p1 - b.p0;
  const auto hx = axis_positions(W, w, sp), hyg = axis_positions(b.H, w, sp);
  std::vector<int32_t> hy;  // local anchor rows [hlo, a1), y relative to p0 (halo < 0)
  for (int iy = b.hlo; iy < b.a1; ++iy) hy.push_back(hyg[iy] - b.p0);
  L.nx = (int)hx.size();
  L.ny = (int)hy.size();
  L.stride2 = !hx.empty() && hx[0] % 2 == 0;
  for (size_t i = 1; i < hx.size(); ++i) L.stride2 = L.stride2 && hx[i] - hx[i - 1] == 2;
  L.nh = b.a0 - b.hlo;
  L.A = (int64_t)L.nx * L.ny;
  L.off = (int64_t)L.nh * L.nx;
  L.Ao = L.A - L.off;
  L.P = (int64_t)W * L.Hl;
  L.xs.alloc(L.nx);
  L.ys.alloc(L.ny);
  L.xs.upload(ctx, hx.data(), hx.size());
  L.ys.upload(ctx, hy.data(), hy.size());
  // covering-anchor ranges: anchors a with a <= x < a + w (local coordinates)
  auto ranges = [&](const std::vector<int32_t>& v, int extent, std::vector<int32_t>& lo,
                    std::vector<int32_t>& hi) {
    lo.resize(extent);
    hi.resize(extent);
    for (int x = 0; x < extent; ++x) {
      lo[x] = (int32_t)(std::lower_bound(v.begin(), v.end(), x - w + 1) - v.begin());
      hi[x] = (int32_t)(std::upper_bound(v.begin(), v.end(), x) - v.begin());
    }
  };
  std::vector<int32_t> cl, ch, rl, rh;
  ranges(hx, W, cl, ch);
  ranges(hy, L.Hu, rl, rh);
  L.col_lo.alloc(W);
  L.col_hi.alloc(W);
  L.row_lo.alloc(L.Hu);
  L.row_hi.alloc(L.Hu);
  L.col_lo.upload(ctx, cl.data(), W);
  L.col_hi.upload(ctx, ch.data(), W);
  L.row_lo.upload(ctx, rl.data(), L.Hu);
  L.row_hi.upload(ctx, rh.data(), L.Hu);
  L.planes.alloc((size_t)L.P * L.C);
  L.mirror.alloc((size_t)L.P * L.C);
  L.cur_idx.alloc(L.A);
  L.cur_dist.alloc(L.A);
  L.irls.alloc(L.A);
  L.pen.alloc(L.A);
  L.eff.alloc(L.A);
  if (!full) return;
  std::vector<int32_t> m((size_t)L.nx * b.ny);
  const int64_t calls = plan_host(W, b.H, w, sp, cfg.patch_width, m.data());
  if (calls < 0) fail(PSG_E_LOGIC, "anchor not covered by any patch tile");
  std::vector<int32_t> mo(m.begin() + (size_t)b.a0 * L.nx, m.begin() + (size_t)b.a1 * L.nx);
  L.nn_calls = 0;
  for (int32_t v : mo) L.nn_calls += v;
  L.mult.alloc(L.Ao);
  L.mult.upload(ctx, mo.data(), L.Ao);
  L.qproj.alloc((size_t)L.Ao * (ix.d > 0 ? ix.d : 1));
  L.d2.alloc(L.Ao);
  L.next_idx.alloc(L.A);
  L.next_dist.alloc(L.A);
  L.after.alloc(L.A);
  L.scanned.alloc(L.Ao);
  L.exact_evals.alloc(L.Ao);
  L.visited.alloc(L.Ao);
  L.resc_list.alloc(L.Ao);
  L.resc_n.alloc(1);
  if (cfg.budget.mode != PSG_EXACT) {
    // the budget searches' escalation lists and the deep-stack scratch are
    // set up here, never inside a (possibly captured) iteration
    L.ovf_list.alloc(L.Ao);
    L.ovf_n.alloc(1);
    L.ovf2_list.alloc(L.Ao);
    L.ovf2_n.alloc(1);
    ensure_deep_scratch(ctx);
  }
  L.stats_dev.alloc(8 + 6 * 296);
  L.tile_order.alloc((size_t)image_tile_count(L.Ao, L.nx));
  if (ctx->pinned_free.empty()) {
    void* blk = nullptr;
    PSG_CUDA(cudaMallocHost(&blk, 64 * 64));
    ctx->pinned_blocks.push_back(blk);
    for (int i = 0; i < 64; ++i)
      ctx->pinned_free.push_back(reinterpret_cast<double*>(static_cast<char*>(blk) + 64 * i));
  }
  L.stats_host = ctx->pinned_free.back();
  ctx->pinned_free.pop_back();
  PSG_CUDA(cudaEventCreate(&L.ev0));
  PSG_CUDA(cudaEventCreate(&L.ev1));
}

void level_setup(psg_level& L, psg_ctx* ctx, const Index& ix, int W, int H,
                 const psg_opt_cfg& cfg, bool full) {
  level_setup_band(L, ctx, ix, shard_plan(W, H, ix.w, cfg.spacing, 0, 1), cfg, full);
}

void level_set_hist(psg_level& L, const double* ex_hist_host) {
  const Index& ix = *L.ix;
  L.hist_on = L.cfg.histogram_matching != 0 && (ex_hist_host || ix.ex_hist);
  if (!L.hist_on) return;
  L.slots = L.cfg.histogram_include_scale ? L.C : 3;
  const int n = L.cfg.histogram_bins * L.slots;
  L.ex_hist.alloc(n);
  if (ex_hist_host) {
    L.ex_hist.upload(L.ctx, ex_hist_host, n);
  } else {
    if (ix.hist_bins != L.cfg.histogram_bins || ix.hist_slots != L.slots)
      fail(PSG_E_SHAPE, "output/exemplar histograms disagree on bins or channels");
    PSG_CUDA(cudaMemcpyAsync(L.ex_hist.p, ix.ex_hist, sizeof(double) * n,
                             cudaMemcpyDeviceToDevice, L.ctx->stream));
  }
  L.counts.alloc(n);
  L.out_mass.alloc(n);
  L.excess.alloc(n);
  // per-candidate penalty table: worth it when anchors outnumber candidates
  if (ix.N > 0 && ix.N <= L.Ao) L.pen_table.alloc(ix.N);
}

AnchorSet owned_anchors(psg_level& L) { return AnchorSet{L.xs.p, L.ys.p + L.nh, L.nx, L.Ao}; }

// E-step over the owned anchors of the level's current (local) image.
// seed: per-owned-anchor exemplar ids evaluated first (only the bound; the
// result does not depend on it), or null.  seed_dist (optional): the full-D
// distances of the seed assignment on this same image (the lsq-after
// diagnostic) — anchors that keep their assignment reuse them.
void level_search(psg_level& L, const int32_t* seed, int32_t* out_idx, double* out_dist,
                  const double* seed_dist = nullptr, cudaEvent_t seed_dist_ready = nullptr) {
  if (!seed || L.ctx->knobs.rescore_all) seed_dist = nullptr;
  psg_ctx* ctx = L.ctx;
  const Index& ix = *L.ix;
  const AnchorSet as = owned_anchors(L);
  if (ix.brute) {  // BruteForceIndex: exact full-D scan on the tensor cores
    RowSrc qs;
    qs.base = L.mirror.p;
    qs.kind = 1;
    qs.img_w = L.W;
    qs.C = L.C;
    qs.w = L.w;
    qs.xs = as.xs;
    qs.ys = as.ys;
    qs.nx = as.nx;
    launch_brute_search(ctx, ix, qs, L.Ao, seed, out_idx + L.off, L.d2.p, L.scanned.p,
                        L.exact_evals.p);
    PSG_CUDA(cudaMemsetAsync(L.visited.p, 0, sizeof(int32_t) * L.Ao, ctx->stream));
    if (seed_dist_ready) PSG_CUDA(cudaStreamWaitEvent(ctx->stream, seed_dist_ready, 0));
    launch_rescore_windows(ctx, L.mirror.p, L.W, L.C, L.w, as, ix, out_idx + L.off,
                           out_dist + L.off, seed_dist ? seed : nullptr, seed_dist, L.resc_list.p,
                           L.resc_n.p);
    L.unique_queries += L.Ao;
    return;
  }
  // exact budget on the tile kernel: tensor-core projection with an error
  // band + exact fallback for the ambiguous queries (kernels_project_tc.cu)
  // (backtrack(m > 2) on the lane-group kernel takes the same projection: every
  // pop and the final winner are checked against the band)
  const bool tc = ix.tc && ix.d > 0 && !ctx->knobs.exact_projection &&
                  ((L.cfg.budget.mode == PSG_EXACT &&
                    search_uses_tiles(ctx, ix.tree, ix.d, true, L.Ao)) ||
                   (search_uses_groups(ctx, ix, L.cfg.budget) && !ctx->knobs.bt_exact_projection));
  const int64_t q8_slice = (int64_t)L.W * L.Hl * 8;
  if (tc) {
    if (!L.q8.p) {
      L.q8.alloc((size_t)4 * q8_slice);
      L.q8_bad.alloc(1);
      L.amb_n.alloc(1);
      L.qdelta.alloc((size_t)L.Ao);
      L.amb.alloc((size_t)L.Ao);
      L.amb_c0.alloc((size_t)L.Ao);
      L.amb_c1.alloc((size_t)L.Ao);
      L.full_anchor.alloc((size_t)L.Ao);
      L.full_n.alloc(1);
      L.seed_c.alloc((size_t)L.Ao);
      L.q_ex.alloc((size_t)L.Ao * ix.d);
    }
    PSG_CUDA(cudaMemsetAsync(L.q8_bad.p, 0, sizeof(int), ctx->stream));
    PSG_CUDA(cudaMemsetAsync(L.amb_n.p, 0, sizeof(int), ctx->stream));
    PSG_CUDA(cudaMemsetAsync(L.full_n.p, 0, sizeof(int), ctx->stream));
    launch_make_digits(ctx, L.mirror.p, L.C, L.W, L.Hl, L.q8.p, q8_slice, L.q8_bad.p);
    launch_project_windows_tc(ctx, L.q8.p, q8_slice, L.W, L.q8_bad.p, as, L.stride2, ix,
                              L.qproj.p, L.qdelta.p, L.cfg.spacing);
  } else if (ix.d > 0) {
    launch_project_windows(ctx, L.mirror.p, L.W, L.C, L.w, as, ix.mean, ix.basis, ix.d, L.qproj.p);
  }
  SearchArgs a{};
  a.q = L.qproj.p;
  a.nq = L.Ao;
  a.d = ix.d;
  a.seed_idx = L.cfg.budget.mode == PSG_EXACT ? seed : nullptr;
  a.proj = ix.proj;
  a.proj_soa = ix.proj_soa;
  a.proj_leaf = ix.proj_leaf;
  a.proj_leaf_il = ix.proj_leaf_il;
  a.proj32_q4 = ix.proj32_q4;
  a.pnorm32 = ix.pnorm32;
  a.pp32 = ix.pp32;
  a.pnorm_max = ix.pnorm_max;
  a.perm = ix.perm;
  a.qxs = L.xs.p;
  a.qys = L.ys.p + L.nh;
  a.qnx = L.nx;
  a.nxe = ix.nxe;
  a.nye = ix.eh - ix.w + 1;
  a.N = ix.N;
  a.tree = ix.tree;
  a.mode = L.cfg.budget.mode;
  a.max_leaves = L.cfg.budget.max_leaves;
  a.out_idx = out_idx + L.off;
  a.out_d2 = L.d2.p;
  a.out_scanned = L.scanned.p;
  a.out_exact = L.exact_evals.p;
  a.out_visited = L.visited.p;
  a.flags = ctx->d_flags;
  a.sched = ctx->d_sched;
  a.ovf_list = L.ovf_list.p;
  a.ovf_count = L.ovf_n.p;
  a.ovf2_list = L.ovf2_list.p;
  a.ovf2_count = L.ovf2_n.p;
  // unseeded exact search (the priming search of an unconverged image): a
  // greedy descent (one leaf per query) supplies the seeds, whose exact
  // distances start every query's bound (~4% faster priming search on the
  // bench stage); the result does not depend on the seeds
  DBuf<int32_t> greedy_seed;
  if (!a.seed_idx && a.mode == PSG_EXACT && !ctx->knobs.no_greedy_seed) {
    greedy_seed.alloc((size_t)L.Ao);
    SearchArgs g = a;
    g.mode = PSG_GREEDY;
    g.max_leaves = 1;
    g.out_idx = greedy_seed.p;
    g.out_exact = nullptr;
    g.out_visited = nullptr;
    g.qdelta = nullptr;
    launch_search(ctx, g);
    a.seed_idx = greedy_seed.p;
  }
  // seeded exact search: the previous search of these anchors left its
  // per-query scan counts in L.scanned -> schedule the costliest tiles first
  DBuf<int32_t>& order = L.tile_order;  // kept: no allocation inside a captured iteration
  if (a.seed_idx && !greedy_seed.p && a.mode == PSG_EXACT && L.scanned_valid &&
      !ctx->knobs.no_tile_order) {
    const size_t nt = (size_t)image_tile_count(a.nq, a.qnx);
    if (order.n < nt) order.alloc(nt);
    if (seed_dist_ready) {  // concurrent mode: the one-CTA sort overlaps the projection
      {
        SideScope side(ctx);
        launch_tile_order(ctx, L.scanned.p, a.nq, a.qnx, order.p);
      }
      PSG_CUDA(cudaEventRecord(ctx->ev_tile, ctx->side));
      PSG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_tile, 0));
    } else {
      launch_tile_order(ctx, L.scanned.p, a.nq, a.qnx, order.p);
    }
    a.tile_order = order.p;
  }
  if (tc) {
    a.qdelta = L.qdelta.p;
    a.amb_list = L.amb.p;
    a.amb_count = L.amb_n.p;
    a.amb_c0 = L.amb_c0.p;
    a.amb_c1 = L.amb_c1.p;
  }
  launch_search(ctx, a);
  if (tc) {
    // queries whose winner is not separated by their band: the reference's
    // exact projection chain, then the exact minimum over the two band
    // candidates -- or, when the band held more, an exact search seeded with
    // the band winner
    ResolveArgs rv{};
    rv.mirror = L.mirror.p;
    rv.img_w = L.W;
    rv.C = L.C;
    rv.w = L.w;
    rv.anchors = as;
    rv.list = L.amb.p;
    rv.count = L.amb_n.p;
    rv.c0 = L.amb_c0.p;
    rv.c1 = L.amb_c1.p;
    rv.idx = out_idx + L.off;
    rv.scanned = L.scanned.p;
    rv.exact = L.exact_evals.p;
    rv.full_anchor = L.full_anchor.p;
    rv.full_seed = L.seed_c.p;
    rv.full_count = L.full_n.p;
    rv.full_q = L.q_ex.p;
    launch_resolve(ctx, rv, ix);
    SearchArgs f = a;
    f.q = L.q_ex.p;
    f.nq_dev = L.full_n.p;
    f.qxs = nullptr;
    f.qys = nullptr;
    f.seed_idx = a.mode == PSG_EXACT ? L.seed_c.p : nullptr;
    f.out_map = L.full_anchor.p;  // results straight to the anchors
    f.out_idx = out_idx + L.off;
    f.out_d2 = nullptr;
    f.out_scanned = L.scanned.p;
    f.out_exact = L.exact_evals.p;
    f.out_visited = nullptr;
    f.qdelta = nullptr;
    f.amb_list = nullptr;
    f.amb_count = nullptr;
    f.amb_c0 = nullptr;
    f.amb_c1 = nullptr;
    f.tile_order = nullptr;
    launch_search(ctx, f);
    if (ctx->knobs.verbose) {
      int n[2] = {0, 0};
      PSG_CUDA(cudaMemcpyAsync(&n[0], L.amb_n.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      PSG_CUDA(cudaMemcpyAsync(&n[1], L.full_n.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      PSG_CUDA(cudaStreamSynchronize(ctx->stream));
      fprintf(stderr, "[persyn] search: %d of %lld queries settled exactly (near-ties), %d of them "
              "re-searched\n", n[0], (long long)L.Ao, n[1]);
    }
  }
  L.scanned_valid = true;
  if (seed_dist_ready) PSG_CUDA(cudaStreamWaitEvent(ctx->stream, seed_dist_ready, 0));
  launch_rescore_windows(ctx, L.mirror.p, L.W, L.C, L.w, as, ix, out_idx + L.off,
                         out_dist + L.off, seed_dist ? seed : nullptr, seed_dist, L.resc_list.p,
                         L.resc_n.p);
  L.unique_queries += L.Ao;
}

void level_read_stats(psg_level& L) {
  L.stats_dev.download(L.ctx, L.stats_host, 6);
  PSG_CUDA(cudaEventRecord(L.ev1, L.ctx->stream));
  check_flags(L.ctx);  // synchronizes the stream
}

// seed (optional, device, one id per owned anchor): see level_search.
void level_prime(psg_level& L, const int32_t* seed = nullptr) {
  if (L.primed) return;
  psg_ctx* ctx = L.ctx;
  PSG_CUDA(cudaEventRecord(L.ev0, ctx->stream));
  level_search(L, seed, L.cur_idx.p, L.cur_dist.p);
  StatsArgs s{};
  s.scanned = L.scanned.p;
  s.mult = L.mult.p;
  s.A = L.Ao;
  s.r = L.cfg.robust_exponent;
  s.out = L.stats_dev.p;
  launch_stats(ctx, s);
  level_read_stats(L);
  float ms = 0.f;
  PSG_CUDA(cudaEventElapsedTime(&ms, L.ev0, L.ev1));
  L.pending_calls = L.nn_calls;
  L.pending_scanned = (int64_t)L.stats_host[4];
  L.pending_ms = ms;
  L.primed = true;
}

MstepArgs mstep_args(psg_level& L) {
  const Index& ix = *L.ix;
  if (ix.N >= (1 << 24))  // mstep_kernel splits ids with a float reciprocal
    fail(PSG_E_DOMAIN, "exemplar has >= 2^24 candidate windows");
  MstepArgs m{};
  m.xs = L.xs.p;
  m.ys = L.ys.p;
  m.nx = L.nx;
  m.ny = L.ny;
  m.col_lo = L.col_lo.p;
  m.col_hi = L.col_hi.p;
  m.row_lo = L.row_lo.p;
  m.row_hi = L.row_hi.p;
  m.idx = L.cur_idx.p;
  m.eff = L.eff.p;
  m.W = L.W;
  m.H = L.Hu;
  m.plane_rows = L.Hl;
  m.C = L.C;
  m.w = L.w;
  m.sp = L.cfg.spacing;
  m.ex_mirror = ix.ex_mirror;
  m.ex8 = L.ctx->knobs.no_ex8 ? nullptr : ix.ex_mirror8;
  m.ew = ix.ew;
  m.nxe = ix.nxe;
  m.planes = L.planes.p;
  m.mirror = L.mirror.p;
  m.flags = L.ctx->d_flags;
  return m;
}

// ---- one EM iteration in four phases (optimizer.cpp:453-497); the exchanges
// of a row-sharded run happen between them (paper_2006_11851_b200/sharding.py).

// Phase 1: IRLS weights of the owned anchors; local histogram counts of the
// owned pixel rows (the caller sums them over ranks: exact integers).
// side: the weights kernel goes to the side stream (joined by ctx->ev_join
// before the effective weights are formed, see phase_penalty).
void phase_weights(psg_level& L, bool side = false, bool mark = true) {
  psg_ctx* ctx = L.ctx;
  if (mark) PSG_CUDA(cudaEventRecord(L.ev0, ctx->stream));  // iteration timer
  if (side) {
    PSG_CUDA(cudaEventRecord(ctx->ev_fork, ctx->stream));
    PSG_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
  }
  WeightArgs wa{};
  wa.dist = L.cur_dist.p + L.off;
  wa.idx = L.cur_idx.p + L.off;
  wa.pen = nullptr;
  wa.A = L.Ao;
  wa.r = L.cfg.robust_exponent;
  wa.eps = L.cfg.distance_epsilon;
  wa.irls = L.irls.p + L.off;
  wa.eff = L.eff.p + L.off;
  wa.flags = ctx->d_flags;
  if (side) {
    {
      SideScope sc(ctx);
      launch_weights(ctx, wa);
    }
    PSG_CUDA(cudaEventRecord(ctx->ev_join, ctx->side));
  } else {
    launch_weights(ctx, wa);
  }
  if (L.hist_on && !L.counts_fresh)
    launch_hist_count(ctx, L.planes.p, (int64_t)L.W * L.Hu, L.P, L.cfg.histogram_bins, L.slots,
                      L.counts.p);
  L.counts_fresh = false;
}

// Phase 2: fold the global counts (1/P over the WHOLE image), penalties and
// effective weights of the owned anchors.
// weights_ready: event the IRLS weights were recorded on (side stream), or null.
void phase_penalty(psg_level& L, const unsigned long long* global_counts,
                   cudaEvent_t weights_ready = nullptr) {
  psg_ctx* ctx = L.ctx;
  if (!L.hist_on) {
    if (weights_ready) PSG_CUDA(cudaStreamWaitEvent(ctx->stream, weights_ready, 0));
    return;
  }
  const int bins = L.cfg.histogram_bins;
  launch_hist_fold(ctx, global_counts, bins, L.slots, (int64_t)L.W * L.H, L.ex_hist.p,
                   L.out_mass.p, L.excess.p);
  if (L.pen_table.p && !ctx->knobs.penalty_per_anchor) {
    launch_penalty_table(ctx, *L.ix, L.excess.p, bins, L.slots, L.pen_table.p);
    if (weights_ready) PSG_CUDA(cudaStreamWaitEvent(ctx->stream, weights_ready, 0));
    launch_eff_gather(ctx, L.irls.p + L.off, L.pen_table.p, L.cur_idx.p + L.off, L.Ao,
                      L.pen.p + L.off, L.eff.p + L.off, ctx->d_flags);
    return;
  }
  launch_penalty(ctx, *L.ix, L.cur_idx.p + L.off, L.Ao, L.excess.p, bins, L.slots,
                 L.pen.p + L.off);
  if (weights_ready) PSG_CUDA(cudaStreamWaitEvent(ctx->stream, weights_ready, 0));
  launch_eff_from(ctx, L.irls.p + L.off, L.pen.p + L.off, L.Ao, L.eff.p + L.off, ctx->d_flags);
}

// Phase 3: M-step of the owned pixel rows (halo anchor rows must be filled).
void phase_update(psg_level& L) {
  MstepArgs m = mstep_args(L);
  if (L.hist_on && !L.ctx->knobs.no_fused_hist) {
    // the next phase 1 histograms exactly the rows this M-step writes
    m.counts = L.counts.p;
    m.bins = L.cfg.histogram_bins;
    m.slots = L.slots;
  }
  launch_mstep(L.ctx, m);
  L.counts_fresh = m.counts != nullptr;
}

// Phase 4: lsq diagnostic, E-step, telemetry partials of the owned anchors.
void phase_search_enqueue(psg_level& L) {
  psg_ctx* ctx = L.ctx;
  // the lsq diagnostic (L1-bound) runs on the side stream, overlapping the
  // projection (fp64-bound); the post-search rescoring waits for it.  Serial
  // when profiling (per-launch events live on the main stream).
  const bool conc = ctx->side && !ctx->profile && !ctx->knobs.serial;
  cudaEvent_t ready = nullptr;
  if (conc) {
    PSG_CUDA(cudaEventRecord(ctx->ev_fork, ctx->stream));
    PSG_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    {
      SideScope side(ctx);
      launch_rescore_windows(ctx, L.mirror.p, L.W, L.C, L.w, owned_anchors(L), *L.ix,
                             L.cur_idx.p + L.off, L.after.p + L.off);
    }
    PSG_CUDA(cudaEventRecord(ctx->ev_join, ctx->side));
    ready = ctx->ev_join;
  } else {
    launch_rescore_windows(ctx, L.mirror.p, L.W, L.C, L.w, owned_anchors(L), *L.ix,
                           L.cur_idx.p + L.off, L.after.p + L.off);
  }
  level_search(L, L.cur_idx.p + L.off, L.next_idx.p, L.next_dist.p, L.after.p + L.off, ready);
  if (ready) PSG_CUDA(cudaStreamWaitEvent(ctx->stream, ready, 0));  // stats read `after`
  StatsArgs s{};
  s.cur_dist = L.cur_dist.p + L.off;
  s.after_dist = L.after.p + L.off;
  s.eff = L.eff.p + L.off;
  s.next_dist = L.next_dist.p + L.off;
  s.cur_idx = L.cur_idx.p + L.off;
  s.next_idx = L.next_idx.p + L.off;
  s.scanned = L.scanned.p;
  s.mult = L.mult.p;
  s.A = L.Ao;
  s.r = L.cfg.robust_exponent;
  s.out = L.stats_dev.p;
  launch_stats(ctx, s);
}

void phase_search(psg_level& L) {
  phase_search_enqueue(L);
  level_read_stats(L);
}

// Closes the iteration: stats record, swap current/next assignments.
// stats_host holds this rank's partials; `global` (may alias) the summed ones.
void phase_commit(psg_level& L, const double* global, psg_iter_stats* st) {
  float ms = 0.f;
  PSG_CUDA(cudaEventElapsedTime(&ms, L.ev0, L.ev1));
  ++L.iter;
  if (st) {
    st->iteration = L.iter;
    st->energy = global[2];
    st->changed = (int64_t)global[3];
    st->nn_calls = (int64_t)global[6] + (int64_t)global[7];
    st->millis = ms + L.pending_ms;
    st->lsq_energy_before = global[0];
    st->lsq_energy_after = global[1];
    st->points_scanned = (int64_t)global[4];
    st->unique_queries = (int64_t)global[8];
    st->unique_points_scanned = (int64_t)global[5];
  }
  L.pending_calls = 0;
  L.pending_scanned = 0;
  L.pending_ms = 0.0;
  std::swap(L.cur_idx, L.next_idx);
  std::swap(L.cur_dist, L.next_dist);
}

// This rank's telemetry partials {lsq_before, lsq_after, energy, changed,
// points_scanned (plan-weighted, incl. priming), unique points scanned,
// nn_calls, pending priming nn_calls, unique queries}.
void phase_partials(psg_level& L, double out[9]) {
  for (int k = 0; k < 6; ++k) out[k] = L.stats_host[k];
  out[4] += (double)L.pending_scanned;
  out[6] = (double)L.nn_calls;
  out[7] = (double)L.pending_calls;
  out[8] = (double)(L.Ao * (L.pending_calls ? 2 : 1));
}

// One EM iteration on a single device (optimizer.cpp:450-513).  Returns true
// when converged under the reference's rule.
// The device work of one iteration, up to the stats read-back into pinned
// memory (plus the device flags into the pinned slot's last word).
// mark: record the iteration timer events (not inside a graph: events
// recorded by graph nodes cannot be timed).
void step_body(psg_level& L, bool conc, bool mark) {
  psg_ctx* ctx = L.ctx;
  phase_weights(L, conc, mark);
  phase_penalty(L, L.counts.p, conc ? ctx->ev_join : nullptr);
  phase_update(L);
  if (mark && L.early_host && !L.early_done && L.iter + 1 >= L.cfg.max_iterations) {
    if (!L.ev_early) PSG_CUDA(cudaEventCreateWithFlags(&L.ev_early, cudaEventDisableTiming));
    PSG_CUDA(cudaEventRecord(L.ev_early, ctx->stream));
    PSG_CUDA(cudaStreamWaitEvent(ctx->copy, L.ev_early, 0));
    PSG_CUDA(cudaMemcpyAsync(L.early_host, L.planes.p, sizeof(double) * (size_t)L.P * L.C,
                             cudaMemcpyDeviceToHost, ctx->copy));
    L.early_done = true;
  }
  phase_search_enqueue(L);
  L.stats_dev.download(ctx, L.stats_host, 6);
  PSG_CUDA(cudaMemcpyAsync(reinterpret_cast<int*>(L.stats_host + 7), ctx->d_flags, sizeof(int),
                           cudaMemcpyDeviceToHost, ctx->stream));
  if (mark) PSG_CUDA(cudaEventRecord(L.ev1, ctx->stream));
}

bool level_step(psg_level& L, psg_iter_stats* st, bool honor) {
  psg_ctx* ctx = L.ctx;
  // IRLS weights (side stream) overlap the histogram fold + penalty table
  const bool conc = ctx->side && !ctx->profile && !ctx->knobs.serial;
  // opt-in (PERSYN_GRAPH=1): one graph launch per iteration in the steady
  // state (same topology once the fused M-step keeps the counts fresh).
  // Measured on the bench stage: +0.3% iterations/s, but -2% e2e (two graph
  // instantiations per level), so launches stay eager by default.
  const bool graph = conc && ctx->knobs.graph && (!L.hist_on || L.counts_fresh);
  if (graph) {
    cudaGraphExec_t& ge = L.graph[L.iter & 1];
    if (!ge) {
      cudaGraph_t gr = nullptr;
      PSG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
      try {
        step_body(L, conc, false);
      } catch (...) {
        cudaStreamEndCapture(ctx->stream, &gr);
        if (gr) cudaGraphDestroy(gr);
        throw;
      }
      PSG_CUDA(cudaStreamEndCapture(ctx->stream, &gr));
      PSG_CUDA(cudaGraphInstantiate(&ge, gr, 0));
      PSG_CUDA(cudaGraphDestroy(gr));
      L.unique_queries -= L.Ao;  // the capture ran the host bookkeeping once
    }
    PSG_CUDA(cudaEventRecord(L.ev0, ctx->stream));
    PSG_CUDA(cudaGraphLaunch(ge, ctx->stream));
    PSG_CUDA(cudaEventRecord(L.ev1, ctx->stream));
    // host bookkeeping of the captured body (level_search, phase_update)
    L.unique_queries += L.Ao;
    L.counts_fresh = L.hist_on;
  } else {
    step_body(L, conc, true);
  }
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  prof_flush(ctx);
  const int f = *reinterpret_cast<const int*>(L.stats_host + 7);
  if (f) check_flags(ctx);  // re-reads, clears and raises
  double g[9];
  phase_partials(L, g);
  phase_commit(L, g, st);
  const int64_t changed = (int64_t)g[3];
  return honor && L.iter >= L.cfg.min_iterations &&
         (double)changed < L.cfg.convergence_fraction * (double)L.Ao;
}

// Host rows [p0, e1) of the global image (planes [C][Hl][W]).
// Device rows [p0, e1) of the global image (planes [C][Hl][W]).
void upload_state_dev(psg_level& L, const double* dev_planes) {
  L.counts_fresh = false;
  PSG_CUDA(cudaMemcpyAsync(L.planes.p, dev_planes, sizeof(double) * (size_t)L.P * L.C,
                           cudaMemcpyDeviceToDevice, L.ctx->stream));
  launch_make_mirror(L.ctx, L.planes.p, L.C, L.W, L.Hl, L.mirror.p);
}

void upload_state(psg_level& L, const double* host_planes) {
  L.counts_fresh = false;
  L.planes.upload(L.ctx, host_planes, (size_t)L.P * L.C);
  launch_make_mirror(L.ctx, L.planes.p, L.C, L.W, L.Hl, L.mirror.p);
}

}  // namespace
}  // namespace psg

namespace psg {
// BruteForceIndex over an exemplar already on the device (psg_index_create_brute,
// psg_synthesize with index_kind = brute force).
std::unique_ptr<psg_index> create_brute_from_device_planes(psg_ctx* ctx, const double* ex_dev,
                                                           int C, int ew, int eh, int w,
                                                           int hist_bins, int hist_include_scale) {
  if (w < 2 || w % 2) fail(PSG_E_DOMAIN, "neighborhood width must be even and >= 2");
  if (ew < w || eh < w) fail(PSG_E_DOMAIN, "exemplar smaller than the neighborhood window");
  auto h = std::make_unique<psg_index>();
  Index& ix = h->impl;
  ix.ctx = ctx;
  ix.brute = true;
  ix.C = C;
  ix.w = w;
  ix.ew = ew;
  ix.eh = eh;
  ix.D = w * w * C;
  ix.nxe = ew - w + 1;
  ix.N = (int64_t)ix.nxe * (eh - w + 1);
  ix.ex_mirror = dalloc<float>((size_t)ew * eh * C);
  launch_make_mirror(ctx, ex_dev, C, ew, eh, ix.ex_mirror);
  if (C <= 8) {
    ix.ex_mirror8 = dalloc<float>((size_t)ew * eh * 8);
    launch_make_mirror8(ctx, ex_dev, C, ew, eh, ix.ex_mirror8);
  }
  build_exemplar_hist(ctx, ix, ex_dev, hist_bins, hist_include_scale);
  brute_prepare(ctx, ix);
  return h;
}
}  // namespace psg

// ===========================================================================
// C ABI
// ===========================================================================
using psg::fail;

template <class F>
static psg_status guarded(F&& f) {
  try {
    f();
    return PSG_OK;
  } catch (const psg::Error& e) {
    psg::g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    psg::g_last_error = std::string("allocation failure: ") + e.what();
    return PSG_E_CUDA;
  } catch (const std::exception& e) {
    psg::g_last_error = e.what();
    return PSG_E_LOGIC;
  }
}

extern "C" {

const char* psg_last_error(void) { return psg::g_last_error.c_str(); }
int psg_abi_version(void) { return PSG_ABI_VERSION; }

psg_status psg_ctx_create(int device, void* stream, psg_ctx** out) {
  return guarded([&] {
    if (!out) fail(PSG_E_DOMAIN, "null output handle");
    *out = nullptr;
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      fail(PSG_E_CUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) fail(PSG_E_DOMAIN, "device ordinal out of range");
    PSG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    PSG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(PSG_E_CUDA, "persyn_b200 is built for sm_100a (B200); device reports sm_" +
                           std::to_string(prop.major) + std::to_string(prop.minor));
    auto c = std::make_unique<psg_ctx>();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    {
      auto on = [](const char* k) { return std::getenv(k) != nullptr; };
      auto& kn = c->knobs;
      const char* e = std::getenv("PERSYN_SEARCH");
      kn.legacy_search = e && std::string(e) == "warp";
      kn.verbose = on("PERSYN_VERBOSE");
      kn.rescore_all = on("PERSYN_RESCORE_ALL");
      kn.no_greedy_seed = on("PERSYN_NO_GREEDY_SEED");
      kn.no_tile_order = on("PERSYN_NO_TILE_ORDER");
      kn.no_ex8 = on("PERSYN_NO_EX8");
      kn.penalty_per_anchor = on("PERSYN_PENALTY_PER_ANCHOR");
      kn.no_fused_hist = on("PERSYN_NO_FUSED_HIST");
      kn.serial = on("PERSYN_SERIAL");
      kn.graph = on("PERSYN_GRAPH");
      kn.project_kpt2 = on("PERSYN_PROJECT_KPT2");
      kn.no_carry = on("PERSYN_NO_CARRY");
      kn.eig_direct = on("PERSYN_EIG");
      kn.exact_projection = on("PERSYN_EXACT_PROJECTION");
      kn.bt_warp = on("PERSYN_BT_WARP");
      kn.bt_thread = on("PERSYN_BT_THREAD");
      kn.no_build_ahead = on("PERSYN_NO_BUILD_AHEAD");
      kn.no_early_download = on("PERSYN_NO_EARLY_DOWNLOAD");
      kn.bt_exact_projection = on("PERSYN_BT_EXACT_PROJECTION");
    }
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      PSG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    {
      cudaMemPool_t pool;
      PSG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = UINT64_MAX;
      PSG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    PSG_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    PSG_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&c->ev_fork, &c->ev_join, &c->ev_tile})
      PSG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    PSG_CUDA(cudaMalloc(&c->d_flags, sizeof(int)));
    PSG_CUDA(cudaMemsetAsync(c->d_flags, 0, sizeof(int), c->stream));
    PSG_CUDA(cudaMalloc(&c->d_sched, 4 * sizeof(int64_t)));  // [2]: stats fold ticket
    PSG_CUDA(cudaMemsetAsync(c->d_sched, 0, 4 * sizeof(int64_t), c->stream));
    psg::create_solver_handles(c.get());  // once per context, not inside a stage build
    *out = c.release();
  });
}

void psg_ctx_destroy(psg_ctx* ctx) {
  if (!ctx) return;
  for (psg_ctx* b : ctx->builders) psg_ctx_destroy(b);
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->copy) {
    cudaStreamSynchronize(ctx->copy);
    cudaStreamDestroy(ctx->copy);
  }
  for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_join, ctx->ev_tile})
    if (e) cudaEventDestroy(e);
  if (ctx->cublas) cublasDestroy(static_cast<cublasHandle_t>(ctx->cublas));
  if (ctx->cusolver) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(ctx->cusolver));
  cudaFree(ctx->d_flags);
  if (ctx->deep_key) cudaFree(ctx->deep_key);
  if (ctx->deep_node) cudaFree(ctx->deep_node);
  cudaFree(ctx->d_sched);
  for (void* b : ctx->pinned_blocks) cudaFreeHost(b);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

psg_status psg_ctx_synchronize(psg_ctx* ctx) {
  return guarded([&] { PSG_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int64_t psg_ctx_launch_count(const psg_ctx* ctx) { return ctx ? ctx->launches : -1; }

psg_status psg_ctx_profile(psg_ctx* ctx, int enable) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx) fail(PSG_E_DOMAIN, "null context");
    psg::prof_flush(ctx);
    ctx->profile = enable != 0;
    for (int k = 0; k < psg::K_COUNT; ++k) {
      ctx->kernel_ms[k] = 0.0;
      ctx->kernel_launches[k] = 0;
    }
  });
}

int psg_ctx_kernel_times(psg_ctx* ctx, const char** names, double* ms, int64_t* launches, int n) {
  if (!ctx) return 0;
  try {
    psg::prof_flush(ctx);
  } catch (...) {
  }
  for (int k = 0; k < psg::K_COUNT && k < n; ++k) {
    if (names) names[k] = psg::kKernelNames[k];
    if (ms) ms[k] = ctx->kernel_ms[k];
    if (launches) launches[k] = ctx->kernel_launches[k];
  }
  return psg::K_COUNT;
}

psg_status psg_index_create(psg_ctx* ctx, const double* ex_planes, int C, int ew, int eh, int w,
                            const double* mean, const double* basis, int d,
                            const psg_index_cfg* cfg, psg_index** out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !ex_planes || !cfg || !out) fail(PSG_E_DOMAIN, "null argument");
    *out = nullptr;
    if (ew < 1 || eh < 1) fail(PSG_E_DOMAIN, "empty exemplar");
    psg::DBuf<double> ex((size_t)C * ew * eh);
    ex.upload(ctx, ex_planes, ex.n);
    auto h = psg::create_index_from_device_planes(ctx, ex.p, C, ew, eh, w, mean, basis, d, *cfg);
    *out = h.release();
  });
}

psg_status psg_index_create_vectors(psg_ctx* ctx, const float* X, int64_t n, int D,
                                    const double* mean, const double* basis, int d,
                                    const psg_index_cfg* cfg, psg_index** out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !X || !cfg || !out) fail(PSG_E_DOMAIN, "null argument");
    *out = nullptr;
    if (n < 1) fail(PSG_E_DOMAIN, "empty candidate set");
    if (D < 1) fail(PSG_E_DOMAIN, "vector dimension must be >= 1");
    auto h = std::make_unique<psg_index>();
    psg::Index& ix = h->impl;
    ix.ctx = ctx;
    ix.from_vectors = true;
    ix.D = D;
    ix.N = n;
    ix.nxe = 1;
    ix.vectors = psg::dalloc<float>((size_t)n * D);
    PSG_CUDA(cudaMemcpyAsync(ix.vectors, X, sizeof(float) * (size_t)n * D, cudaMemcpyHostToDevice,
                             ctx->stream));
    psg::finish_index(ctx, ix, mean, basis, d, *cfg);
    *out = h.release();
  });
}

psg_status psg_index_create_brute(psg_ctx* ctx, const double* ex_planes, int C, int ew, int eh,
                                  int w, int hist_bins, int hist_include_scale, psg_index** out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !ex_planes || !out) fail(PSG_E_DOMAIN, "null argument");
    *out = nullptr;
    if (ew < 1 || eh < 1) fail(PSG_E_DOMAIN, "empty exemplar");
    if (C < 4 || C > 8) fail(PSG_E_SHAPE, "channels must be 3 + G with G in [1, 5]");
    psg::DBuf<double> ex((size_t)C * ew * eh);
    ex.upload(ctx, ex_planes, ex.n);
    *out = psg::create_brute_from_device_planes(ctx, ex.p, C, ew, eh, w, hist_bins,
                                                hist_include_scale)
               .release();
  });
}

psg_status psg_index_create_brute_vectors(psg_ctx* ctx, const float* X, int64_t n, int D,
                                          psg_index** out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !X || !out) fail(PSG_E_DOMAIN, "null argument");
    *out = nullptr;
    if (n < 1) fail(PSG_E_DOMAIN, "empty candidate set");  // optimizer.cpp:171
    if (D < 1) fail(PSG_E_DOMAIN, "vector dimension must be >= 1");
    auto h = std::make_unique<psg_index>();
    psg::Index& ix = h->impl;
    ix.ctx = ctx;
    ix.brute = true;
    ix.from_vectors = true;
    ix.D = D;
    ix.N = n;
    ix.nxe = 1;
    ix.vectors = psg::dalloc<float>((size_t)n * D);
    PSG_CUDA(cudaMemcpyAsync(ix.vectors, X, sizeof(float) * (size_t)n * D, cudaMemcpyHostToDevice,
                             ctx->stream));
    psg::brute_prepare(ctx, ix);
    *out = h.release();
  });
}

void psg_index_destroy(psg_index* index) { delete index; }

psg_status psg_index_info(const psg_index* index, int64_t dims[10]) {
  return guarded([&] {
    const psg::Index& ix = index->impl;
    const int64_t v[10] = {ix.N, ix.D, ix.d, ix.C, ix.w, ix.ew, ix.eh, ix.tree.n_nodes,
                           ix.htree.n_leaves, ix.tree.max_depth};
    std::memcpy(dims, v, sizeof(v));
  });
}

psg_status psg_index_pca(const psg_index* index, double* mean, double* basis, double* variances) {
  return guarded([&] {
    const psg::Index& ix = index->impl;
    if (mean) std::copy(ix.h_mean.begin(), ix.h_mean.end(), mean);
    if (basis) std::copy(ix.h_basis.begin(), ix.h_basis.end(), basis);
    if (variances) std::copy(ix.h_var.begin(), ix.h_var.end(), variances);
  });
}

psg_status psg_index_projected(const psg_index* index, double* out) {
  return guarded([&] {
    const psg::Index& ix = index->impl;
    if (ix.d > 0) {
      PSG_CUDA(cudaMemcpyAsync(out, ix.proj, sizeof(double) * ix.N * ix.d, cudaMemcpyDeviceToHost,
                               ix.ctx->stream));
      PSG_CUDA(cudaStreamSynchronize(ix.ctx->stream));
    }
  });
}

psg_status psg_index_leaves(const psg_index* index, int32_t* ids, int32_t* sizes,
                            int64_t* n_leaves) {
  return guarded([&] {
    const psg::HostTree& t = index->impl.htree;
    *n_leaves = t.n_leaves;
    int64_t li = 0, off = 0;
    for (size_t i = 0; i < t.n_children.size(); ++i) {  // leaves in node (BFS) order
      if (t.n_children[i] != 0) continue;
      if (sizes) sizes[li] = t.leaf_count[i];
      if (ids)
        std::copy(t.perm.begin() + t.leaf_start[i], t.perm.begin() + t.leaf_start[i] + t.leaf_count[i],
                  ids + off);
      off += t.leaf_count[i];
      ++li;
    }
  });
}

psg_status psg_reference_tree_host(const double* proj, int64_t N, int d, int branching,
                                   int leaf_threshold, uint64_t seed, int32_t* n_children,
                                   int64_t* n_nodes, int32_t* leaf_sizes, int64_t* n_leaves,
                                   int32_t* leaf_ids) {
  return guarded([&] {
    if (!proj || !n_children || !n_nodes || !leaf_sizes || !n_leaves || !leaf_ids)
      fail(PSG_E_DOMAIN, "null argument");
    std::vector<int32_t> nc, ls, li;
    psg::reference_tree_walk(proj, N, d, branching, leaf_threshold, seed, nc, ls, li);
    std::copy(nc.begin(), nc.end(), n_children);
    std::copy(ls.begin(), ls.end(), leaf_sizes);
    std::copy(li.begin(), li.end(), leaf_ids);
    *n_nodes = (int64_t)nc.size();
    *n_leaves = (int64_t)ls.size();
  });
}

psg_status psg_index_import_tree(psg_ctx* ctx, psg_index* index, const psg_tree_import* tree) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !index || !tree || !tree->n_children || !tree->leaf_sizes || !tree->leaf_ids)
      fail(PSG_E_DOMAIN, "null argument");
    psg::Index& ix = index->impl;
    if (ix.d < 1) fail(PSG_E_DOMAIN, "tree import needs a PCA dimension >= 1");
    std::vector<double> hp((size_t)ix.N * ix.d);
    PSG_CUDA(cudaMemcpyAsync(hp.data(), ix.proj, sizeof(double) * hp.size(),
                             cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    ix.htree = psg::import_tree_host(hp.data(), ix.N, ix.d, tree->n_children, tree->n_nodes,
                                     tree->leaf_sizes, tree->n_leaves, tree->leaf_ids);
    psg::upload_tree(ctx, ix);
  });
}

psg_status psg_index_histograms(const psg_index* index, double* mass) {
  return guarded([&] {
    const psg::Index& ix = index->impl;
    if (ix.h_ex_hist.empty()) fail(PSG_E_DOMAIN, "index was built without a histogram");
    std::copy(ix.h_ex_hist.begin(), ix.h_ex_hist.end(), mass);
  });
}

psg_status psg_index_query(psg_ctx* ctx, const psg_index* index, const float* Q, int64_t nq,
                           psg_budget budget, int32_t* idx, double* dist, double* dist_pca,
                           int64_t* scanned) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !index || !Q || !idx || !dist) fail(PSG_E_DOMAIN, "null argument");
    psg::validate_budget(budget);
    const psg::Index& ix = index->impl;
    if (nq <= 0) return;
    psg::DBuf<float> q((size_t)nq * ix.D);
    q.upload(ctx, Q, q.n);
    psg::DBuf<double> qp((size_t)nq * (ix.d > 0 ? ix.d : 1)), d2(nq), dd(nq);
    psg::DBuf<int32_t> id(nq);
    psg::DBuf<int64_t> sc(nq);
    if (ix.brute) {
      psg::RowSrc qs;
      qs.base = q.p;
      qs.kind = 0;
      qs.D = ix.D;
      psg::launch_brute_search(ctx, ix, qs, nq, nullptr, id.p, d2.p, sc.p, nullptr);
    }
    if (ix.d > 0) psg::launch_project_vectors(ctx, q.p, nq, ix.D, ix.mean, ix.basis, ix.d, qp.p);
    psg::SearchArgs a{};
    a.q = qp.p;
    a.nq = nq;
    a.d = ix.d;
    a.proj = ix.proj;
    a.proj_soa = ix.proj_soa;
    a.proj_leaf = ix.proj_leaf;
    a.proj_leaf_il = ix.proj_leaf_il;
    a.proj32_q4 = ix.proj32_q4;
    a.pnorm32 = ix.pnorm32;
    a.pp32 = ix.pp32;
    a.pnorm_max = ix.pnorm_max;
    a.perm = ix.perm;
    a.N = ix.N;
    a.tree = ix.tree;
    a.mode = budget.mode;
    a.max_leaves = budget.max_leaves;
    a.out_idx = id.p;
    a.out_d2 = d2.p;
    a.out_scanned = sc.p;
    a.flags = ctx->d_flags;
    a.sched = ctx->d_sched;
    const bool reorder = budget.mode == PSG_EXACT && nq >= 64 && ix.d > 0 && !ctx->knobs.legacy_search;
    if (ix.brute) {
      // searched above (the budget does not apply, optimizer.cpp:172-173)
    } else if (reorder) {
      // tiles of 32 queries share a traversal: give them neighbours in the tree
      psg::DBuf<uint32_t> k0(nq), k1(nq);
      psg::DBuf<int32_t> o0(nq), o1(nq), id_s(nq);
      psg::DBuf<double> qs((size_t)nq * ix.d), d2_s(nq);
      psg::DBuf<int64_t> sc_s(nq);
      psg::launch_greedy_keys(ctx, qp.p, nq, ix.d, ix.tree, k0.p, o0.p);
      const size_t tb = psg::sort_pairs_temp_bytes(nq);
      psg::DBuf<char> tmp(tb ? tb : 1);
      psg::sort_pairs_u32(ctx, k0.p, k1.p, o0.p, o1.p, nq, tmp.p, tb);
      psg::launch_gather_rows_f64(ctx, qp.p, o1.p, nq, ix.d, qs.p);
      a.q = qs.p;
      a.out_idx = id_s.p;
      a.out_d2 = d2_s.p;
      a.out_scanned = sc_s.p;
      psg::launch_search(ctx, a);
      psg::launch_scatter_i32(ctx, id_s.p, o1.p, nq, id.p);
      psg::launch_scatter_f64(ctx, d2_s.p, o1.p, nq, d2.p);
      psg::launch_scatter_i64(ctx, sc_s.p, o1.p, nq, sc.p);
      PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
      psg::launch_search(ctx, a);
    }
    if (ix.from_vectors) {
      psg::launch_rescore_vectors(ctx, q.p, nq, ix, id.p, dd.p);
    } else {
      // window index queried with explicit vectors: rescore against the
      // candidate window gathered from the exemplar
      psg::launch_rescore_query_windows(ctx, q.p, nq, ix, id.p, dd.p);
    }
    id.download(ctx, idx, nq);
    dd.download(ctx, dist, nq);
    std::vector<double> h2;
    if (dist_pca) {
      h2.resize(nq);
      d2.download(ctx, h2.data(), nq);
    }
    if (scanned) sc.download(ctx, scanned, nq);
    psg::check_flags(ctx);
    if (dist_pca)
      for (int64_t i = 0; i < nq; ++i) dist_pca[i] = std::sqrt(h2[i]);
  });
}

psg_status psg_search_step(psg_ctx* ctx, const psg_index* index, const double* out_planes, int W,
                           int H, int spacing, int patch_width, psg_budget budget, int32_t* idx,
                           double* dist, int64_t* nn_calls, int64_t* scanned) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !index || !out_planes || !idx || !dist) fail(PSG_E_DOMAIN, "null argument");
    const psg::Index& ix = index->impl;
    if (ix.from_vectors) fail(PSG_E_SHAPE, "candidate dim does not match the grid window");
    psg::validate_grid(ix.w, spacing, W, H);
    psg::validate_budget(budget);
    if (patch_width < 1) fail(PSG_E_DOMAIN, "patch width must be >= 1");
    if (W < patch_width || H < patch_width) fail(PSG_E_DOMAIN, "output smaller than the patch");
    psg_opt_cfg cfg{};
    cfg.spacing = spacing;
    cfg.patch_width = patch_width;
    cfg.budget = budget;
    cfg.robust_exponent = 0.8;
    psg_level L;
    psg::level_setup(L, ctx, ix, W, H, cfg, true);
    psg::upload_state(L, out_planes);
    psg::level_prime(L);
    L.cur_idx.download(ctx, idx, L.A);
    L.cur_dist.download(ctx, dist, L.A);
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (nn_calls) *nn_calls = L.nn_calls;
    if (scanned) *scanned = L.pending_scanned;
  });
}

psg_status psg_update_step(psg_ctx* ctx, const psg_index* index, const int32_t* idx,
                           const double* irls, const double* pen, int W, int H, int spacing,
                           double* out_planes) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !index || !idx || !irls || !pen || !out_planes) fail(PSG_E_DOMAIN, "null argument");
    const psg::Index& ix = index->impl;
    if (ix.from_vectors) fail(PSG_E_SHAPE, "update_step needs an exemplar-window index");
    psg::validate_grid(ix.w, spacing, W, H);
    psg_opt_cfg cfg{};
    cfg.spacing = spacing;
    cfg.patch_width = 1;
    psg_level L;
    psg::level_setup(L, ctx, ix, W, H, cfg, false);
    for (int64_t a = 0; a < L.A; ++a)
      if (idx[a] < 0 || idx[a] >= ix.N) fail(PSG_E_SHAPE, "assignment index out of range");
    L.cur_idx.upload(ctx, idx, L.A);
    L.irls.upload(ctx, irls, L.A);
    L.pen.upload(ctx, pen, L.A);
    psg::launch_eff_from(ctx, L.irls.p, L.pen.p, L.A, L.eff.p, ctx->d_flags);
    psg::check_flags(ctx);
    psg::MstepArgs m = psg::mstep_args(L);
    m.mirror = nullptr;
    psg::launch_mstep(ctx, m);
    L.planes.download(ctx, out_planes, (size_t)L.P * L.C);
    psg::check_flags(ctx);
  });
}

psg_status psg_level_create(psg_ctx* ctx, const psg_index* index, const double* init, int W,
                            int H, const psg_opt_cfg* cfg, const double* ex_hist,
                            psg_level** out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !index || !init || !cfg || !out) fail(PSG_E_DOMAIN, "null argument");
    *out = nullptr;
    const psg::Index& ix = index->impl;
    if (ix.from_vectors) fail(PSG_E_SHAPE, "optimize_level needs an exemplar-window index");
    psg::validate_cfg(*cfg, ix.w, W, H);
    auto L = std::make_unique<psg_level>();
    // the image copy is issued first: from pinned host memory it is a DMA that
    // overlaps the host-side level setup (plan, covering ranges, lattices)
    psg::DBuf<double> staged((size_t)W * H * ix.C);
    staged.upload(ctx, init, (size_t)W * H * ix.C);
    psg::level_setup(*L, ctx, ix, W, H, *cfg, true);
    psg::level_set_hist(*L, ex_hist);
    psg::upload_state_dev(*L, staged.p);
    *out = L.release();
  });
}

psg_status psg_shard_plan(int W, int H, int w, int spacing, int rank, int world, psg_band* out) {
  return guarded([&] {
    if (!out) fail(PSG_E_DOMAIN, "null output");
    *out = psg::shard_plan(W, H, w, spacing, rank, world);
  });
}

psg_status psg_band_create(psg_ctx* ctx, const psg_index* index, const double* rows,
                           const psg_band* band, const psg_opt_cfg* cfg, const double* ex_hist,
                           psg_level** out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (!ctx || !index || !rows || !band || !cfg || !out) fail(PSG_E_DOMAIN, "null argument");
    *out = nullptr;
    const psg::Index& ix = index->impl;
    if (ix.from_vectors) fail(PSG_E_SHAPE, "optimize_level needs an exemplar-window index");
    psg::validate_cfg(*cfg, ix.w, band->W, band->H);
    const psg_band chk = psg::shard_plan(band->W, band->H, ix.w, cfg->spacing, band->rank,
                                         band->world);
    if (std::memcmp(&chk, band, sizeof(psg_band)) != 0) fail(PSG_E_SHAPE, "inconsistent band plan");
    auto L = std::make_unique<psg_level>();
    psg::level_setup_band(*L, ctx, ix, *band, *cfg, true);
    psg::level_set_hist(*L, ex_hist);
    psg::upload_state(*L, rows);
    *out = L.release();
  });
}

psg_status psg_band_phase1(psg_level* level, unsigned long long* counts_dev) {
  return guarded([&] {
    psg::StreamScope _ss(level->ctx->stream);
    psg::level_prime(*level);
    psg::phase_weights(*level);
    if (level->hist_on && counts_dev)
      PSG_CUDA(cudaMemcpyAsync(counts_dev, level->counts.p,
                               sizeof(unsigned long long) * level->counts.n,
                               cudaMemcpyDeviceToDevice, level->ctx->stream));
    // stream-ordered: the exchange that follows must be enqueued on (or
    // synchronised with) the context stream; device flags are checked in phase 4
  });
}

psg_status psg_band_phase2(psg_level* level, const unsigned long long* global_counts_dev,
                           int send_row0, void* send_dev) {
  return guarded([&] {
    psg_level& L = *level;
    psg::StreamScope _ss(L.ctx->stream);
    psg::phase_penalty(L, global_counts_dev ? global_counts_dev : L.counts.p);
    if (send_dev && send_row0 < L.band.a1) {
      if (send_row0 < L.band.a0) fail(PSG_E_DOMAIN, "send rows start below the owned rows");
      const int64_t first = (int64_t)(send_row0 - L.band.hlo) * L.nx;
      const int64_t n = (int64_t)(L.band.a1 - send_row0) * L.nx;
      char* dst = static_cast<char*>(send_dev);
      PSG_CUDA(cudaMemcpyAsync(dst, L.eff.p + first, sizeof(double) * n,
                               cudaMemcpyDeviceToDevice, L.ctx->stream));
      PSG_CUDA(cudaMemcpyAsync(dst + sizeof(double) * n, L.cur_idx.p + first, sizeof(int32_t) * n,
                               cudaMemcpyDeviceToDevice, L.ctx->stream));
    }
  });
}

psg_status psg_band_phase3(psg_level* level, const void* recv_dev, int n_send_rows,
                           float* send_rows_dev) {
  return guarded([&] {
    psg_level& L = *level;
    psg::StreamScope _ss(L.ctx->stream);
    if (L.nh > 0) {
      if (!recv_dev) fail(PSG_E_DOMAIN, "halo anchors required");
      const int64_t n = L.off;
      const char* src = static_cast<const char*>(recv_dev);
      PSG_CUDA(cudaMemcpyAsync(L.eff.p, src, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                               L.ctx->stream));
      PSG_CUDA(cudaMemcpyAsync(L.cur_idx.p, src + sizeof(double) * n, sizeof(int32_t) * n,
                               cudaMemcpyDeviceToDevice, L.ctx->stream));
    }
    psg::phase_update(L);
    if (n_send_rows > 0 && send_rows_dev) {
      if (n_send_rows > L.Hu) fail(PSG_E_DOMAIN, "more halo rows requested than owned");
      PSG_CUDA(cudaMemcpyAsync(send_rows_dev, L.mirror.p,
                               sizeof(float) * (size_t)n_send_rows * L.W * L.C,
                               cudaMemcpyDeviceToDevice, L.ctx->stream));
    }
  });
}

psg_status psg_band_phase4(psg_level* level, const float* recv_rows_dev, double* partials) {
  return guarded([&] {
    psg_level& L = *level;
    psg::StreamScope _ss(L.ctx->stream);
    if (L.Hl > L.Hu) {
      if (!recv_rows_dev) fail(PSG_E_DOMAIN, "halo rows required");
      PSG_CUDA(cudaMemcpyAsync(L.mirror.p + (size_t)L.Hu * L.W * L.C, recv_rows_dev,
                               sizeof(float) * (size_t)(L.Hl - L.Hu) * L.W * L.C,
                               cudaMemcpyDeviceToDevice, L.ctx->stream));
    }
    psg::phase_search(L);
    if (partials) psg::phase_partials(L, partials);
  });
}

psg_status psg_band_commit(psg_level* level, const double* global_partials, psg_iter_stats* st) {
  return guarded([&] {
    psg::StreamScope _ss(level->ctx->stream);
    double g[9];
    if (global_partials) {
      std::memcpy(g, global_partials, sizeof(g));
    } else {
      psg::phase_partials(*level, g);
    }
    psg::phase_commit(*level, g, st);
  });
}

psg_status psg_level_prime(psg_level* level) {
  return guarded([&] {
    psg::StreamScope _ss(level->ctx->stream);
    psg::level_prime(*level);
  });
}

psg_status psg_level_iterate(psg_level* level, int n, int honor_convergence,
                             psg_iter_stats* stats, int* n_done) {
  return guarded([&] {
    psg::StreamScope _ss(level->ctx->stream);
    psg::level_prime(*level);
    int done = 0;
    for (int i = 0; i < n; ++i) {
      const bool conv = psg::level_step(*level, stats ? stats + i : nullptr, honor_convergence != 0);
      ++done;
      if (conv) break;
    }
    if (n_done) *n_done = done;
  });
}

psg_status psg_level_download(psg_level* level, double* planes, int32_t* idx, double* dist) {
  return guarded([&] {
    psg::StreamScope _ss(level->ctx->stream);
    psg_ctx* ctx = level->ctx;
    if (planes) level->planes.download(ctx, planes, (size_t)level->P * level->C);
    if (idx) level->cur_idx.download(ctx, idx, level->A);
    if (dist) level->cur_dist.download(ctx, dist, level->A);
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

psg_status psg_level_state_dev(psg_level* level, void** planes_dev, void** idx_dev,
                               void** dist_dev) {
  return guarded([&] {
    psg::StreamScope _ss(level->ctx->stream);
    if (planes_dev) *planes_dev = level->planes.p;
    level->counts_fresh = false;  // the caller may write the planes
    if (idx_dev) *idx_dev = level->cur_idx.p;
    if (dist_dev) *dist_dev = level->cur_dist.p;
  });
}

psg_status psg_level_query_stats(psg_level* level, int64_t* scanned, int64_t* exact_evals,
                                 int32_t* nodes_visited) {
  return guarded([&] {
    psg::StreamScope _ss(level->ctx->stream);
    psg_ctx* ctx = level->ctx;
    if (scanned) level->scanned.download(ctx, scanned, level->A);
    if (exact_evals) level->exact_evals.download(ctx, exact_evals, level->A);
    if (nodes_visited) level->visited.download(ctx, nodes_visited, level->A);
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

void psg_level_destroy(psg_level* level) { delete level; }

psg_status psg_optimize_level(psg_ctx* ctx, const psg_index* index, const double* init, int W,
                              int H, const psg_opt_cfg* cfg, const double* ex_hist,
                              double* out_planes, psg_iter_stats* stats, int* n_iters) {
  psg_level* L = nullptr;
  psg_status s = psg_level_create(ctx, index, init, W, H, cfg, ex_hist, &L);
  if (s != PSG_OK) return s;
  std::unique_ptr<psg_level> hold(L);
  {  // a pinned (page-locked) result buffer can take the image early, asynchronously
    cudaPointerAttributes at{};
    if (out_planes && cudaPointerGetAttributes(&at, out_planes) == cudaSuccess &&
        at.type == cudaMemoryTypeHost && !ctx->knobs.graph && !ctx->knobs.no_early_download)
      L->early_host = out_planes;
    cudaGetLastError();  // (unregistered memory may leave an error state on old drivers)
  }
  int done = 0;
  s = psg_level_iterate(L, cfg->max_iterations, 1, stats, &done);
  if (s != PSG_OK) return s;
  if (n_iters) *n_iters = done;
  if (L->early_done)  // the final image is already on its way
    return guarded([&] {
      PSG_CUDA(cudaStreamSynchronize(ctx->copy));
      PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
  return psg_level_download(L, out_planes, nullptr, nullptr);
}

int psg_axis_positions(int extent, int window, int step, int* out) {
  if (window < 1 || step < 1 || extent < window) return 0;
  const auto v = psg::axis_positions(extent, window, step);
  if (out) std::copy(v.begin(), v.end(), out);
  return (int)v.size();
}

int64_t psg_plan(int W, int H, int w, int spacing, int patch_width, int32_t* mult) {
  if (w < 1 || spacing < 1 || patch_width < 1 || W < w || H < w || W < patch_width ||
      H < patch_width)
    return -1;
  return psg::plan_host(W, H, w, spacing, patch_width, mult);
}

double psg_pow_cr(double x, double y) { return psg::pow_cr_host(x, y); }

double psg_hist_mass(int64_t count, int64_t pixels) {
  return psg::hist_mass(count, 1.0 / (double)pixels);
}

}  // extern "C"

// ===========================================================================
// Pyramid driver: synthesize (pipeline.cpp:216-315), stage schedule
// (level x neighbourhood size) per the BASELINE configs.
// ===========================================================================

namespace psg {
namespace {

// The stages' indexes built AHEAD of the EM loop: an index depends only on
// the exemplar level and the stage's configuration, never on the output, so
// the next stages' PCA fits / projections / tree builds (many small kernels
// and host synchronisations, or the host replica of KmTree::build) run in up
// to three worker threads, each on its own context (own stream, own cuBLAS /
// cuSOLVER handles), while the current stage's EM iterations saturate the GPU
// from the caller's stream.  Results do not depend on the overlap; PERSYN_NO_BUILD_AHEAD
// builds each index inline on the caller's context.
class IndexAhead {
 public:
  using Build = std::function<std::unique_ptr<psg_index>(psg_ctx*)>;
  static constexpr int kWorkers = 3;  // stages in flight ahead of the EM loop
  IndexAhead(psg_ctx* main, std::vector<Build> jobs) : main_(main), jobs_(std::move(jobs)) {
    done_.resize(jobs_.size());
    if (main_->knobs.no_build_ahead || jobs_.size() < 2) return;
    const int nw = (int)std::min<size_t>(kWorkers, jobs_.size());
    while ((int)main_->builders.size() < nw) {
      psg_ctx* b = nullptr;
      if (psg_ctx_create(main_->device, nullptr, &b) != PSG_OK)
        fail(PSG_E_CUDA, "cannot create an index builder context: " + g_last_error);
      main_->builders.push_back(b);
    }
    for (int i = 0; i < nw; ++i) workers_.emplace_back([this, i, nw] { run(i, nw); });
  }
  ~IndexAhead() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // index of stage k (stages are taken in order); ms = its build time
  std::unique_ptr<psg_index> take(size_t k, double* ms) {
    if (workers_.empty()) {
      const double t = now_ms();
      auto ix = jobs_[k](main_);
      *ms = now_ms() - t;
      return ix;
    }
    std::unique_lock<std::mutex> lk(m_);
    taken_ = k + 1;
    cv_.notify_all();
    cv_.wait(lk, [&] { return done_[k].ready; });
    if (done_[k].err) std::rethrow_exception(done_[k].err);
    *ms = done_[k].ms;
    // the builder's stream is idle for this index: from here on it belongs to
    // the caller's context, whose stream orders its (stream-ordered) frees
    // after every kernel that reads it -- also when an exception unwinds
    done_[k].index->impl.ctx = main_;
    return std::move(done_[k].index);
  }

 private:
  struct Slot {
    std::unique_ptr<psg_index> index;
    double ms = 0.0;
    std::exception_ptr err;
    bool ready = false;
  };
  // worker i builds stages i, i + nw, ... on its own context, never more than
  // nw stages ahead of the stage the EM loop has taken
  void run(int i, int nw) {
    cudaSetDevice(main_->device);
    psg_ctx* b = main_->builders[(size_t)i];
    StreamScope ss(b->stream);
    for (size_t k = (size_t)i; k < jobs_.size(); k += (size_t)nw) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || k < taken_ + (size_t)nw; });
        if (stop_) return;
      }
      Slot s;
      const double t = now_ms();
      try {
        s.index = jobs_[k](b);
        cudaStreamSynchronize(b->stream);  // ready for the caller's stream
      } catch (...) {
        s.err = std::current_exception();
      }
      s.ms = now_ms() - t;
      s.ready = true;
      const bool failed = (bool)s.err;
      {
        std::lock_guard<std::mutex> lk(m_);
        done_[k] = std::move(s);
      }
      cv_.notify_all();
      if (failed) return;
    }
  }
  psg_ctx* main_;
  std::vector<Build> jobs_;
  std::vector<Slot> done_;
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_;
  size_t taken_ = 0;
  bool stop_ = false;
};

}  // namespace
}  // namespace psg

extern "C" psg_status psg_synthesize(psg_ctx* ctx, const psg_request* req, double* out_planes,
                                     psg_report* report) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    using namespace psg;
    if (!ctx || !req || !out_planes) fail(PSG_E_DOMAIN, "null argument");
    const int C = req->C, G = C - 3;
    if (C < 4 || C > 8) fail(PSG_E_SHAPE, "channels must be 3 + G with G in [1, 5]");
    if (req->levels < 1) fail(PSG_E_DOMAIN, "levels must be >= 1");
    if (req->out_w < 1 || req->out_h < 1) fail(PSG_E_DOMAIN, "empty output size");
    if (req->stages.n_sizes < 1 || req->stages.n_sizes > 4)
      fail(PSG_E_DOMAIN, "1..4 neighbourhood sizes per level");
    if (req->guidance_kind != 0 && !req->out_guidance)
      fail(PSG_E_DOMAIN, "explicit guidance requires out_guidance planes");
    const double t0 = now_ms();
    psg_report rep{};
    const int L = req->levels;
    const int EW = req->ew, EH = req->eh;
    const size_t EP = (size_t)EW * EH;
    DBuf<double> ex_full((size_t)C * EP);
    ex_full.upload(ctx, req->exemplar, ex_full.n);
    DBuf<double> out_guid;
    if (req->guidance_kind != 0) {
      out_guid.alloc((size_t)G * req->out_w * req->out_h);
      out_guid.upload(ctx, req->out_guidance, out_guid.n);
    }
    // Per-level exemplar and output guidance (device).
    std::vector<DBuf<double>> ex_lv(L), og_lv(L);
    std::vector<int> ew(L), eh(L), ow(L), oh(L);
    for (int l = 0; l < L; ++l) {
      const int shift = L - 1 - l;
      const int f = 1 << shift;
      ow[l] = req->out_w >> shift;
      oh[l] = req->out_h >> shift;
      ew[l] = EW / f;
      eh[l] = EH / f;
      if (ow[l] < 1 || oh[l] < 1 || ew[l] < 1 || eh[l] < 1)
        fail(PSG_E_DOMAIN, "level " + std::to_string(l) + " has no pixels");
      const size_t lp = (size_t)ew[l] * eh[l];
      ex_lv[l].alloc((size_t)C * lp);
      for (int c = 0; c < 3; ++c) {
        if (f == 1)
          PSG_CUDA(cudaMemcpyAsync(ex_lv[l].p + c * lp, ex_full.p + c * EP, sizeof(double) * lp,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
        else
          launch_downsample(ctx, ex_full.p + c * EP, EW, EH, f, ex_lv[l].p + c * lp);
      }
      const size_t op = (size_t)ow[l] * oh[l];
      og_lv[l].alloc((size_t)G * op);
      if (req->guidance_kind == 0) {  // ramps generated on the device
        launch_ramp_planes(ctx, G, ew[l], eh[l], ex_lv[l].p + 3 * lp);
        launch_ramp_planes(ctx, G, ow[l], oh[l], og_lv[l].p);
      } else {
        for (int g = 0; g < G; ++g) {
          if (f == 1) {
            PSG_CUDA(cudaMemcpyAsync(ex_lv[l].p + (3 + g) * lp, ex_full.p + (3 + g) * EP,
                                     sizeof(double) * lp, cudaMemcpyDeviceToDevice, ctx->stream));
            PSG_CUDA(cudaMemcpyAsync(og_lv[l].p + g * op,
                                     out_guid.p + (size_t)g * req->out_w * req->out_h,
                                     sizeof(double) * op, cudaMemcpyDeviceToDevice, ctx->stream));
          } else {
            launch_downsample(ctx, ex_full.p + (3 + g) * EP, EW, EH, f, ex_lv[l].p + (3 + g) * lp);
            launch_downsample(ctx, out_guid.p + (size_t)g * req->out_w * req->out_h, req->out_w,
                              req->out_h, f, og_lv[l].p + g * op);
          }
        }
      }
    }
    // Part 1 at the coarsest level: initialize_output (pipeline.cpp:96-175)
    // with the first guidance plane (row ramp) as the normalised scale map,
    // bounds [0, 1]: the exemplar's S plane is its scale, the output's ramp
    // (fp32 values) its target; further guidance planes are copied.
    std::vector<double> hex((size_t)C * ew[0] * eh[0]), hog((size_t)G * ow[0] * oh[0]);
    ex_lv[0].download(ctx, hex.data(), hex.size());
    og_lv[0].download(ctx, hog.data(), hog.size());
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    // the stages in schedule order and their index builds (IndexAhead: one
    // stage ahead of the EM loop; the exemplar levels are complete here)
    struct StageJob {
      int l, si, w;
    };
    std::vector<StageJob> stage_jobs;
    std::vector<IndexAhead::Build> builds;
    for (int l = 0; l < L; ++l)
      for (int si = 0; si < req->stages.n_sizes; ++si) {
        const int w = req->stages.sizes[si];
        if (w < 2 || w % 2) fail(PSG_E_DOMAIN, "neighbourhood sizes must be even and >= 2");
        if (ow[l] < w || oh[l] < w || ew[l] < w || eh[l] < w) continue;
        if ((int64_t)(ew[l] - w + 1) * (eh[l] - w + 1) < 2) continue;  // fit_pca needs n >= 2
        psg_index_cfg icfg = req->index;
        // level_seed (pipeline.cpp:54-56); several sizes per level (the
        // BASELINE configs' stages) also mix in the window width
        icfg.seed = (req->seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(l + 1))) ^
                    (req->stages.n_sizes > 1 ? (uint64_t)w : 0ull);
        if (req->cfg.histogram_matching) {
          icfg.hist_bins = req->cfg.histogram_bins;
          icfg.hist_include_scale = req->cfg.histogram_include_scale;
        }
        const int s_id = l * req->stages.n_sizes + si;
        const double* s_mean = req->stage_mean ? req->stage_mean[s_id] : nullptr;
        const double* s_basis = req->stage_basis ? req->stage_basis[s_id] : nullptr;
        const int s_d = (s_basis && req->stage_d) ? req->stage_d[s_id] : 0;
        if ((s_mean == nullptr) != (s_basis == nullptr))
          fail(PSG_E_DOMAIN, "stage PCA injection needs both mean and basis");
        const double* exl = ex_lv[l].p;
        const int ewl = ew[l], ehl = eh[l];
        const bool brute = req->index_kind == PSG_INDEX_BRUTE_FORCE;
        stage_jobs.push_back({l, si, w});
        builds.push_back([=](psg_ctx* bctx) {
          return brute ? create_brute_from_device_planes(bctx, exl, C, ewl, ehl, w, icfg.hist_bins,
                                                         icfg.hist_include_scale)
                       : create_index_from_device_planes(bctx, exl, C, ewl, ehl, w, s_mean,
                                                         s_basis, s_d, icfg);
        });
      }
    IndexAhead ahead(ctx, std::move(builds));
    size_t stage_no = 0;
    const size_t op0 = (size_t)ow[0] * oh[0];
    std::vector<double> init((size_t)C * op0);
    {
      std::vector<float> target(op0);
      for (size_t i = 0; i < op0; ++i) target[i] = (float)hog[i];
      initialize_output_host(hex.data(), C, ew[0], eh[0], target.data(), ow[0], oh[0], 0.0, 1.0,
                             req->seed, init.data());
      for (int g = 1; g < G; ++g)
        std::copy(hog.begin() + g * op0, hog.begin() + (g + 1) * op0, init.begin() + (3 + g) * op0);
    }
    DBuf<double> state((size_t)C * op0);
    state.upload(ctx, init.data(), init.size());
    rep.part1_millis = now_ms() - t0;

    const double t1 = now_ms();
    int n_trace = 0;  // iterations recorded into req->trace
    // the previous stage's final assignment seeds each stage's first search
    struct Carry {
      DBuf<int32_t> idx, xs, ys;
      int nx = 0, ny = 0, nh = 0, w = 0, nxe = 0, level = -1;
      int64_t off = 0;
    } carry;
    for (int l = 0; l < L; ++l) {
      const int W = ow[l], H = oh[l];
      const size_t op = (size_t)W * H;
      if (l > 0) {
        const int pw = ow[l - 1], ph = oh[l - 1];
        DBuf<double> next((size_t)C * op), up((size_t)(2 * pw) * (2 * ph));
        for (int c = 0; c < 3; ++c) {
          launch_upsample_bilinear(ctx, state.p + (size_t)c * pw * ph, pw, ph, 2, up.p);
          launch_fit_to(ctx, up.p, 2 * pw, 2 * ph, W, H, next.p + c * op);
        }
        PSG_CUDA(cudaMemcpyAsync(next.p + 3 * op, og_lv[l].p, sizeof(double) * G * op,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        state = std::move(next);
      }
      for (int si = 0; si < req->stages.n_sizes; ++si) {
        const int w = req->stages.sizes[si];
        if (w < 2 || w % 2) fail(PSG_E_DOMAIN, "neighbourhood sizes must be even and >= 2");
        if (W < w || H < w || ew[l] < w || eh[l] < w) continue;
        if ((int64_t)(ew[l] - w + 1) * (eh[l] - w + 1) < 2) continue;  // fit_pca needs n >= 2
        const double ti = now_ms();
        {  // stage scope: index and level are released before the next stage
        if (stage_no >= stage_jobs.size() || stage_jobs[stage_no].l != l ||
            stage_jobs[stage_no].si != si)
          fail(PSG_E_LOGIC, "stage schedule mismatch");
        double index_ms = 0.0;
        auto index = ahead.take(stage_no++, &index_ms);
        psg_opt_cfg cfg = req->cfg;
        cfg.spacing = std::max(1, w / 4);
        cfg.patch_width = std::min(std::max(1, cfg.patch_width), cfg.spacing);
        validate_cfg(cfg, w, W, H);
        const double to = now_ms();
        psg_level lv;
        level_setup(lv, ctx, index->impl, W, H, cfg, true);
        level_set_hist(lv, nullptr);
        PSG_CUDA(cudaMemcpyAsync(lv.planes.p, state.p, sizeof(double) * C * op,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        launch_make_mirror(ctx, lv.planes.p, C, W, H, lv.mirror.p);
        DBuf<int32_t> seeds;
        if (carry.level >= 0 && !ctx->knobs.no_carry) {
          const AnchorSet as = owned_anchors(lv);
          seeds.alloc((size_t)as.count);
          CarryArgs ca{};
          ca.xs = as.xs;
          ca.ys = as.ys;
          ca.nx = as.nx;
          ca.nq = as.count;
          ca.w = w;
          ca.nxe = index->impl.nxe;
          ca.nye = index->impl.eh - w + 1;
          ca.pidx = carry.idx.p + carry.off;
          ca.pxs = carry.xs.p;
          ca.pys = carry.ys.p + carry.nh;
          ca.pnx = carry.nx;
          ca.pny = carry.ny;
          ca.pw = carry.w;
          ca.pnxe = carry.nxe;
          ca.scale = 1 << (l - carry.level);
          ca.out = seeds.p;
          launch_carry_seed(ctx, ca);
        }
        level_prime(lv, seeds.p);
        if (ctx->knobs.verbose)
          fprintf(stderr, "[persyn] stage l=%d w=%d: first search %.2f ms (%s)\n", l, w,
                  lv.pending_ms, seeds.p ? "carried seed" : "unseeded");
        psg_iter_stats last{};
        int iters = 0;
        int64_t calls = 0;
        const bool verbose = ctx->knobs.verbose;
        std::string its;
        const int trace_first = n_trace;
        for (int it = 0; it < cfg.max_iterations; ++it) {
          const bool conv = level_step(lv, &last, true);
          if (req->trace && n_trace < req->trace_cap) req->trace[n_trace] = last;
          ++n_trace;
          calls += last.nn_calls;
          ++iters;
          if (verbose) its += " " + std::to_string(last.millis).substr(0, 5);
          if (conv) break;
        }
        if (verbose) fprintf(stderr, "[persyn] stage l=%d w=%d: iteration ms%s\n", l, w, its.c_str());
        PSG_CUDA(cudaMemcpyAsync(state.p, lv.planes.p, sizeof(double) * C * op,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        std::swap(carry.idx, lv.cur_idx);  // the level frees the swapped-in buffers
        std::swap(carry.xs, lv.xs);
        std::swap(carry.ys, lv.ys);
        carry.nx = lv.nx;
        carry.ny = (int)(lv.Ao / lv.nx);
        carry.nh = lv.nh;
        carry.off = lv.off;
        carry.w = w;
        carry.nxe = index->impl.nxe;
        carry.level = l;
        PSG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (rep.n_stages < 16) {
          psg_stage_report& sr = rep.stages[rep.n_stages++];
          sr.level = l;
          sr.w = w;
          sr.W = W;
          sr.H = H;
          sr.ew = ew[l];
          sr.eh = eh[l];
          sr.d = index->impl.d;
          sr.iterations = iters;
          sr.final_energy = last.energy;
          sr.nn_calls = calls;
          sr.index_millis = index_ms;
          sr.optimize_millis = now_ms() - to;
          sr.trace_first = trace_first;
          sr.trace_count = n_trace - trace_first;
        }
        rep.total_nn_calls += calls;
        rep.final_energy = last.energy;
        if (ctx->knobs.verbose)
          fprintf(stderr, "[persyn] stage l=%d w=%d: index %.2f ms, optimize %.2f ms\n", l, w,
                  index_ms, now_ms() - to);
        }
        if (ctx->knobs.verbose) {
          cudaMemPool_t pool;
          uint64_t cur = 0, high = 0;
          PSG_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
          PSG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &cur));
          PSG_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high));
          fprintf(stderr, "[persyn] stage l=%d w=%d: wall incl. teardown %.2f ms (pool reserved "
                  "%.0f MB, used high %.0f MB)\n", l, w, now_ms() - ti, cur / 1e6, high / 1e6);
        }
      }
    }
    rep.part2_millis = now_ms() - t1;
    rep.n_trace = n_trace;
    if (ctx->knobs.verbose)
      fprintf(stderr, "[persyn] synthesize: part1 %.2f ms, part2 %.2f ms\n", rep.part1_millis,
              rep.part2_millis);
    state.download(ctx, out_planes, (size_t)C * req->out_w * req->out_h);
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (report) *report = rep;
  });
}

// ---------------------------------------------------------------------------
// Part 1 and the resampling between levels, as standalone entry points.
extern "C" psg_status psg_initialize_output(const double* ex_planes, int C, int ew, int eh,
                                            const float* out_scale, int ow, int oh,
                                            double s_min, double s_max, uint64_t seed,
                                            double* out4) {
  return guarded([&] {
    if (!ex_planes || !out_scale || !out4) fail(PSG_E_DOMAIN, "null argument");
    psg::initialize_output_host(ex_planes, C, ew, eh, out_scale, ow, oh, s_min, s_max, seed,
                                out4);
  });
}

namespace {
// in [C][H][W] (host) -> device, f(plane_in, plane_out) per plane, -> out (host)
template <class F>
void resample_planes(psg_ctx* ctx, const double* in, int C, int W, int H, int ow, int oh,
                     double* out, F&& f) {
  using namespace psg;
  if (!ctx || !in || !out) fail(PSG_E_DOMAIN, "null argument");
  if (C < 1 || W < 1 || H < 1) fail(PSG_E_DOMAIN, "empty image");
  const size_t ip = (size_t)W * H, op = (size_t)ow * oh;
  DBuf<double> din((size_t)C * ip), dout((size_t)C * op);
  din.upload(ctx, in, din.n);
  for (int c = 0; c < C; ++c) f(din.p + c * ip, dout.p + c * op);
  dout.download(ctx, out, dout.n);
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
}
}  // namespace

extern "C" psg_status psg_downsample(psg_ctx* ctx, const double* in, int C, int W, int H,
                                     int factor, double* out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (factor < 1) fail(PSG_E_DOMAIN, "downsample factor must be >= 1");
    const int ow = W / factor, oh = H / factor;
    if (ow < 1 || oh < 1) fail(PSG_E_DOMAIN, "downsample leaves no pixels");
    resample_planes(ctx, in, C, W, H, ow, oh, out, [&](const double* a, double* b) {
      psg::launch_downsample(ctx, a, W, H, factor, b);
    });
  });
}

extern "C" psg_status psg_upsample_bilinear(psg_ctx* ctx, const double* in, int C, int W, int H,
                                            int factor, double* out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (factor < 1) fail(PSG_E_DOMAIN, "upsample factor must be >= 1");
    if ((int64_t)W * factor * (int64_t)H * factor > (int64_t{1} << 30))
      fail(PSG_E_DOMAIN, "upsampled image would be unreasonably large");
    resample_planes(ctx, in, C, W, H, W * factor, H * factor, out,
                    [&](const double* a, double* b) {
                      if (factor == 1)
                        PSG_CUDA(cudaMemcpyAsync(b, a, sizeof(double) * W * H,
                                                 cudaMemcpyDeviceToDevice, ctx->stream));
                      else
                        psg::launch_upsample_bilinear(ctx, a, W, H, factor, b);
                    });
  });
}

extern "C" psg_status psg_fit_to(psg_ctx* ctx, const double* in, int C, int W, int H, int ow,
                                 int oh, double* out) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    if (ow < 1 || oh < 1) fail(PSG_E_DOMAIN, "image dimensions must be at least 1x1");
    resample_planes(ctx, in, C, W, H, ow, oh, out, [&](const double* a, double* b) {
      psg::launch_fit_to(ctx, a, W, H, ow, oh, b);
    });
  });
}

extern "C" psg_status psg_debug_projection(psg_ctx* ctx, const psg_index* index,
                                           const double* planes, int W, int H, int spacing,
                                           double* q_tc, float* delta, double* q_exact) {
  return guarded([&] {
    psg::StreamScope _ss(ctx ? ctx->stream : nullptr);
    using namespace psg;
    if (!ctx || !index || !planes) fail(PSG_E_DOMAIN, "null argument");
    const Index& ix = index->impl;
    if (!ix.tc) fail(PSG_E_DOMAIN, "index has no tensor-core projection operand");
    validate_grid(ix.w, spacing, W, H);
    const auto hx = axis_positions(W, ix.w, spacing), hy = axis_positions(H, ix.w, spacing);
    const int64_t A = (int64_t)hx.size() * hy.size(), P = (int64_t)W * H;
    DBuf<int32_t> xs(hx.size()), ys(hy.size());
    xs.upload(ctx, hx.data(), hx.size());
    ys.upload(ctx, hy.data(), hy.size());
    DBuf<double> pl((size_t)ix.C * P), qt((size_t)A * ix.d), qe((size_t)A * ix.d);
    DBuf<float> mir((size_t)P * ix.C), dl((size_t)A);
    DBuf<uint8_t> q8((size_t)4 * P * 8);
    DBuf<int> bad(1);
    pl.upload(ctx, planes, pl.n);
    launch_make_mirror(ctx, pl.p, ix.C, W, H, mir.p);
    PSG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
    launch_make_digits(ctx, mir.p, ix.C, W, H, q8.p, P * 8, bad.p);
    const AnchorSet as{xs.p, ys.p, (int)hx.size(), A};
    bool stride2 = hx[0] % 2 == 0;
    for (size_t i = 1; i < hx.size(); ++i) stride2 = stride2 && hx[i] - hx[i - 1] == 2;
    launch_project_windows_tc(ctx, q8.p, P * 8, W, bad.p, as, stride2, ix, qt.p, dl.p, spacing);
    launch_project_windows(ctx, mir.p, W, ix.C, ix.w, as, ix.mean, ix.basis, ix.d, qe.p);
    if (q_tc) qt.download(ctx, q_tc, qt.n);
    if (delta) dl.download(ctx, delta, dl.n);
    if (q_exact) qe.download(ctx, q_exact, qe.n);
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    check_flags(ctx);
  });
}

// ---------------------------------------------------------------------------
// Row-band helpers for shard.cpp.
namespace psg {
void band_info(const psg_level* L, psg_band* plan, psg_opt_cfg* cfg, int* C, int* hist_on,
               int* iterations_done) {
  if (plan) *plan = L->band;
  if (cfg) *cfg = L->cfg;
  if (C) *C = L->C;
  if (hist_on) *hist_on = L->hist_on ? 1 : 0;
  if (iterations_done) *iterations_done = L->iter;
}

psg_status band_download_owned(psg_level* L, double* rows) {
  return guarded([&] {
    StreamScope _ss(L->ctx->stream);
    const size_t own = (size_t)L->Hu * L->W;
    for (int c = 0; c < L->C; ++c)
      PSG_CUDA(cudaMemcpyAsync(rows + c * own, L->planes.p + (size_t)c * L->P, sizeof(double) * own,
                               cudaMemcpyDeviceToHost, L->ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(L->ctx->stream));
  });
}

int index_window(const psg_index* ix) { return ix->impl.w; }
int index_channels(const psg_index* ix) { return ix->impl.C; }
}  // namespace psg
