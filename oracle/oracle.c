/*
 * TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * Plain-C restatement of the reference's EM hot path (persyn,
 * /root/reference/proj/core/src), generalised from the reference's
 * hard-coded C = 4 channels (image.hpp:70) to C = 3 + G guidance planes so
 * it can check the C = 5 configuration the reference itself cannot run.
 * At C = 4 it is pinned bit-for-bit against the reference's own TUs
 * (oracle/_ref/libpersyn_ref.so, see tests/test_oracle_pins.py) and against
 * the committed golden vectors in tests/golden/.
 *
 * Arithmetic contract: fp64, index-ascending loops,
 * separate multiply and add (compiled with -ffp-contract=off), fp32 features
 * = (float) of fp64 planes.  Exact nearest neighbour = lexicographic minimum
 * of (fp64 dist^2 in PCA space, index), which is what KmTree::query(exact)
 * returns (km_tree.cpp:251-278, pinned by ann_test.cpp:225-245).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 *
 * Image layout everywhere: planes [C][H][W] fp64, row-major, row 0 = bottom
 * (image.hpp:11-12,57-59).  Feature layout: pixel-major (dy, dx), channel
 * minor (neighborhood.cpp:128-135).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define OR_OK 0
#define OR_E_DOMAIN 1
#define OR_E_SHAPE 2
#define OR_E_LOGIC 3

int oracle_version(void) { return 1; }

/* ---- L1 geometry ------------------------------------------------------- */

/* neighborhood.cpp:12-18 — multiples of step that fit, plus extent-window. */
int or_axis_positions(int extent, int window, int step, int *out) {
  int n = 0;
  for (int p = 0; p + window <= extent; p += step) {
    if (out) out[n] = p;
    n++;
  }
  const int last = extent - window;
  int back = -1;
  if (n > 0) back = out ? out[n - 1] : ((extent - window) / step) * step;
  if (n == 0 || back != last) {
    if (out) out[n] = last;
    n++;
  }
  return n;
}

/* neighborhood.cpp:22-35 */
int or_grid_validate(int w, int sp, int W, int H) {
  if (w < 2 || (w % 2) != 0 || sp < 1 || sp > w) return OR_E_DOMAIN;
  if (W < w || H < w) return OR_E_DOMAIN;
  return OR_OK;
}

/* Number of entries a in [lo, hi] of the sorted array xs. */
static int count_in(const int *xs, int n, int lo, int hi) {
  int c = 0;
  for (int i = 0; i < n; ++i)
    if (xs[i] >= lo && xs[i] <= hi) c++;
  return c;
}

/*
 * Plan of search_step (optimizer.cpp:288-296): every p x p tile queries each
 * anchor whose window contains it (neighborhood.cpp:56-85).  The plan is
 * separable: mult(a) = mx(ax) * my(ay), nn_calls = Cx * Cy.  Writes the
 * per-anchor multiplicity (A = nx * ny entries, row-major) when mult != NULL
 * and returns nn_calls, or -1 when an anchor is uncovered
 * (optimizer.cpp:342-346, std::logic_error).
 */
int64_t or_plan(int W, int H, int w, int sp, int p, int32_t *mult) {
  int *xs = malloc(sizeof(int) * (W + 2)), *ys = malloc(sizeof(int) * (H + 2));
  int *tx = malloc(sizeof(int) * (W + 2)), *ty = malloc(sizeof(int) * (H + 2));
  const int nx = or_axis_positions(W, w, sp, xs), ny = or_axis_positions(H, w, sp, ys);
  const int ntx = or_axis_positions(W, p, p, tx), nty = or_axis_positions(H, p, p, ty);
  int64_t cx = 0, cy = 0, uncovered = 0;
  for (int t = 0; t < ntx; ++t) cx += count_in(xs, nx, tx[t] + p - w, tx[t]);
  for (int t = 0; t < nty; ++t) cy += count_in(ys, ny, ty[t] + p - w, ty[t]);
  int32_t *mx = malloc(sizeof(int32_t) * nx), *my = malloc(sizeof(int32_t) * ny);
  for (int i = 0; i < nx; ++i) mx[i] = count_in(tx, ntx, xs[i], xs[i] + w - p);
  for (int i = 0; i < ny; ++i) my[i] = count_in(ty, nty, ys[i], ys[i] + w - p);
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix) {
      const int32_t m = mx[ix] * my[iy];
      if (mult) mult[(int64_t)iy * nx + ix] = m;
      if (m == 0) uncovered++;
    }
  free(xs); free(ys); free(tx); free(ty); free(mx); free(my);
  return uncovered ? -1 : cx * cy;
}

/* neighborhood.cpp:120-137, generalised to C channels. */
void or_extract_window(const double *planes, int C, int W, int H, int ax, int ay, int w,
                       float *out) {
  const size_t P = (size_t)W * H;
  size_t o = 0;
  for (int dy = 0; dy < w; ++dy) {
    size_t row = (size_t)(ay + dy) * W + ax;
    for (int dx = 0; dx < w; ++dx, ++row)
      for (int c = 0; c < C; ++c) out[o++] = (float)planes[c * P + row];
  }
}

/* neighborhood.cpp:103-118 (rows in ascending row-major anchor order). */
int64_t or_extract_all(const double *planes, int C, int W, int H, int w, int sp, float *out) {
  int *xs = malloc(sizeof(int) * (W + 2)), *ys = malloc(sizeof(int) * (H + 2));
  const int nx = or_axis_positions(W, w, sp, xs), ny = or_axis_positions(H, w, sp, ys);
  const size_t D = (size_t)w * w * C;
  int64_t i = 0;
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix, ++i)
      if (out) or_extract_window(planes, C, W, H, xs[ix], ys[iy], w, out + i * D);
  free(xs); free(ys);
  return i;
}

/* ---- L2 index math ------------------------------------------------------ */

/* pca.cpp:27-41 — acc += (double(v[j]) - mean[j]) * basis[k][j], j ascending. */
void or_project(const float *v, int64_t D, const double *mean, const double *basis, int d,
                double *out) {
  for (int k = 0; k < d; ++k) {
    const double *row = basis + (size_t)k * D;
    double acc = 0.0;
    for (int64_t j = 0; j < D; ++j) {
      const double c = (double)v[j] - mean[j];
      const double p = c * row[j];
      acc = acc + p;
    }
    out[k] = acc;
  }
}

/* km_tree.cpp:15-22 */
double or_dist2(const double *a, const double *b, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = a[j] - b[j];
    const double s = t * t;
    acc = acc + s;
  }
  return acc;
}

/* Exact NN: lexicographic min of (dist^2, id) — scan_leaf's rule
 * (km_tree.cpp:128-139) over all points, = KmTree exact = brute_force_nearest. */
int32_t or_nearest_lexmin(const double *pts, int64_t n, int d, const double *q,
                          double *best_d2_out) {
  double best = INFINITY;
  int32_t best_id = -1;
  for (int64_t i = 0; i < n; ++i) {
    const double dd = or_dist2(pts + (size_t)i * d, q, d);
    if (dd < best || (dd == best && i < best_id)) {
      best = dd;
      best_id = (int32_t)i;
    }
  }
  if (best_d2_out) *best_d2_out = best;
  return best_id;
}

/* optimizer.cpp:117-124 */
double or_full_distance(const float *a, const float *b, int64_t D) {
  double acc = 0.0;
  for (int64_t j = 0; j < D; ++j) {
    const double t = (double)a[j] - (double)b[j];
    const double s = t * t;
    acc = acc + s;
  }
  return sqrt(acc);
}

/* pca.cpp:103-113 */
void or_project_all(const float *X, int64_t n, int64_t D, const double *mean,
                    const double *basis, int d, double *out) {
  for (int64_t i = 0; i < n; ++i) or_project(X + (size_t)i * D, D, mean, basis, d, out + (size_t)i * d);
}

/* ---- thread helper ------------------------------------------------------ */

typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; } range_job;

static void *range_trampoline(void *p) {
  range_job *j = (range_job *)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

static void parallel_for(int64_t n, int threads, range_fn fn, void *ctx) {
  if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads == 1 || n < 64) {
    fn(ctx, 0, n);
    return;
  }
  pthread_t th[256];
  range_job jobs[256];
  const int64_t chunk = (n + threads - 1) / threads;
  int used = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
    if (lo >= hi) break;
    jobs[t] = (range_job){fn, ctx, lo, hi};
    pthread_create(&th[t], NULL, range_trampoline, &jobs[t]);
    used++;
  }
  for (int t = 0; t < used; ++t) pthread_join(th[t], NULL);
}

/* ---- L4 search step ------------------------------------------------------ */

typedef struct {
  const double *planes; int C, W, H, w, nx;
  const int *xs, *ys;
  const float *cand; const double *mean, *basis, *proj; int64_t N; int d;
  int32_t *idx; double *dist; const int32_t *only; /* optional anchor subset */
} search_ctx;

static void search_range(void *p, int64_t lo, int64_t hi) {
  search_ctx *s = (search_ctx *)p;
  const int64_t D = (int64_t)s->w * s->w * s->C;
  float *v = malloc(sizeof(float) * D);
  double *q = malloc(sizeof(double) * (s->d > 0 ? s->d : 1));
  for (int64_t i = lo; i < hi; ++i) {
    const int64_t a = s->only ? s->only[i] : i;
    or_extract_window(s->planes, s->C, s->W, s->H, s->xs[a % s->nx], s->ys[a / s->nx], s->w, v);
    or_project(v, D, s->mean, s->basis, s->d, q);
    const int32_t id = or_nearest_lexmin(s->proj, s->N, s->d, q, NULL);
    s->idx[i] = id;
    s->dist[i] = or_full_distance(v, s->cand + (size_t)id * D, D);  /* optimizer.cpp:234 */
  }
  free(v); free(q);
}

/*
 * search_step (optimizer.cpp:275-348) in exact mode.  Every plan entry of
 * one anchor computes the same query on the same image, so each anchor is
 * queried once (result identical to the reference's last-writer scatter).
 * `only`/n_only restrict the evaluation to a subset of anchors (sampled
 * parity at full size); then idx/dist have n_only entries.
 */
int or_search_step(const double *planes, int C, int W, int H, int w, int sp, int p,
                   const float *cand, const double *proj, int64_t N, const double *mean,
                   const double *basis, int d, const int32_t *only, int64_t n_only,
                   int threads, int32_t *idx, double *dist, int64_t *nn_calls) {
  if (or_grid_validate(w, sp, W, H)) return OR_E_DOMAIN;
  int *xs = malloc(sizeof(int) * (W + 2)), *ys = malloc(sizeof(int) * (H + 2));
  const int nx = or_axis_positions(W, w, sp, xs), ny = or_axis_positions(H, w, sp, ys);
  const int64_t calls = or_plan(W, H, w, sp, p, NULL);
  if (nn_calls) *nn_calls = calls;
  if (calls < 0) { free(xs); free(ys); return OR_E_LOGIC; }
  search_ctx s = {planes, C, W, H, w, nx, xs, ys, cand, mean, basis, proj, N, d, idx, dist, only};
  parallel_for(only ? n_only : (int64_t)nx * ny, threads, search_range, &s);
  free(xs); free(ys);
  return OR_OK;
}

/* ---- weights, histograms, energy (optimizer.cpp:44-131) ----------------- */

/* optimizer.cpp:112-115 */
double or_irls_weight(double d, double r, double eps) {
  const double d2 = d * d;
  return pow(d2 + eps, (r - 2.0) / 2.0);
}

/* optimizer.cpp:126-131 */
double or_energy(const double *d, int64_t n, double r) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc = acc + pow(d[i], r);
  return acc;
}

/* optimizer.cpp:69-88: slot s counts channel s (0..2 = RGB, then guidance
 * planes when include_scale); mass[b] += 1/P, pixels in row-major order. */
void or_build_histograms(const double *planes, int W, int H, int bins, int nslots,
                         double *mass) {
  const size_t P = (size_t)W * H;
  const double inv = 1.0 / (double)P;
  for (int s = 0; s < nslots; ++s) {
    double *m = mass + (size_t)s * bins;
    for (int b = 0; b < bins; ++b) m[b] = 0.0;
    for (size_t i = 0; i < P; ++i) {
      int b = (int)floor(planes[s * P + i] * bins);
      b = b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
      m[b] = m[b] + inv;
    }
  }
}

/* optimizer.cpp:60-63 — floor(value * bins) evaluated in fp32. */
int or_bin_of(float v, int bins) {
  const float prod = v * (float)bins;
  int b = (int)floorf(prod);
  return b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
}

/* optimizer.cpp:90-108 over a neighbourhood of npix pixels x C channels. */
double or_histogram_penalty(const float *nb, int64_t npix, int C, int nslots, int bins,
                            const double *out_mass, const double *ex_mass) {
  if (npix == 0) return 0.0;
  double total = 0.0;
  for (int64_t p = 0; p < npix; ++p)
    for (int s = 0; s < nslots; ++s) {
      const int b = or_bin_of(nb[p * C + s], bins);
      const double diff = out_mass[(size_t)s * bins + b] - ex_mass[(size_t)s * bins + b];
      total = total + (diff > 0.0 ? diff : 0.0);
    }
  return total / (double)npix;
}

/* ---- M-step (optimizer.cpp:350-401) ---------------------------------------- */

/*
 * Candidates are the exemplar's dense windows (pipeline.cpp:276-277), so the
 * candidate value at window offset (dx, dy) of row `id` is the exemplar pixel
 * at (id % nxe + dx, id / nxe + dy) — read from cand[] directly here.
 */
int or_update_step(int C, int W, int H, int w, int sp, const float *cand, const int32_t *idx,
                   const double *irls, const double *pen, double *out_planes) {
  if (or_grid_validate(w, sp, W, H)) return OR_E_DOMAIN;
  int *xs = malloc(sizeof(int) * (W + 2)), *ys = malloc(sizeof(int) * (H + 2));
  const int nx = or_axis_positions(W, w, sp, xs), ny = or_axis_positions(H, w, sp, ys);
  const size_t P = (size_t)W * H, D = (size_t)w * w * C;
  double *acc = calloc(P * C, sizeof(double)), *wsum = calloc(P, sizeof(double));
  int status = OR_OK;
  for (int64_t a = 0; a < (int64_t)nx * ny && status == OR_OK; ++a) {
    const double we = irls[a] / (1.0 + pen[a]);  /* optimizer.hpp:32-34 */
    if (!(we > 0.0) || !isfinite(we)) { status = OR_E_DOMAIN; break; }
    const int ax = xs[a % nx], ay = ys[a / nx];
    const float *z = cand + (size_t)idx[a] * D;
    for (int dy = 0; dy < w; ++dy) {
      size_t pix = (size_t)(ay + dy) * W + ax;
      const float *zrow = z + (size_t)dy * w * C;
      for (int dx = 0; dx < w; ++dx, ++pix) {
        for (int c = 0; c < C; ++c) {
          const double t = we * (double)zrow[(size_t)dx * C + c];
          acc[pix * C + c] = acc[pix * C + c] + t;
        }
        wsum[pix] = wsum[pix] + we;
      }
    }
  }
  for (size_t pix = 0; pix < P && status == OR_OK; ++pix) {
    if (wsum[pix] <= 0.0) { status = OR_E_LOGIC; break; }
    const double inv = 1.0 / wsum[pix];
    for (int c = 0; c < C; ++c) {
      double v = acc[pix * C + c] * inv;
      v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
      out_planes[c * P + pix] = v;
    }
  }
  free(acc); free(wsum); free(xs); free(ys);
  return status;
}

/* optimizer.cpp:149-162 */
int or_assignment_distances(const double *planes, int C, int W, int H, int w, int sp,
                            const float *cand, const int32_t *idx, double *out) {
  int *xs = malloc(sizeof(int) * (W + 2)), *ys = malloc(sizeof(int) * (H + 2));
  const int nx = or_axis_positions(W, w, sp, xs), ny = or_axis_positions(H, w, sp, ys);
  const int64_t D = (int64_t)w * w * C;
  float *v = malloc(sizeof(float) * D);
  for (int64_t a = 0; a < (int64_t)nx * ny; ++a) {
    or_extract_window(planes, C, W, H, xs[a % nx], ys[a / nx], w, v);
    out[a] = or_full_distance(v, cand + (size_t)idx[a] * D, D);
  }
  free(v); free(xs); free(ys);
  return OR_OK;
}

/* ---- EM loop (optimizer.cpp:426-516), exact search --------------------------- */

/*
 * stats: 7 doubles per iteration {iter, energy, changed, nn_calls,
 * lsq_before, lsq_after, points_scanned} (optimizer.hpp:153-163);
 * points_scanned here = sum over plan entries of N (brute-force scan).
 * ex_mass == NULL disables histogram reweighting (pipeline.cpp:379-393).
 */
int or_optimize_level(const double *init, int C, int W, int H, int w, int sp, int p,
                      const float *cand, const double *proj, int64_t N, const double *mean,
                      const double *basis, int d, double r, double eps, int max_it, int min_it,
                      double frac, int bins, int nslots, const double *ex_mass, int threads,
                      double *out_planes, double *stats, int *n_iters) {
  if (or_grid_validate(w, sp, W, H)) return OR_E_DOMAIN;
  if (!(r > 0.0 && r < 2.0) || !(eps > 0.0) || max_it < 1 || min_it < 1 || min_it > max_it ||
      !(frac > 0.0 && frac < 1.0) || bins < 2 || p < 1 || p > sp)
    return OR_E_DOMAIN;  /* optimizer.cpp:24-42 */
  const int nx = or_axis_positions(W, w, sp, NULL), ny = or_axis_positions(H, w, sp, NULL);
  const int64_t A = (int64_t)nx * ny;
  const size_t P = (size_t)W * H;
  memcpy(out_planes, init, sizeof(double) * P * C);
  int32_t *cur = malloc(sizeof(int32_t) * A), *nxt = malloc(sizeof(int32_t) * A);
  double *cd = malloc(sizeof(double) * A), *nd = malloc(sizeof(double) * A);
  double *irls = malloc(sizeof(double) * A), *pen = malloc(sizeof(double) * A);
  double *after = malloc(sizeof(double) * A);
  double *omass = malloc(sizeof(double) * (size_t)bins * (nslots > 0 ? nslots : 1));
  const int64_t D = (int64_t)w * w * C;
  int64_t calls = 0;
  int st = or_search_step(out_planes, C, W, H, w, sp, p, cand, proj, N, mean, basis, d, NULL, 0,
                          threads, cur, cd, &calls);
  int64_t pending_calls = calls;
  int it_done = 0;
  for (int iter = 1; iter <= max_it && st == OR_OK; ++iter) {
    for (int64_t i = 0; i < A; ++i) { irls[i] = or_irls_weight(cd[i], r, eps); pen[i] = 0.0; }
    if (ex_mass) {
      or_build_histograms(out_planes, W, H, bins, nslots, omass);
      for (int64_t i = 0; i < A; ++i)
        pen[i] = or_histogram_penalty(cand + (size_t)cur[i] * D, (int64_t)w * w, C, nslots, bins,
                                      omass, ex_mass);
    }
    double lsq_before = 0.0;
    for (int64_t i = 0; i < A; ++i) {
      const double we = irls[i] / (1.0 + pen[i]);
      lsq_before = lsq_before + we * cd[i] * cd[i];
    }
    st = or_update_step(C, W, H, w, sp, cand, cur, irls, pen, out_planes);
    if (st) break;
    or_assignment_distances(out_planes, C, W, H, w, sp, cand, cur, after);
    double lsq_after = 0.0;
    for (int64_t i = 0; i < A; ++i) {
      const double we = irls[i] / (1.0 + pen[i]);
      lsq_after = lsq_after + we * after[i] * after[i];
    }
    st = or_search_step(out_planes, C, W, H, w, sp, p, cand, proj, N, mean, basis, d, NULL, 0,
                        threads, nxt, nd, &calls);
    if (st) break;
    int64_t changed = 0;
    for (int64_t i = 0; i < A; ++i) changed += nxt[i] != cur[i];
    double *s = stats + 7 * (iter - 1);
    s[0] = iter;
    s[1] = or_energy(nd, A, r);
    s[2] = (double)changed;
    s[3] = (double)(calls + pending_calls);
    s[4] = lsq_before;
    s[5] = lsq_after;
    s[6] = (double)(calls + pending_calls) * (double)N;
    pending_calls = 0;
    it_done = iter;
    memcpy(cur, nxt, sizeof(int32_t) * A);
    memcpy(cd, nd, sizeof(double) * A);
    if (iter >= min_it && (double)changed < frac * (double)A) break;
  }
  *n_iters = it_done;
  free(cur); free(nxt); free(cd); free(nd); free(irls); free(pen); free(after); free(omass);
  return st;
}

/* ---- L0 resampling + driver helpers ------------------------------------------ */

/* image.cpp:38-62, one plane. */
int or_downsample_plane(const double *in, int W, int H, int f, double *out) {
  if (f < 1) return OR_E_DOMAIN;
  const int ow = W / f, oh = H / f;
  if (ow < 1 || oh < 1) return OR_E_DOMAIN;
  const double inv = 1.0 / ((double)f * f);
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) {
      double acc = 0.0;
      for (int dy = 0; dy < f; ++dy)
        for (int dx = 0; dx < f; ++dx) acc = acc + in[(size_t)(y * f + dy) * W + x * f + dx];
      out[(size_t)y * ow + x] = acc * inv;
    }
  return OR_OK;
}

static void src_coord(int dst, int limit, double inv, int *lo, int *hi, double *frac) {
  const double s = (dst + 0.5) * inv - 0.5;
  const double fl = floor(s);
  *lo = (int)fl;
  *frac = s - fl;
  *hi = *lo + 1 < limit - 1 ? *lo + 1 : limit - 1;
  if (*lo < 0) *lo = 0;
  if (*hi < *lo) *hi = *lo;
}

/* image.cpp:64-109, one plane. */
int or_upsample_bilinear_plane(const double *in, int W, int H, int f, double *out) {
  if (f < 1) return OR_E_DOMAIN;
  const int ow = W * f, oh = H * f;
  if (f == 1) { memcpy(out, in, sizeof(double) * (size_t)W * H); return OR_OK; }
  const double inv = 1.0 / f;
  for (int y = 0; y < oh; ++y) {
    int y0, y1; double fy;
    src_coord(y, H, inv, &y0, &y1, &fy);
    for (int x = 0; x < ow; ++x) {
      int x0, x1; double fx;
      src_coord(x, W, inv, &x0, &x1, &fx);
      const double v00 = in[(size_t)y0 * W + x0], v10 = in[(size_t)y0 * W + x1];
      const double v01 = in[(size_t)y1 * W + x0], v11 = in[(size_t)y1 * W + x1];
      const double a = (1.0 - fx) * v00 + fx * v10;
      const double b = (1.0 - fx) * v01 + fx * v11;
      out[(size_t)y * ow + x] = (1.0 - fy) * a + fy * b;
    }
  }
  return OR_OK;
}

/* pipeline.cpp:39-52, one plane: crop or edge-replicate. */
void or_fit_to_plane(const double *in, int W, int H, int ow, int oh, double *out) {
  for (int y = 0; y < oh; ++y) {
    const int sy = y < H - 1 ? y : H - 1;
    for (int x = 0; x < ow; ++x) {
      const int sx = x < W - 1 ? x : W - 1;
      out[(size_t)y * ow + x] = in[(size_t)sy * W + sx];
    }
  }
}
