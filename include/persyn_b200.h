/*
 * persyn_b200.h — C ABI of the B200-native EM hot path of persyn
 * (perspective texture synthesis by energy optimisation, arXiv 2006.11851).
 *
 * This is the drop-in boundary for the reference's hot path.  Each entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/proj/core).  The reference is C++ with a per-query virtual
 * plug-in (SearchIndex::nearest, include/persyn/optimizer.hpp:111-119); a GPU
 * is fed at batch granularity, so the boundary sits at the reference's batch
 * entry points (search_step / update_step / optimize_level / synthesize) and a
 * batched SearchIndex::nearest.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *  - HOST pointers unless a name ends in `_dev` (device-resident variants used
 *    by the benchmark; they take CUDA device pointers).
 *  - Images are planar fp64, planes [C][H][W], row-major, row 0 = bottom
 *    (include/persyn/image.hpp:11-12,57-59).  C = 3 + G: R, G, B then G >= 1
 *    guidance planes (the reference hard-codes G = 1, image.hpp:70; G = 2 is
 *    the cfg-3 extension).
 *  - Neighbourhood vectors are fp32, pixel-major (dy, dx), channel-minor
 *    (src/neighborhood.cpp:128-135).  D = w * w * C.
 *  - Caller owns every host array; handles own device memory; results are
 *    copied into caller buffers.
 *  - Errors: every call returns psg_status; psg_last_error() returns the
 *    thread-local message of the last failure.  No exception crosses the ABI.
 *    The mapping mirrors include/persyn/errors.hpp:8-36 and the reference's
 *    std::logic_error invariants (src/optimizer.cpp:342-346,390-392).
 *  - Arithmetic: fp64 with separate multiply and add in the reference's index
 *    order; fp32 features = (float) of fp64 state.  NN results in exact mode
 *    are bit-identical to the reference's KmTree exact query / brute force.
 *  - No CPU fallback: without a usable sm_100 device psg_ctx_create fails
 *    with PSG_E_CUDA.
 */
#ifndef PERSYN_B200_H
#define PERSYN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSG_ABI_VERSION 2

typedef enum {
  PSG_OK = 0,
  PSG_E_DOMAIN = 1, /* persyn::DomainError (errors.hpp:33-36)            */
  PSG_E_SHAPE = 2,  /* persyn::ShapeError  (errors.hpp:26-30)            */
  PSG_E_LOGIC = 3,  /* std::logic_error    (optimizer.cpp:344,391)       */
  PSG_E_IO = 4,     /* persyn::IoError     (errors.hpp:14-18)            */
  PSG_E_FORMAT = 5, /* persyn::FormatError (errors.hpp:20-24)            */
  PSG_E_CUDA = 6,   /* CUDA runtime / driver / library failure           */
  PSG_E_NCCL = 7    /* NCCL failure (multi-GPU row sharding)             */
} psg_status;

/* QueryBudget (include/persyn/km_tree.hpp:13-25). */
typedef enum { PSG_GREEDY = 0, PSG_BACKTRACK = 1, PSG_EXACT = 2 } psg_mode;
typedef struct {
  int mode;       /* psg_mode */
  int max_leaves; /* backtrack only, >= 1 */
} psg_budget;

/* Per-stage index build parameters (PcaTreeIndex ctor, optimizer.cpp:216-224,
 * extended with the BASELINE configs' d cap and tree depth). */
typedef struct {
  double variance_target; /* fit_pca target in (0,1] (pca.cpp:79-87)          */
  int d_cap;              /* 0 = no cap; else retained dim <= d_cap           */
  int d_fixed;            /* 0 = variance rule; else exactly d_fixed comps    */
  int branching;          /* k-means tree branching b >= 2                    */
  int max_depth;          /* 0 = until leaves < leaf_threshold; else cap      */
  int leaf_threshold;     /* 0 = branching (optimizer.cpp:223)                */
  uint64_t seed;          /* tree seed (pipeline.cpp:54-56 level_seed)        */
  int hist_bins;          /* exemplar histogram bins, 0 = none                */
  int hist_include_scale; /* histogram over guidance planes too               */
  int tree_kind;          /* psg_tree_kind                                    */
} psg_index_cfg;

/* Which k-means tree an index builds.  Exact queries return the same answer on
 * any tree (km_tree.cpp:251-278); greedy / backtrack(m) answers depend on it.
 *  PSG_TREE_DEVICE    : built on the device, level-synchronous, one RNG stream
 *                       per node, optional depth cap (max_depth).
 *  PSG_TREE_REFERENCE : the reference's own tree, KmTree::build
 *                       (km_tree.cpp:141-195) replicated exactly -- one
 *                       std::mt19937_64 consumed in the recursion's order,
 *                       unbounded depth (max_depth must be 0) -- so that
 *                       greedy / backtrack(m) answers equal the reference's
 *                       make_pca_tree_index (optimizer.cpp:214-224). */
typedef enum { PSG_TREE_DEVICE = 0, PSG_TREE_REFERENCE = 1 } psg_tree_kind;

/* OptimizerConfig (include/persyn/optimizer.hpp:37-52). */
typedef struct {
  double robust_exponent;      /* r in (0,2), default 0.8            */
  double distance_epsilon;     /* > 0, default 1e-4                  */
  int max_iterations;          /* >= 1                               */
  int min_iterations;          /* in [1, max_iterations]             */
  double convergence_fraction; /* in (0,1)                           */
  int histogram_bins;          /* >= 2                               */
  int histogram_matching;      /* bool                               */
  int histogram_include_scale; /* bool                               */
  int spacing;                 /* anchor lattice step (GridSpec)     */
  int patch_width;             /* PatchSpec, <= spacing              */
  psg_budget budget;
} psg_opt_cfg;

/* IterationStats (include/persyn/optimizer.hpp:153-163). */
typedef struct {
  int iteration;
  double energy;
  int64_t changed;
  int64_t nn_calls;
  double millis;
  double lsq_energy_before;
  double lsq_energy_after;
  int64_t points_scanned;   /* sum over the reference's query plan */
  int64_t unique_queries;   /* anchors actually searched on device */
  int64_t unique_points_scanned; /* points scanned by those searches */
} psg_iter_stats;

typedef struct psg_ctx psg_ctx;
typedef struct psg_index psg_index;
typedef struct psg_level psg_level;

/* ---- context ------------------------------------------------------------ */
const char* psg_last_error(void);
int psg_abi_version(void);
/* stream: a cudaStream_t (NULL = the context creates its own). */
psg_status psg_ctx_create(int device, void* stream, psg_ctx** out);
void psg_ctx_destroy(psg_ctx* ctx);
psg_status psg_ctx_synchronize(psg_ctx* ctx);
/* Number of kernel launches issued by this context so far. */
int64_t psg_ctx_launch_count(const psg_ctx* ctx);
/* Per-kernel CUDA-event timing on the context stream (benchmark/roofline).
 * enable != 0 starts recording (and resets the totals). */
psg_status psg_ctx_profile(psg_ctx* ctx, int enable);
/* Copies up to n (name, total milliseconds, launches) entries of the kernels
 * timed since profiling was enabled; returns the number of kernel kinds. */
int psg_ctx_kernel_times(psg_ctx* ctx, const char** names, double* ms, int64_t* launches, int n);

/* ---- search index (SearchIndex plug-in, optimizer.hpp:111-129) ----------- */
/*
 * Replaces make_pca_tree_index(extract_all(exemplar, {w,1,..}), variance,
 * branching, seed) (optimizer.cpp:256-262, pipeline.cpp:276-284).  The dense
 * database is never materialised: windows are gathered from the exemplar on
 * device.  mean/basis: optional injected PCA model (PcaModel ctor,
 * pca.hpp:18-19) — mean[D], basis[d][D] row-major; NULL = fit on device.
 */
psg_status psg_index_create(psg_ctx* ctx, const double* ex_planes, int C, int ew, int eh, int w,
                            const double* mean, const double* basis, int d,
                            const psg_index_cfg* cfg, psg_index** out);
/* Same over an explicit fp32 vector set X[n][D] (search-only workloads). */
psg_status psg_index_create_vectors(psg_ctx* ctx, const float* X, int64_t n, int D,
                                    const double* mean, const double* basis, int d,
                                    const psg_index_cfg* cfg, psg_index** out);
/*
 * Replaces make_brute_force_index(extract_all(exemplar, {w,1,..}))
 * (optimizer.hpp:122-129, optimizer.cpp:168-212, the pixel-brute bench mode
 * persyn_main.cpp:205-212): exact full-D nearest neighbour, the first index of
 * the minimum fp64 dist^2; QueryBudget is ignored; points_scanned = N per
 * query.  Computed as a tf32 tensor-core distance filter with exact fp64
 * re-evaluation of the survivors (bit-identical result).  hist_bins > 0 also
 * builds the exemplar histogram used by optimize_level.
 */
psg_status psg_index_create_brute(psg_ctx* ctx, const double* ex_planes, int C, int ew, int eh,
                                  int w, int hist_bins, int hist_include_scale, psg_index** out);
/* Same over an explicit fp32 candidate set X[n][D]. */
psg_status psg_index_create_brute_vectors(psg_ctx* ctx, const float* X, int64_t n, int D,
                                          psg_index** out);
void psg_index_destroy(psg_index* index);
/* dims: {N, D, d, C, w, ew, eh, n_nodes, n_leaves, max_depth_built} */
psg_status psg_index_info(const psg_index* index, int64_t dims[10]);
/* PcaModel accessors (pca.hpp:21-31): mean[D], basis[d][D], variances[D]. */
psg_status psg_index_pca(const psg_index* index, double* mean, double* basis, double* variances);
/* ProjectedMatrix of the database (pca.cpp:103-113), [N][d] row-major. */
psg_status psg_index_projected(const psg_index* index, double* out);
/* Leaves in tree order (KmTree::leaves, km_tree.cpp:286-298). */
psg_status psg_index_leaves(const psg_index* index, int32_t* ids, int32_t* sizes,
                            int64_t* n_leaves);
/*
 * Tree replay: replaces the index's k-means tree by an externally built one,
 * e.g. the reference's KmTree (KmTree::build, km_tree.cpp:141-195) recovered
 * from its public structure_json() and leaves() (km_tree.cpp:286-318).  With
 * the reference's tree imported, greedy and backtrack(m) queries reproduce
 * KmTree::query (km_tree.cpp:213-250) bit-for-bit, including the heap
 * tie-break on the reference's post-order node ids.  Centroids and radii are
 * recomputed from the leaf membership with the reference's ordered loops.
 *   n_children[n_nodes]: child counts in pre-order DFS (children in order)
 *   leaf_sizes[n_leaves], leaf_ids[N]: KmTree::leaves(), concatenated
 */
typedef struct {
  int64_t n_nodes;
  const int32_t* n_children;
  int64_t n_leaves;
  const int32_t* leaf_sizes;
  const int32_t* leaf_ids;
} psg_tree_import;
psg_status psg_index_import_tree(psg_ctx* ctx, psg_index* index, const psg_tree_import* tree);

/* The library's replica of KmTree::build (km_tree.cpp:141-195: one
 * std::mt19937_64 consumed in the recursion's order) over N projected points
 * proj[N][d], on the HOST (no device needed) -- what tree_kind =
 * PSG_TREE_REFERENCE builds inside psg_index_create.  Outputs in
 * psg_tree_import's form: n_children (pre-order, capacity 2N), leaf_sizes
 * (capacity N), leaf_ids (N).  leaf_threshold <= 0: the branching. */
psg_status psg_reference_tree_host(const double* proj, int64_t N, int d, int branching,
                                   int leaf_threshold, uint64_t seed, int32_t* n_children,
                                   int64_t* n_nodes, int32_t* leaf_sizes, int64_t* n_leaves,
                                   int32_t* leaf_ids);
/* Exemplar histogram [slots][bins] (pipeline.cpp:286-292). */
psg_status psg_index_histograms(const psg_index* index, double* mass);
/*
 * Batched SearchIndex::nearest (PcaTreeIndex::nearest, optimizer.cpp:226-236):
 * project -> tree query -> full-D rescoring.  Q[nq][D] fp32.
 * dist_pca (optional): sqrt of the PCA-space dist^2 of the winner (what
 * KmTree::query returns before PcaTreeIndex replaces it).
 */
psg_status psg_index_query(psg_ctx* ctx, const psg_index* index, const float* Q, int64_t nq,
                           psg_budget budget, int32_t* idx, double* dist, double* dist_pca,
                           int64_t* scanned);

/* ---- EM hot path --------------------------------------------------------- */
/*
 * search_step (optimizer.hpp:141-143, optimizer.cpp:275-348).  out_planes is
 * the W x H current image (C planes, C = index C).  idx/dist: A = nx*ny
 * anchors in ascending id.  nn_calls = the reference's plan size
 * (optimizer.cpp:333); scanned = points scanned summed over the plan.
 */
psg_status psg_search_step(psg_ctx* ctx, const psg_index* index, const double* out_planes, int W,
                           int H, int spacing, int patch_width, psg_budget budget, int32_t* idx,
                           double* dist, int64_t* nn_calls, int64_t* scanned);
/*
 * update_step (optimizer.hpp:149-151, optimizer.cpp:350-401) with
 * WeightMap{irls, hist_penalty} (optimizer.hpp:27-35).  Writes the new image.
 */
psg_status psg_update_step(psg_ctx* ctx, const psg_index* index, const int32_t* idx,
                           const double* irls, const double* pen, int W, int H, int spacing,
                           double* out_planes);
/*
 * optimize_level (optimizer.hpp:181-183, optimizer.cpp:426-516).
 * ex_hist: optional exemplar histogram [slots][bins]; NULL with
 * cfg->histogram_matching uses the index's own exemplar histogram.
 * stats: array of cfg->max_iterations entries (may be NULL).
 */
psg_status psg_optimize_level(psg_ctx* ctx, const psg_index* index, const double* init, int W,
                              int H, const psg_opt_cfg* cfg, const double* ex_hist,
                              double* out_planes, psg_iter_stats* stats, int* n_iters);

/* ---- device-resident level (benchmark / driver internals) ---------------- */
psg_status psg_level_create(psg_ctx* ctx, const psg_index* index, const double* init, int W,
                            int H, const psg_opt_cfg* cfg, const double* ex_hist,
                            psg_level** out);
/* Priming search (optimize_level's first search_step, optimizer.cpp:444-448). */
psg_status psg_level_prime(psg_level* level);
/* Run up to n EM iterations; stops early on the reference's convergence rule
 * only when honor_convergence != 0.  Appends stats. */
psg_status psg_level_iterate(psg_level* level, int n, int honor_convergence,
                             psg_iter_stats* stats, int* n_done);
psg_status psg_level_download(psg_level* level, double* planes, int32_t* idx, double* dist);
/* Device pointers of the level's fp64 state planes (for device-side checks). */
psg_status psg_level_state_dev(psg_level* level, void** planes_dev, void** idx_dev,
                               void** dist_dev);
/* Per-anchor QueryStats of the level's last search (km_tree.hpp:27-30):
 * points scanned, points evaluated in exact fp64, tree nodes visited. */
psg_status psg_level_query_stats(psg_level* level, int64_t* scanned, int64_t* exact_evals,
                                 int32_t* nodes_visited);
void psg_level_destroy(psg_level* level);

/* ---- row-sharded multi-GPU ---------------------------------- */
/* Rank `rank` of `world` owns anchor rows [a0, a1) and pixel rows [p0, p1) of
 * the W x H output; its windows read rows [p0, e1) (halo rows [p1, e1) come
 * from rank+1) and its pixels are also covered by anchor rows [hlo, a0) of
 * rank-1, accumulated in ascending anchor id: bit-identical to one device. */
typedef struct {
  int W, H, w, spacing, rank, world;
  int p0, p1, e1;
  int hlo, a0, a1;
  int nx, ny; /* anchors per row, anchor rows of the whole image */
} psg_band;
psg_status psg_shard_plan(int W, int H, int w, int spacing, int rank, int world, psg_band* out);
/* rows: host [C][e1-p0][W], the band's local rows of the initial image. */
psg_status psg_band_create(psg_ctx* ctx, const psg_index* index, const double* rows,
                           const psg_band* band, const psg_opt_cfg* cfg, const double* ex_hist,
                           psg_level** out);
/* One EM iteration = phase1..4 + commit; exchanges happen in between:
 *  phase1: IRLS weights; owned-row histogram counts -> counts_dev (u64 [slots*bins], device)
 *  [all-reduce(sum) of the counts]
 *  phase2: fold global counts, penalties, weights; pack {eff[n] (f64), idx[n] (i32)} of owned
 *          anchor rows [send_row0, a1) into send_dev (device) for rank+1
 *  [send to rank+1 / receive rank-1's rows [hlo, a0) in the same format]
 *  phase3: M-step of owned pixel rows; copy owned mirror rows [p0, p0+n_send_rows) (f32
 *          [rows][W][C]) into send_rows_dev for rank-1
 *  [send to rank-1 / receive rows [p1, e1) from rank+1]
 *  phase4: halo rows in; lsq diagnostic, E-step; partials[9] = {lsq_before, lsq_after, energy,
 *          changed, points_scanned, unique points scanned, nn_calls, priming nn_calls,
 *          unique queries} of this rank
 *  [sum the partials over ranks in rank order]
 *  commit: record global stats (sums over ranks) and advance.
 * phase1..3 only ENQUEUE work on the context stream (no host synchronisation):
 * the exchanges must be ordered against that stream -- enqueued on it (NCCL
 * with the context created on the communicator's stream) or preceded by
 * psg_ctx_synchronize.  phase4 synchronises (it returns host partials) and
 * reports device-side errors raised by any phase of the iteration. */
psg_status psg_band_phase1(psg_level* level, unsigned long long* counts_dev);
psg_status psg_band_phase2(psg_level* level, const unsigned long long* global_counts_dev,
                           int send_row0, void* send_dev);
psg_status psg_band_phase3(psg_level* level, const void* recv_dev, int n_send_rows,
                           float* send_rows_dev);
psg_status psg_band_phase4(psg_level* level, const float* recv_rows_dev, double* partials);
psg_status psg_band_commit(psg_level* level, const double* global_partials, psg_iter_stats* st);

/* ---- multi-GPU: NCCL inside the library (shard.cpp) -------------------------
 * One process (or thread) per GPU, one psg_ctx per GPU.  Rank 0 makes a
 * unique id (128 bytes) and the caller distributes it (MPI, a file,
 * torch.distributed, ...); every rank then creates its communicator.  NCCL is
 * loaded at psg_comm_unique_id / psg_comm_create (libnccl.so.2).
 * psg_band_iterate runs n EM iterations of a band created with
 * psg_band_create (after psg_level_prime) with the four exchanges of the
 * phase list above enqueued as NCCL collectives / send-recv on the context
 * stream; the convergence rule (optimizer.cpp:509-513) uses the global
 * `changed`, so every rank stops after the same iteration, and stats hold the
 * global (rank-order) sums.  Results are bit-identical to one device. */
typedef struct psg_comm psg_comm;
psg_status psg_comm_unique_id(void* id128);
psg_status psg_comm_create(psg_ctx* ctx, const void* id128, int world, int rank, psg_comm** out);
void psg_comm_destroy(psg_comm* comm);
psg_status psg_band_iterate(psg_level* band, psg_comm* comm, int n, int honor_convergence,
                            psg_iter_stats* stats, int* n_done);
/* optimize_level (optimizer.cpp:426-516) of this rank's row band:
 * rows = [C][e1-p0][W] host rows of the initial image (psg_shard_plan(W, H, w,
 * spacing, rank, world)); out_rows = [C][p1-p0][W] the band's owned rows. */
psg_status psg_optimize_level_sharded(psg_ctx* ctx, psg_comm* comm, const psg_index* index,
                                      const double* rows, int W, int H, const psg_opt_cfg* cfg,
                                      const double* ex_hist, double* out_rows,
                                      psg_iter_stats* stats, int* n_iters);
/* The same band schedule for `world` bands of one image in this process, the
 * exchanges as device copies (tests the exchange buffers on one GPU). */
psg_status psg_optimize_level_loopback(psg_ctx* ctx, const psg_index* index, const double* init,
                                       int W, int H, const psg_opt_cfg* cfg, const double* ex_hist,
                                       int world, double* out_planes, psg_iter_stats* stats,
                                       int* n_iters);

/* ---- pyramid driver (synthesize, pipeline.hpp:69, pipeline.cpp:216-315) --- */
typedef struct {
  int n_sizes;
  int sizes[4]; /* neighbourhood widths per level, coarse stages first, e.g. {32,16,8} */
} psg_stage_list;

typedef struct {
  const double* exemplar;  /* [C][eh][ew] fp64: RGB + guidance planes */
  int C, ew, eh;
  const double* out_guidance; /* [C-3][H][W] guidance planes of the finest output level */
  int out_w, out_h;
  int levels;
  psg_stage_list stages;   /* per-level neighbourhood sizes; spacing = w / 4 */
  psg_opt_cfg cfg;         /* spacing ignored (w/4 per stage) */
  psg_index_cfg index;
  uint64_t seed;           /* initialize_output's engine seed; trees use level_seed(seed, l) */
  int guidance_kind;       /* 0 = guidance planes are row/col ramps recomputed per level */
  /* Optional injected PCA model per stage (stage s = level * n_sizes + size
   * index; NULL arrays or a NULL entry = fit on the device): mean [D],
   * basis [d][D] row-major, d = stage_d[s].  The reference fits with Eigen
   * (absent here): injection makes stage-by-stage parity checkable. */
  const double* const* stage_mean;
  const double* const* stage_basis;
  const int* stage_d;
  int index_kind;          /* a psg_index_kind: IndexKind, pipeline.hpp:13-16 */
  psg_iter_stats* trace;   /* optional [trace_cap]: every stage's iterations, in order */
  int trace_cap;
} psg_request;

/* IndexKind (pipeline.hpp): the per-stage SearchIndex of synthesize. */
typedef enum { PSG_INDEX_PCA_TREE = 0, PSG_INDEX_BRUTE_FORCE = 1 } psg_index_kind;

typedef struct {
  int level, w, W, H, ew, eh, d, iterations;
  double final_energy;
  int64_t nn_calls;
  double index_millis, optimize_millis;
  int trace_first, trace_count; /* this stage's iterations in psg_request.trace */
} psg_stage_report;

typedef struct {
  int n_stages;
  psg_stage_report stages[16];
  double part1_millis, part2_millis;
  int64_t total_nn_calls;
  double final_energy;
  int n_trace; /* iterations run (may exceed trace_cap) */
} psg_report;

/* out_planes: [C][out_h][out_w] fp64 final state (RGB = the synthesized image).
 * Part 1 is the reference's initialize_output (below) with the guidance row
 * ramp (plane 3) as the normalised scale map (bounds [0, 1]); each level l > 0
 * starts from upsample_bilinear(x2) + fit_to of the previous level's RGB with
 * the level's guidance re-imposed (pipeline.cpp:269-274).
 * Threads: the stages' indexes are built ahead of the EM loop by up to three
 * worker threads of this call, each on a context owned by `ctx` (created on
 * first use, destroyed with it); they are joined before the call returns.
 * index_millis is a stage's own build time (stages overlap, so the sum may
 * exceed the wall time).  Results do not depend on the overlap. */
psg_status psg_synthesize(psg_ctx* ctx, const psg_request* req, double* out_planes,
                          psg_report* report);

/* initialize_output (pipeline.hpp:61-62, pipeline.cpp:96-175): scale-matched
 * copy of exemplar pixels.  ex_planes [C >= 4][eh][ew] with plane 3 = the
 * exemplar's S channel (normalised scale); out_scale [oh][ow] = the output
 * ScaleMap's raw (unnormalised) float values; bounds {s_min, s_max}; seed of
 * the std::mt19937_64 the reference passes in.  out4 [4][oh][ow] = RGB + the
 * normalised target S (normalized_plane, pipeline.cpp:23-35).  Host code:
 * sequential draws from one engine, exactly the reference's picks. */
psg_status psg_initialize_output(const double* ex_planes, int C, int ew, int eh,
                                 const float* out_scale, int ow, int oh, double s_min,
                                 double s_max, uint64_t seed, double* out4);

/* Diagnostics of the E-step's projection at every anchor (spacing sp) of an
 * image [C][H][W]: q_tc = the tensor-core approximation, delta = its rigorous
 * error bound (2-norm), q_exact = the reference's fp64 chain (pca.cpp:27-41).
 * Any output may be NULL.  Fails with PSG_E_DOMAIN when the index has no
 * tensor-core operand (vector index, d > 64, ...). */
psg_status psg_debug_projection(psg_ctx* ctx, const psg_index* index, const double* planes, int W,
                                int H, int spacing, double* q_tc, float* delta, double* q_exact);

/* ---- resampling between levels (device kernels over host buffers) ---------- */
/* downsample (image.cpp:38-62): block mean, factor >= 1, C planes [C][H][W] ->
 * [C][H/f][W/f]. */
psg_status psg_downsample(psg_ctx* ctx, const double* in, int C, int W, int H, int factor,
                          double* out);
/* upsample_bilinear (image.cpp:64-109): half-pixel centres, clamped border ->
 * [C][H*f][W*f]. */
psg_status psg_upsample_bilinear(psg_ctx* ctx, const double* in, int C, int W, int H,
                                 int factor, double* out);
/* fit_to (pipeline.cpp:39-52): crop or edge-replicate to [C][oh][ow]. */
psg_status psg_fit_to(psg_ctx* ctx, const double* in, int C, int W, int H, int ow, int oh,
                      double* out);

/* ---- geometry helpers (neighborhood.cpp) ---------------------------------- */
/* axis_positions (neighborhood.cpp:12-18); returns count, fills out if non-NULL. */
int psg_axis_positions(int extent, int window, int step, int* out);
/* Plan size (nn_calls) and per-anchor multiplicity of search_step's plan
 * (optimizer.cpp:288-296); mult may be NULL.  Returns -1 if an anchor is
 * uncovered (the reference's logic_error, optimizer.cpp:342-346). */
int64_t psg_plan(int W, int H, int w, int spacing, int patch_width, int32_t* mult);

/* ---- numerics helpers (host; the device kernels use the same code) -------- */
/* Correctly rounded x^y (double-double), used for the IRLS weight where the
 * reference calls glibc pow (optimizer.cpp:114, :129). */
double psg_pow_cr(double x, double y);
/* The exact value of `count` sequential additions of 1/pixels starting from 0
 * (build_histograms' mass, optimizer.cpp:76-86). */
double psg_hist_mass(int64_t count, int64_t pixels);

#ifdef __cplusplus
}
#endif

#endif /* PERSYN_B200_H */
