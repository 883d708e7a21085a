// Internal declarations shared by the host runtime and the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "persyn_b200.h"

namespace psg {
// largest retained PCA dimension (the warp search kernels and the fp64
// projection; the tile search and the tensor-core projection take d <= 64)
constexpr int kMaxDP = 128;

// ---- error plumbing (status codes of include/persyn_b200.h) -----------------
struct Error : std::runtime_error {
  psg_status code;
  Error(psg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(psg_status c, const std::string& m) { throw Error(c, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    fail(PSG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                         std::to_string(line) + ")");
}
#define PSG_CUDA(x) ::psg::cuda_check((x), #x, __FILE__, __LINE__)
#define PSG_LAUNCHED(ctx) \
  do {                      \
    PSG_CUDA(cudaGetLastError()); \
    (ctx)->launches++;      \
  } while (0)

// Device-side error flags (bit set -> status at the next host check).
enum DevFlag : int {
  FLAG_BAD_WEIGHT = 1,     // non-positive / non-finite update weight (optimizer.cpp:367-369)
  FLAG_UNCOVERED = 2,      // pixel with wsum <= 0 (optimizer.cpp:390-392)
  FLAG_STACK_OVERFLOW = 4, // traversal stack exhausted (must never happen)
  FLAG_BAD_DISTANCE = 8,   // negative distance into irls_weight (optimizer.cpp:113)
};

// Tree in breadth-first layout: children of a node are contiguous.
struct DevTree {
  int n_nodes = 0;
  int max_depth = 0;
  int max_children = 0;
  double* centroid = nullptr;  // [n_nodes][d]
  double* radius = nullptr;    // [n_nodes]
  int32_t* first_child = nullptr;
  int32_t* n_children = nullptr;  // 0 = leaf
  int32_t* leaf_start = nullptr;  // leaves: range in the leaf-ordered point arrays
  int32_t* leaf_count = nullptr;
  // fp32 bound data (conservative: radius and norms rounded up, boxes outward)
  float* centroid32 = nullptr;  // [n_nodes][d]
  float* centroid32T = nullptr; // [d][n_nodes]: children of a node are contiguous per dim
  float* radius32 = nullptr;
  float* cnorm32 = nullptr;     // |centroid|
  float* boxlo = nullptr;       // [kBoxDims][n_nodes] per-dim minimum over the subtree
  float* boxhi = nullptr;       // [kBoxDims][n_nodes]
  float* box2 = nullptr;        // [n_nodes][kBoxDims][2]: (lo_j, -hi_j) per node, 64 contiguous bytes
  int2* meta = nullptr;         // {first_child, -n_children} or {leaf_start, leaf_count}
  int32_t* tie = nullptr;       // optional backtrack tie-break id per node (null = node index)
  // fp64 centroid rows, pair-interleaved per sibling block (search_backtrack_group_kernel)
  double* centroid_il = nullptr;
};
#ifndef PSG_BOX_DIMS
#define PSG_BOX_DIMS 8
#endif
constexpr int kBoxDims = PSG_BOX_DIMS;  // leading PCA dims carrying bounding boxes

struct HostTree {
  std::vector<double> centroid, radius;
  std::vector<int32_t> first_child, n_children, leaf_start, leaf_count, depth;
  std::vector<int32_t> perm;  // leaf order -> point id
  std::vector<double> boxlo, boxhi;  // [n_nodes][kBoxDims]
  std::vector<int32_t> tie;          // empty = node index (own trees)
  int max_depth = 0;
  int n_leaves = 0;
};

// Per-stage index: exemplar level + PCA model + projected DB + tree.
struct Index {
  psg_ctx* ctx = nullptr;
  bool from_vectors = false;
  int C = 0, w = 0, ew = 0, eh = 0, D = 0, d = 0;
  int64_t N = 0;
  int nxe = 0;              // dense DB anchors per row (ew - w + 1)
  float* ex_mirror = nullptr;  // [eh][ew][C] fp32 (image index)
  float* ex_mirror8 = nullptr; // [eh][ew][8] fp32, channels zero-padded (C <= 8)
  float* vectors = nullptr;    // [N][D] fp32 (vector index)
  double* mean = nullptr;      // [D]
  double* basis = nullptr;     // [d][D]
  double* proj = nullptr;      // [N][d] original order
  double* proj_soa = nullptr;  // [d][N] leaf order
  double* proj_leaf = nullptr; // [N][d] leaf order (budget searches: a leaf's rows are contiguous)
  double* proj_leaf_il = nullptr;  // the same rows pair-interleaved per leaf (search_backtrack_group_kernel)
  float* proj32_q4 = nullptr;  // [dp/4][N] float4 groups, leaf order, fp32 filter copy
  int dp = 32;
  float* pnorm32 = nullptr;    // [N] leaf order, |p| rounded up
  float2* pp32 = nullptr;      // [N] leaf order, (|p~|^2, |p~_B|^2) of the fp32 point (B: kernels_search.cu P2_SPLIT_DEN)
  float pnorm_max = 0.f;
  int32_t* perm = nullptr;     // leaf order -> id
  DevTree tree;
  HostTree htree;
  std::vector<double> h_mean, h_basis, h_var;
  // exemplar histogram
  int hist_bins = 0, hist_slots = 0;
  std::vector<double> h_ex_hist;
  double* ex_hist = nullptr;
  // brute-force index (BruteForceIndex, optimizer.cpp:168-212): tensor-core
  // filter operand, tf32-rounded centred rows in UMMA tiles + norms
  bool brute = false;
  int brute_nch = 0;            // K chunks of 32 fp32
  int brute_ptiles = 0;         // 256-point tiles
  float* brute_op = nullptr;    // [ptiles][nch][256 * 32]
  float* brute_n2 = nullptr;    // [ptiles * 256] |p - mu|^2 (fp32)
  float* brute_nup = nullptr;   // [ptiles * 256] |p - mu| rounded up
  float* brute_mu = nullptr;    // [nch * 32] centring vector
  float* brute_tmax = nullptr;  // [ptiles] largest |p - mu| bound per tile
  // tensor-core window projection (kernels_project_tc.cu): the basis rounded to
  // Bq = rint(B * 2^22) as three signed base-256 digit slices in UMMA K-major
  // layout over 8-byte pixels, plus row sums for the error bound
  bool tc = false;
  int tc_kb = 0;               // K bytes per slice: w * w * 8 (8-byte pixels), multiple of 32
  int8_t* tc_b = nullptr;      // [d/32 blocks][kb / 16][4 digits x 32 rows][16]
  double* tc_bmu = nullptr;    // [d] B . mean (rounded from long double)
  float tc_delta = 0.f;        // rigorous |q^ - q| bound (2-norm) of every query
  ~Index();
};

// A set of fp32 rows read in the reference's feature order: explicit vectors
// [n][D], or w x w windows of an fp32 mirror [H][img_w][C] (pixel-major,
// channel-minor, neighborhood.cpp:128-135) at anchors (xs[r % nx], ys[r / nx])
// — or the dense lattice (r % nx, r / nx) when xs is null.
struct RowSrc {
  const float* base = nullptr;
  int kind = 0;  // 0 = vectors, 1 = windows
  int D = 0;
  int img_w = 0, C = 0, w = 0;
  const int32_t* xs = nullptr;
  const int32_t* ys = nullptr;
  int nx = 1;
};

}  // namespace psg

namespace psg {
enum KernelKind : int {
  K_MIRROR = 0, K_PROJECT, K_SEARCH, K_RESCORE, K_WEIGHTS, K_HIST, K_PENALTY, K_MSTEP, K_STATS,
  K_BUILD, K_PYRAMID, K_SCHED, K_FALLBACK, K_COUNT
};
extern const char* const kKernelNames[K_COUNT];
}  // namespace psg

struct psg_ctx {
  double* deep_key = nullptr;   // frontier scratch of the deep-stack backtrack kernel (lazy)
  int32_t* deep_node = nullptr;
  std::vector<psg_ctx*> builders;  // contexts of psg_synthesize's index build-ahead threads (owned)
  // per-kernel event timing (psg_ctx_profile)
  bool profile = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Pending { int kind; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  double kernel_ms[psg::K_COUNT] = {};
  int64_t kernel_launches[psg::K_COUNT] = {};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t launches = 0;
  int num_sms = 148;
  // cuBLAS / cuSOLVER handles (opaque here, created lazily by pca.cpp)
  void* cublas = nullptr;
  void* cusolver = nullptr;
  // pinned staging: 64-byte slots for per-level stats read-back, carved from
  // pinned blocks that live as long as the context (cudaMallocHost/FreeHost
  // synchronise the device and cost milliseconds: never per level)
  std::vector<void*> pinned_blocks;
  std::vector<double*> pinned_free;
  // side stream for kernels that overlap the critical path (fork / join by events)
  cudaStream_t side = nullptr;
  cudaStream_t copy = nullptr;  // early download of the final image (psg_optimize_level)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_tile = nullptr;
  int* d_flags = nullptr;
  int64_t* d_sched = nullptr;  // [0..1] search tile scheduler, [2] stats fold ticket
  // Scheduling / variant switches, read ONCE from the environment at
  // psg_ctx_create (never inside per-iteration code).  Every variant computes
  // bit-identical results (tests/test_variants.py); the defaults are the
  // measured-fastest choices.
  struct Knobs {
    bool legacy_search = false;       // PERSYN_SEARCH=warp: per-query warp kernel, no tiles
    bool verbose = false;             // PERSYN_VERBOSE: stage / phase timings on stderr
    bool rescore_all = false;         // PERSYN_RESCORE_ALL: rescore every anchor after a search
    bool no_greedy_seed = false;      // PERSYN_NO_GREEDY_SEED: unseeded priming search
    bool no_tile_order = false;       // PERSYN_NO_TILE_ORDER: tiles in index order
    bool no_ex8 = false;              // PERSYN_NO_EX8: unpadded exemplar mirror
    bool penalty_per_anchor = false;  // PERSYN_PENALTY_PER_ANCHOR: no per-candidate table
    bool no_fused_hist = false;       // PERSYN_NO_FUSED_HIST: separate histogram pass
    bool serial = false;              // PERSYN_SERIAL: no side stream
    bool graph = false;               // PERSYN_GRAPH: one CUDA graph per EM iteration
    bool project_kpt2 = false;        // PERSYN_PROJECT_KPT2: 2-per-lane d<=48 projection
    bool no_carry = false;            // PERSYN_NO_CARRY: stages do not seed from the previous
    bool eig_direct = false;          // PERSYN_EIG: dense eigensolver instead of subspace iteration
    bool exact_projection = false;    // PERSYN_EXACT_PROJECTION: fp64 SIMT projection of every query
    bool bt_warp = false;             // PERSYN_BT_WARP: backtrack(m > 2) warp per query (not lane groups)
    bool bt_thread = false;           // PERSYN_BT_THREAD: greedy / backtrack(m <= 2) thread per query
    bool no_build_ahead = false;      // PERSYN_NO_BUILD_AHEAD: synthesize builds each index inline
    bool no_early_download = false;   // PERSYN_NO_EARLY_DOWNLOAD: optimize_level downloads the image at the end
    bool bt_exact_projection = false; // PERSYN_BT_EXACT_PROJECTION: fp64 projection for greedy / backtrack
  } knobs;
};

struct psg_index {
  psg::Index impl;
};

namespace psg {
extern thread_local std::string g_last_error;
void set_last_error(const std::string& m);
// Stream of the C-ABI call in flight (set by StreamScope in every entry point
// that allocates): DBuf allocations are ordered on it.
extern thread_local cudaStream_t t_stream;
// Stream of the API call in flight: per-call buffers come from the device's
// stream-ordered memory pool (cudaMallocAsync), which keeps freed blocks, so
// repeated optimize_level / search_step calls do not pay cudaMalloc.
struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(t_stream) { t_stream = s; }
  ~StreamScope() { t_stream = prev; }
};

// Launches inside the scope go to the context's side stream (the launchers
// use ctx->stream); the caller orders it against the main stream with events.
struct SideScope {
  psg_ctx* ctx;
  cudaStream_t main;
  explicit SideScope(psg_ctx* c) : ctx(c), main(c->stream) { ctx->stream = ctx->side; }
  ~SideScope() { ctx->stream = main; }
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr, o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(s, o.s);
    return *this;
  }
  void alloc(size_t count) {
    release();
    n = count;
    s = t_stream;
    // every C-ABI entry point that allocates sets its context stream
    // (StreamScope): a block freed on the legacy stream could be reused
    // under a kernel still running on the context's non-blocking stream
    if (count && !s) throw Error(PSG_E_LOGIC, "device allocation outside a context stream scope");
    if (count) PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  void upload(psg_ctx* ctx, const T* h, size_t count) {
    if (count) PSG_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->stream));
  }
  void download(psg_ctx* ctx, T* h, size_t count) const {
    if (count) PSG_CUDA(cudaMemcpyAsync(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost, ctx->stream));
  }
};


// ---- row-band helpers shared by runtime.cpp and shard.cpp ------------------------
void band_info(const psg_level* L, psg_band* plan, psg_opt_cfg* cfg, int* C, int* hist_on,
               int* iterations_done);
psg_status band_download_owned(psg_level* L, double* rows);  // [C][p1-p0][W] host
int index_window(const psg_index* ix);
int index_channels(const psg_index* ix);
}  // namespace psg

namespace psg {

// RAII event pair around one kernel launch when profiling is enabled.
struct ProfScope {
  psg_ctx* ctx;
  int kind;
  cudaEvent_t a = nullptr;
  ProfScope(psg_ctx* c, int k);
  ~ProfScope();
};
void prof_flush(psg_ctx* ctx);  // after a stream sync: accumulate elapsed times

// ---- kernel launchers (kernels_*.cu) ------------------------------------------
struct AnchorSet {
  const int32_t* xs;  // device [nx]
  const int32_t* ys;  // device [ny]
  int nx;
  int64_t count;      // nx * ny
};

// planes [C][H][W] fp64 -> mirror [H][W][C] fp32
void launch_make_mirror(psg_ctx* ctx, const double* planes, int C, int W, int H, float* mirror);
void launch_make_mirror8(psg_ctx* ctx, const double* planes, int C, int W, int H, float* out);
// Exact fp64 projection of window features (pca.cpp:27-41).
void launch_project_windows(psg_ctx* ctx, const float* mirror, int img_w, int C, int w,
                            AnchorSet anchors, const double* mean, const double* basis, int d,
                            double* out);
// ---- tensor-core projection (kernels_project_tc.cu) --------------------------------
// Quantised digit mirror of an fp32 mirror: V = rint(v * 2^29) for v in [0, 1]
// as four u8 base-256 digits, 8-byte pixels (channels >= C zero): q8
// [4][H][W][8] bytes.  A value outside [0, 1] (or NaN) sets *bad (the
// projection then reports delta = +inf for every query: exact fallback).
void launch_make_digits(psg_ctx* ctx, const float* mirror, int C, int W, int H, uint8_t* q8,
                        int64_t slice_bytes, int* bad);
// Builds ix.tc_* from the host basis (false: basis not representable, keep the
// exact fp64 projection).
bool tc_prepare(psg_ctx* ctx, Index& ix);
// q^ = B^ v^ - B.mu on the tensor cores (tcgen05.mma kind::i8, exact int32
// accumulation), delta[q] = a rigorous bound on |q^ - q| (2-norm; +inf when a
// window holds a value outside [0, 1]).  out [n][d] fp64.
// stride2: every anchor x is even and consecutive anchors are 2 pixels apart
// (spacing 2, W - w even): the strip-mode kernel applies.
void launch_project_windows_tc(psg_ctx* ctx, const uint8_t* q8, int64_t slice_bytes, int img_w,
                               const int* bad, AnchorSet anchors, bool stride2, const Index& ix,
                               double* out, float* delta, int sp = 0);
// Exact fallback for the ambiguous queries of an approximate search (count
// read on the device): the reference's projection chain of each listed
// window, then either the exact lexicographic min over its two band
// candidates (c1 >= 0: written to idx[], counters += 2) or, when the band
// held more, the projection appended to a re-search list (full_*).
struct ResolveArgs {
  const float* mirror;
  int img_w, C, w;
  AnchorSet anchors;
  const int32_t* list;
  const int* count;
  const int32_t* c0;
  const int32_t* c1;
  int32_t* idx;
  int64_t* scanned;
  int64_t* exact;
  int32_t* full_anchor;
  int32_t* full_seed;
  int* full_count;
  double* full_q;  // [count][d]
};
void launch_resolve(psg_ctx* ctx, const ResolveArgs& r, const Index& ix);
// compact seeds / scatter of a fallback search over listed anchors
void launch_list_gather_i32(psg_ctx* ctx, const int32_t* src, const int32_t* list,
                            const int* count, int32_t* out);
void launch_list_scatter(psg_ctx* ctx, const int32_t* list, const int* count,
                         const int32_t* idx_c, const int64_t* sc_c, const int64_t* ex_c,
                         int32_t* idx, int64_t* scanned, int64_t* exact);
void launch_project_vectors(psg_ctx* ctx, const float* X, int64_t n, int D, const double* mean,
                            const double* basis, int d, double* out);
// Exact NN search over the tree (km_tree.cpp:197-284 semantics).
struct SearchArgs {
  const double* q;      // [nq][d]
  int64_t nq;
  int d;
  const int32_t* seed_idx;  // optional initial candidate per query (upper bound)
  const double* proj;       // [N][d] original order (seed distances)
  const double* proj_soa;   // [d][N] leaf order
  const double* proj_leaf = nullptr;  // [N][d] leaf order
  const double* proj_leaf_il = nullptr;  // pair-interleaved per leaf (lane-group backtrack)
  const float* proj32_q4;   // [dp/4][N] float4 groups, leaf order (fp32 filter)
  const float* pnorm32;     // [N] leaf order
  const float2* pp32 = nullptr;  // [N] leaf order (|p~|^2, |p~_B|^2) (expanded-form filter)
  float pnorm_max;          // max of pnorm32 (rounded up)
  const int32_t* perm;
  int64_t N;
  // coherence seeds (image index only): query anchor lattice + DB lattice
  const int32_t* qxs;       // [qnx] query anchor x positions (null: no neighbour seeds)
  const int32_t* qys;
  int qnx;
  int nxe, nye;             // dense DB anchors per row / column
  DevTree tree;
  int mode, max_leaves;
  int32_t* out_idx;
  double* out_d2;
  int64_t* out_scanned;
  int64_t* out_exact;       // optional: points evaluated in exact fp64
  int32_t* out_visited;     // optional: nodes visited (QueryStats, km_tree.hpp:27-30)
  int* flags;
  int64_t* sched = nullptr;  // [2] tile ticket + warps done (self re-arming, zeroed at ctx creation)
  const int32_t* tile_order = nullptr;  // optional tile permutation (image tiles)
  // approximate queries (tensor-core projection): q holds q^ with |q^ - q|
  // <= qdelta[i]; the search keeps every point within (|q^ - p*| + 2 delta)
  // and lists the queries whose winner is not separated by that band
  const float* qdelta = nullptr;
  int32_t* amb_list = nullptr;  // [nq] ambiguous query ids
  int32_t* amb_c0 = nullptr;    // [nq] their band winner
  int32_t* amb_c1 = nullptr;    // [nq] the only other point in the band, or -1 (re-search)
  int* amb_count = nullptr;     // device counter (zeroed by the caller)
  const int* nq_dev = nullptr;  // optional: query count read on the device
  const int32_t* out_map = nullptr;  // optional (warp kernel): query -> output slot, counters add
  int32_t* ovf_list = nullptr;       // backtrack: queries whose frontier outgrew the pool (re-run)
  int32_t* ovf2_list = nullptr;      // optional: the second (large-pool) pass's overflow list
  int* ovf2_count = nullptr;
  const int32_t* q_list = nullptr;   // lane-group kernel: work item -> query id (a listed pass)
  double* deep_key = nullptr;        // deep-stack kernel: per-warp global frontier scratch
  int32_t* deep_node = nullptr;
  int deep_cap = 0;
  int* ovf_count = nullptr;
};
// Tile permutation for the next exact search of the same anchors: descending
// previous per-tile work (order: [image_tile_count(nq, qnx)]).
int64_t image_tile_count(int64_t nq, int qnx);
void launch_tile_order(psg_ctx* ctx, const int64_t* prev_scanned, int64_t nq, int qnx,
                       int32_t* order);
// Brute-force index: build the filter operand once per index; exact search of
// nq query rows (lexicographic min of (fp64 dist^2, id), optimizer.cpp:175-205).
void brute_prepare(psg_ctx* ctx, Index& ix);
// seed (optional, [nq]): a known candidate per query (e.g. the previous
// assignment) whose exact distance starts the filter's upper bound.
void launch_brute_search(psg_ctx* ctx, const Index& ix, const RowSrc& qsrc, int64_t nq,
                         const int32_t* seed, int32_t* out_idx, double* out_d2,
                         int64_t* out_scanned, int64_t* out_exact);
void launch_search(psg_ctx* ctx, const SearchArgs& a);
// allocates the deep-stack backtrack kernel's global frontier scratch (once per context)
void ensure_deep_scratch(psg_ctx* ctx);
// true when an exact search of this tree runs on the tile kernel
// nq >= 0: an image search of nq anchors (few anchors -> warp-per-query kernel)
bool search_uses_tiles(psg_ctx* ctx, const DevTree& tree, int d, bool exact, int64_t nq = -1);
// true when a backtrack(m) search of this index runs on the lane-group kernel
// (which also takes tensor-core-projected queries with an error band)
bool search_uses_groups(psg_ctx* ctx, const Index& ix, const psg_budget& budget);
// tcgen05 (UMMA) tile search; returns false when the tree shape is unsupported.
// Tile search with the leaf filter on mma.sync (bf16 split); false if unsupported.
// Locality ordering of unstructured queries (search-only workloads).
void launch_greedy_keys(psg_ctx* ctx, const double* q, int64_t nq, int d, const DevTree& tree,
                        uint32_t* keys, int32_t* order);
size_t sort_pairs_temp_bytes(int64_t n);
void sort_pairs_u32(psg_ctx* ctx, const uint32_t* kin, uint32_t* kout, const int32_t* vin,
                    int32_t* vout, int64_t n, void* temp, size_t temp_bytes);
void launch_interleave_blocks(psg_ctx* ctx, const double* rows, const int2* meta, int n_nodes,
                              int d, int dE, bool leaves, int64_t n_rows, double* out);
void launch_gather_rows_f64(psg_ctx* ctx, const double* src, const int32_t* order, int64_t n,
                            int width, double* dst);
void launch_scatter_i32(psg_ctx* ctx, const int32_t* src, const int32_t* order, int64_t n,
                        int32_t* dst);
void launch_scatter_f64(psg_ctx* ctx, const double* src, const int32_t* order, int64_t n,
                        double* dst);
void launch_scatter_i64(psg_ctx* ctx, const int64_t* src, const int32_t* order, int64_t n,
                        int64_t* dst);
void launch_make_fp32_copies(psg_ctx* ctx, const double* soa, int64_t N, int d, int dp,
                             float* aos32, float* pn, float2* pp);
// Full-D distance between query windows and assigned candidates (optimizer.cpp:117-124).
void launch_rescore_windows(psg_ctx* ctx, const float* mirror, int img_w, int C, int w,
                            AnchorSet anchors, const Index& ix, const int32_t* idx, double* dist,
                            const int32_t* prev_idx = nullptr, const double* prev_dist = nullptr,
                            int32_t* list = nullptr, int* count = nullptr);  // [count] scratch (changed-only)
void launch_rescore_query_windows(psg_ctx* ctx, const float* Q, int64_t nq, const Index& ix,
                                  const int32_t* idx, double* dist);
void launch_rescore_vectors(psg_ctx* ctx, const float* Q, int64_t nq, const Index& ix,
                            const int32_t* idx, double* dist);
// M-step pieces.
struct WeightArgs {
  const double* dist;
  const int32_t* idx;
  const double* pen;   // may be null
  int64_t A;
  double r, eps;
  double* irls;        // out
  double* eff;         // out: irls / (1 + pen)
  int* flags;
};
void launch_weights(psg_ctx* ctx, const WeightArgs& a);
void launch_eff_from(psg_ctx* ctx, const double* irls, const double* pen, int64_t A, double* eff,
                     int* flags);
void launch_hist_count(psg_ctx* ctx, const double* planes, int64_t P, int64_t stride, int bins,
                       int slots, unsigned long long* counts);
void launch_hist_fold(psg_ctx* ctx, const unsigned long long* counts, int bins, int slots,
                      int64_t P, const double* ex_mass, double* mass, double* excess);
void launch_penalty(psg_ctx* ctx, const Index& ix, const int32_t* idx, int64_t A,
                    const double* excess, int bins, int slots, double* pen);
// Penalty of every candidate id [0, N) (table), then per-anchor gather + eff.
void launch_penalty_table(psg_ctx* ctx, const Index& ix, const double* excess, int bins,
                          int slots, double* table);
void launch_eff_gather(psg_ctx* ctx, const double* irls, const double* table, const int32_t* idx,
                       int64_t A, double* pen, double* eff, int* flags);
struct MstepArgs {
  const int32_t* xs;
  const int32_t* ys;
  int nx, ny;
  const int32_t* col_lo;  // [W] covering-anchor column range
  const int32_t* col_hi;
  const int32_t* row_lo;  // [H]
  const int32_t* row_hi;
  const int32_t* idx;     // [A]
  const double* eff;      // [A]
  int W, H, C, w;     // H = rows written (a band writes its owned rows only)
  int sp = 0;         // grid spacing (bounds the anchors covering a pixel tile)
  int plane_rows;     // rows allocated per plane (plane stride = W * plane_rows)
  const float* ex_mirror;
  int ew, nxe;
  const float* ex8 = nullptr;  // optional [eh][ew][8] padded candidate pixels
  double* planes;  // out [C][plane_rows][W]
  float* mirror;   // out [H][W][C]
  int* flags;
  // optional: histogram counts of the written pixels (build_histograms of the
  // updated image, fused), u64 [slots][bins], zeroed by the launcher
  unsigned long long* counts = nullptr;
  int bins = 0, slots = 0;
};
void launch_mstep(psg_ctx* ctx, const MstepArgs& a);
// Deterministic reductions for telemetry.
struct StatsArgs {
  const double* cur_dist;   // distances the weights came from
  const double* after_dist; // distances after update (fixed assignment)
  const double* eff;
  const double* next_dist;
  const int32_t* cur_idx;
  const int32_t* next_idx;
  const int64_t* scanned;
  const int32_t* mult;
  int64_t A;
  double r;
  double* out;  // [6]: lsq_before, lsq_after, energy, changed, scanned_plan, unique_scanned
  unsigned long long* ticket = nullptr;  // self re-arming last-block counter (ctx->d_sched + 2)
};
void launch_stats(psg_ctx* ctx, const StatsArgs& a);
// PCA helpers.
void launch_window_mean(psg_ctx* ctx, const float* mirror, int img_w, int C, int w, int nxe,
                        int64_t N, double* mean);
void launch_center_windows(psg_ctx* ctx, const float* mirror, int img_w, int C, int w, int nxe,
                           int64_t N, const double* mean, double* Xc);
// Covariance [D][D] (full, symmetric) of the dense window database of an
// exemplar mirror, from its window means (kernels_pca.cu).
void launch_window_cov(psg_ctx* ctx, const float* ex_mirror, int ew, int eh, int C, int w,
                       const double* wmean, double* cov);
void launch_vector_mean(psg_ctx* ctx, const float* X, int64_t N, int D, double* mean);
void launch_center_vectors(psg_ctx* ctx, const float* X, int64_t N, int D, const double* mean,
                           double* Xc);
void launch_gather_soa(psg_ctx* ctx, const double* proj, int64_t N, int d, const int32_t* perm,
                       double* soa);
// Pyramid helpers.
void launch_downsample(psg_ctx* ctx, const double* in, int W, int H, int f, double* out);
// G guidance ramps [G][H][W] (row ramp on even planes, column ramp on odd ones).
void launch_ramp_planes(psg_ctx* ctx, int G, int W, int H, double* out);
// Synthesize driver: first-search seeds carried from the previous stage.
struct CarryArgs {
  const int32_t* xs;   // new stage: owned anchor columns / rows (device)
  const int32_t* ys;
  int nx;
  int64_t nq;
  int w, nxe, nye;     // new window, exemplar window grid
  const int32_t* pidx; // previous stage: final assignment [pny][pnx]
  const int32_t* pxs;
  const int32_t* pys;
  int pnx, pny, pw, pnxe;
  int scale;           // previous pixel grid -> new (1, or 2^levels)
  int32_t* out;        // [nq]
};
void launch_carry_seed(psg_ctx* ctx, const CarryArgs& a);
void launch_upsample_bilinear(psg_ctx* ctx, const double* in, int W, int H, int f, double* out);
void launch_fit_to(psg_ctx* ctx, const double* in, int W, int H, int ow, int oh, double* out);

// ---- host pieces --------------------------------------------------------------
// KmTree::build replica (tree_kind = PSG_TREE_REFERENCE): the reference's own
// tree, bit for bit (host, the shared sequential engine; tree_host.cpp).
// the walk alone: pre-order child counts and the leaves' id lists in DFS order
void reference_tree_walk(const double* proj, int64_t N, int d, int branching, int leaf_threshold,
                         uint64_t seed, std::vector<int32_t>& n_children,
                         std::vector<int32_t>& leaf_sizes, std::vector<int32_t>& leaf_ids);
HostTree build_reference_tree_host(const double* proj, int64_t N, int d, int branching,
                                   int leaf_threshold, uint64_t seed);
// Same construction on the device (level-synchronous, deterministic); P is
// the device [N][d] projected database.
HostTree build_tree_device(psg_ctx* ctx, const double* P, int64_t N, int d, int branching,
                           int max_depth, int leaf_threshold, uint64_t seed);
// Replay of an external tree (pre-order child counts + DFS leaf lists).
HostTree import_tree_host(const double* proj, int64_t N, int d, const int32_t* n_children_pre,
                          int64_t n_nodes, const int32_t* leaf_sizes, int64_t n_leaves,
                          const int32_t* leaf_ids);
void fit_pca_device(psg_ctx* ctx, Index& ix, const psg_index_cfg& cfg);
// initialize_output (pipeline.cpp:96-175), part1_host.cpp
void initialize_output_host(const double* ex_planes, int C, int ew, int eh,
                            const float* out_scale, int ow, int oh, double s_min, double s_max,
                            uint64_t seed, double* out4);
void create_solver_handles(psg_ctx* ctx);  // cuBLAS + cuSOLVER handles of a context
int64_t plan_host(int W, int H, int w, int sp, int p, int32_t* mult);
std::vector<int32_t> axis_positions(int extent, int window, int step);

// Correctly-rounded (double-double) pow used for the IRLS weight; exposed on
// the host for tests via psg_pow_cr.
double pow_cr_host(double x, double y);

}  // namespace psg
