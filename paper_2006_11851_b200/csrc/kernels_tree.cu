// k-means tree build on the device (KmTree::build, km_tree.cpp:34-195),
// level-synchronous: every node of a tree level is processed by the same
// kernels, points of a node are a contiguous segment of one id permutation.
//
// Per level: node statistics (centroid = mean over ascending ids, radius =
// max distance, 8-dim bounding box) -> for splittable nodes (>= leaf_threshold
// points, below the depth cap, km_tree.cpp:174-184) k = min(b, n) clusters by
// k-means++ (D^2 sampling, km_tree.cpp:40-66) and <= 20 Lloyd sweeps (strict-<
// reassignment, empty clusters keep their centroid, stop when the largest move
// < 1e-6, km_tree.cpp:68-111) -> stable partition of each node's segment by
// cluster, empty clusters dropped (km_tree.cpp:113-117).  Sums run over fixed
// 1024-point chunks combined in chunk order, so the build is deterministic
// (no floating-point atomics).  The random stream is one splitmix64 per node
// (seeded by its breadth-first id) as in the host builder; exact search does
// not depend on the tree (km_tree.cpp:251-278).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "psg_internal.h"

namespace psg {

namespace {

constexpr int kChunk = 1024;
constexpr int kMaxB = 32;

__host__ __device__ inline uint64_t smix_next(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t tree_node_seed(uint64_t seed, int64_t node) {
  uint64_t s = seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(node + 1));
  return smix_next(s);
}

__device__ __forceinline__ double dist2_p(const double* __restrict__ a,
                                          const double* __restrict__ b, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = a[j] - b[j];
    acc += t * t;
  }
  return acc;
}

struct Lv {
  const double* P;
  int d, KB;
  int64_t N;
  const int32_t* ids;
  int L;
  const int64_t* nstart;
  const int32_t* ncount;
  const int32_t* nch0;  // first chunk of each node
  const int32_t* nnch;  // chunks of each node
  int nchunks;
  const int32_t* cnode;
  const int64_t* cbeg;
  const int32_t* clen;
  const int32_t* node_of;  // [N] position -> node
  const int32_t* kk;       // [L] clusters requested (0 = leaf)
};

#define GRID_LOOP(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (int64_t)gridDim.x * blockDim.x)

__global__ void node_of_kernel(Lv v, int32_t* node_of) {
  GRID_LOOP(t, (int64_t)v.nchunks * kChunk) {  // (chunk, offset): one position each
    const int ch = (int)(t / kChunk), i = (int)(t % kChunk);
    if (i < v.clen[ch]) node_of[v.cbeg[ch] + i] = v.cnode[ch];
  }
}

// ---- node statistics ---------------------------------------------------------------
__global__ void stats_part_kernel(Lv v, double* psum, double* pmin, double* pmax) {
  GRID_LOOP(t, (int64_t)v.nchunks * v.d) {
    const int ch = (int)(t / v.d), j = (int)(t - (int64_t)ch * v.d);
    const int64_t b = v.cbeg[ch];
    const int n = v.clen[ch];
    double s = 0.0, mn = 0.0, mx = 0.0;
    for (int i = 0; i < n; ++i) {
      const double x = v.P[(int64_t)v.ids[b + i] * v.d + j];
      s += x;
      if (i == 0 || x < mn) mn = x;
      if (i == 0 || x > mx) mx = x;
    }
    psum[t] = s;
    if (j < v.KB) {
      pmin[(int64_t)ch * kBoxDims + j] = mn;
      pmax[(int64_t)ch * kBoxDims + j] = mx;
    }
  }
}

__global__ void stats_node_kernel(Lv v, const double* psum, const double* pmin,
                                  const double* pmax, double* cent, double* blo, double* bhi) {
  GRID_LOOP(t, (int64_t)v.L * v.d) {
    const int node = (int)(t / v.d), j = (int)(t - (int64_t)node * v.d);
    const int c0 = v.nch0[node], nc = v.nnch[node];
    double s = 0.0, mn = 0.0, mx = 0.0;
    for (int c = 0; c < nc; ++c) {
      s += psum[(int64_t)(c0 + c) * v.d + j];
      if (j < v.KB) {
        const double a = pmin[(int64_t)(c0 + c) * kBoxDims + j];
        const double b = pmax[(int64_t)(c0 + c) * kBoxDims + j];
        if (c == 0 || a < mn) mn = a;
        if (c == 0 || b > mx) mx = b;
      }
    }
    cent[t] = s / (double)v.ncount[node];
    if (j < v.KB) {
      blo[(int64_t)node * kBoxDims + j] = mn;
      bhi[(int64_t)node * kBoxDims + j] = mx;
    }
  }
}

// radius = max sqrt(dist^2) (order-free: max of non-negative doubles = max of
// their bit patterns)
__global__ void radius_kernel(Lv v, const double* cent, unsigned long long* rbits) {
  GRID_LOOP(p, v.N) {
    const int node = v.node_of[p];
    if (node < 0) continue;
    const double r = sqrt(dist2_p(v.P + (int64_t)v.ids[p] * v.d, cent + (int64_t)node * v.d, v.d));
    atomicMax(rbits + node, (unsigned long long)__double_as_longlong(r));
  }
}

// ---- k-means++ ------------------------------------------------------------------------
struct Km {
  double* centers;   // [L][kMaxB][d]
  int32_t* nc;       // [L] centres chosen
  int32_t* picking;  // [L]
  uint64_t* rng;     // [L]
  int32_t* done;     // [L] Lloyd converged
  int32_t* asg;      // [N]
  double* d2;        // [N]
  const int32_t* gid;  // [L] breadth-first node id
  uint64_t seed;
};

__global__ void kpp_first_kernel(Lv v, Km k) {
  GRID_LOOP(node, v.L) {
    k.done[node] = 0;
    k.nc[node] = 0;
    k.picking[node] = 0;
    if (v.kk[node] <= 0) continue;
    uint64_t s = tree_node_seed(k.seed, k.gid[node]);
    const int64_t first = (int64_t)(smix_next(s) % (uint64_t)v.ncount[node]);
    const double* src = v.P + (int64_t)v.ids[v.nstart[node] + first] * v.d;
    for (int j = 0; j < v.d; ++j) k.centers[((int64_t)node * kMaxB) * v.d + j] = src[j];
    k.nc[node] = 1;
    k.picking[node] = v.kk[node] > 1;
    k.rng[node] = s;
  }
}

__global__ void kpp_d2_kernel(Lv v, Km k, int c) {
  GRID_LOOP(p, v.N) {
    const int node = v.node_of[p];
    if (node < 0 || !k.picking[node] || k.nc[node] != c) continue;
    const double dd = dist2_p(v.P + (int64_t)v.ids[p] * v.d,
                              k.centers + ((int64_t)node * kMaxB + c - 1) * v.d, v.d);
    k.d2[p] = c == 1 ? dd : fmin(k.d2[p], dd);
  }
}

__global__ void kpp_part_kernel(Lv v, Km k, int c, double* pd2) {
  GRID_LOOP(ch, v.nchunks) {
    const int node = v.cnode[ch];
    if (!k.picking[node] || k.nc[node] != c) continue;
    double s = 0.0;
    const int64_t b = v.cbeg[ch];
    for (int i = 0; i < v.clen[ch]; ++i) s += k.d2[b + i];
    pd2[ch] = s;
  }
}

// D^2 sampling: r = u * total, first point where the running remainder
// reaches <= 0 (km_tree.cpp:54-63), walked chunk by chunk.  One warp per
// node: lanes load 32 consecutive values (coalesced) and the sequential
// subtraction runs over shuffled registers, in the same order as a serial walk.
__global__ void kpp_pick_kernel(Lv v, Km k, int c, const double* pd2) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t node = wid; node < v.L; node += nw) {
    if (!k.picking[node] || k.nc[node] != c) continue;  // warp-uniform
    const int c0 = v.nch0[node], nch = v.nnch[node];
    double total = 0.0;
    for (int g = 0; g < nch; g += 32) {
      const double x = g + lane < nch ? pd2[c0 + g + lane] : 0.0;
      const int m = min(32, nch - g);
      for (int i = 0; i < m; ++i) total += __shfl_sync(0xffffffffu, x, i);
    }
    if (!(total > 0.0)) {
      if (lane == 0) k.picking[node] = 0;
      continue;
    }
    uint64_t s = k.rng[node];
    double r = (double)(smix_next(s) >> 11) * (1.0 / 9007199254740992.0) * total;
    int64_t chosen = v.nstart[node] + v.ncount[node] - 1;
    // chunk walk: skip whole chunks while the remainder stays positive
    int ch_sel = nch - 1;
    for (int g = 0; g < nch; g += 32) {
      const double x = g + lane < nch ? pd2[c0 + g + lane] : 0.0;
      const int m = min(32, nch - g);
      int hit = -1;
      for (int i = 0; i < m; ++i) {
        const double xi = __shfl_sync(0xffffffffu, x, i);
        if (hit < 0) {
          if (r - xi > 0.0 && g + i + 1 < nch) r -= xi;
          else hit = g + i;
        }
      }
      if (hit >= 0) {
        ch_sel = hit;
        break;
      }
    }
    {
      const int ch = c0 + ch_sel;
      const int64_t b = v.cbeg[ch];
      const int n = v.clen[ch];
      bool found = false;
      for (int g = 0; g < n && !found; g += 32) {
        const double x = g + lane < n ? k.d2[b + g + lane] : 0.0;
        const int m = min(32, n - g);
        for (int i = 0; i < m; ++i) {
          const double xi = __shfl_sync(0xffffffffu, x, i);
          if (!found) {
            r -= xi;
            if (r <= 0.0) {
              chosen = b + g + i;
              found = true;
            }
          }
        }
      }
    }
    if (lane == 0) k.rng[node] = s;
    const double* src = v.P + (int64_t)v.ids[chosen] * v.d;
    for (int j = lane; j < v.d; j += 32) k.centers[((int64_t)node * kMaxB + c) * v.d + j] = src[j];
    if (lane == 0) {
      k.nc[node] = c + 1;
      if (c + 1 >= v.kk[node]) k.picking[node] = 0;
    }
  }
}

// ---- Lloyd ------------------------------------------------------------------------------
// Nearest centre per point (strict <: the lowest centre wins ties,
// km_tree.cpp:76-80).  DP > 0: the point is held in registers (loaded once for
// all centres); DP = 0: generic d.
template <int DP>
__global__ void assign_kernel(Lv v, Km k) {
  GRID_LOOP(p, v.N) {
    const int node = v.node_of[p];
    if (node < 0 || v.kk[node] <= 0 || k.done[node]) continue;
    const double* x = v.P + (int64_t)v.ids[p] * v.d;
    const double* cs = k.centers + (int64_t)node * kMaxB * v.d;
    const int nc = k.nc[node];
    int best = 0;
    double bd = 0.0;
    if (DP > 0) {
      double xr[DP > 0 ? DP : 1];
#pragma unroll
      for (int j = 0; j < DP; ++j) xr[j] = j < v.d ? x[j] : 0.0;
      for (int c = 0; c < nc; ++c) {
        const double* cc = cs + (int64_t)c * v.d;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < DP; ++j)
          if (j < v.d) {
            const double t = xr[j] - cc[j];
            acc += t * t;
          }
        if (c == 0 || acc < bd) {
          bd = acc;
          best = c;
        }
      }
    } else {
      bd = dist2_p(x, cs, v.d);
      for (int c = 1; c < nc; ++c) {
        const double dd = dist2_p(x, cs + (int64_t)c * v.d, v.d);
        if (dd < bd) {
          bd = dd;
          best = c;
        }
      }
    }
    k.asg[p] = best;
  }
}

// Per chunk, the positions of each cluster in chunk order (a stable counting
// sort): the sums below then walk only their own cluster's points.
__global__ void lloyd_sort_kernel(Lv v, Km k, int32_t* sorted, int32_t* pcnt) {
  // one warp per chunk: ballots per cluster over groups of 32 points
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t ch = wid; ch < v.nchunks; ch += nw) {
    const int node = v.cnode[ch];
    if (v.kk[node] <= 0 || k.done[node]) continue;  // warp-uniform
    const int64_t b = v.cbeg[ch];
    const int n = v.clen[ch], nc = k.nc[node];
    // counts
    int my = 0;  // lane c < nc holds cluster c's count
    for (int g = 0; g < n; g += 32) {
      const int a = g + lane < n ? k.asg[b + g + lane] : -1;
      for (int c = 0; c < nc; ++c) {
        const int cnt = __popc(__ballot_sync(0xffffffffu, a == c));
        if (lane == c) my += cnt;
      }
    }
    if (lane < nc) pcnt[(int64_t)ch * kMaxB + lane] = my;
    // exclusive offsets
    int off = 0;
    for (int c = 0; c < nc; ++c) {
      const int cc = __shfl_sync(0xffffffffu, my, c);
      if (lane > c) off += cc;
    }
    // stable scatter: chunk order within each cluster
    for (int g = 0; g < n; g += 32) {
      const int a = g + lane < n ? k.asg[b + g + lane] : -1;
      for (int c = 0; c < nc; ++c) {
        const unsigned m = __ballot_sync(0xffffffffu, a == c);
        const int base = __shfl_sync(0xffffffffu, off, c);
        if (a == c) sorted[b + base + __popc(m & lt)] = (int32_t)(g + lane);
        if (lane == c) off += __popc(m);
      }
    }
  }
}

__global__ void lloyd_part_kernel(Lv v, Km k, const int32_t* sorted, const int32_t* pcnt,
                                  double* psc) {
  GRID_LOOP(t, (int64_t)v.nchunks * kMaxB * v.d) {
    const int j = (int)(t % v.d);
    const int64_t cc = t / v.d;
    const int c = (int)(cc % kMaxB);
    const int ch = (int)(cc / kMaxB);
    const int node = v.cnode[ch];
    if (v.kk[node] <= 0 || k.done[node] || c >= k.nc[node]) continue;
    const int64_t b = v.cbeg[ch];
    int first = 0;
    for (int o = 0; o < c; ++o) first += pcnt[(int64_t)ch * kMaxB + o];
    const int n = pcnt[cc];
    double s = 0.0;
#pragma unroll 4
    for (int i = 0; i < n; ++i)  // chunk order within the cluster
      s += v.P[(int64_t)v.ids[b + sorted[b + first + i]] * v.d + j];
    psc[t] = s;
  }
}

__global__ void lloyd_update_kernel(Lv v, Km k, const double* psc, const int32_t* pcnt,
                                    double* mv2) {
  GRID_LOOP(t, (int64_t)v.L * kMaxB * v.d) {
    const int j = (int)(t % v.d);
    const int64_t nc_ = t / v.d;
    const int node = (int)(nc_ / kMaxB), c = (int)(nc_ % kMaxB);
    mv2[t] = 0.0;
    if (v.kk[node] <= 0 || k.done[node] || c >= k.nc[node]) continue;
    const int c0 = v.nch0[node], nch = v.nnch[node];
    int64_t n = 0;
    for (int i = 0; i < nch; ++i) n += pcnt[(int64_t)(c0 + i) * kMaxB + c];
    if (n == 0) continue;  // empty cluster keeps its centroid (km_tree.cpp:95-96)
    double s = 0.0;
    for (int i = 0; i < nch; ++i) s += psc[(((int64_t)(c0 + i) * kMaxB) + c) * v.d + j];
    const double nv = s / (double)n;
    double* ctr = k.centers + ((int64_t)node * kMaxB + c) * v.d;
    const double dd = nv - ctr[j];
    mv2[t] = dd * dd;
    ctr[j] = nv;
  }
}

__global__ void lloyd_conv_kernel(Lv v, Km k, const double* mv2, int* active) {
  GRID_LOOP(node, v.L) {
    if (v.kk[node] <= 0 || k.done[node]) continue;
    double m = 0.0;
    for (int c = 0; c < k.nc[node]; ++c) {
      double m2 = 0.0;  // squared move of centre c, dims in order
      for (int j = 0; j < v.d; ++j) m2 += mv2[((int64_t)node * kMaxB + c) * v.d + j];
      m = fmax(m, sqrt(m2));
    }
    if (m < 1e-6) k.done[node] = 1;  // km_tree.cpp:109
    else atomicAdd(active, 1);
  }
}

// ---- stable partition of each split node's segment by cluster -------------------------
__global__ void part_count_kernel(Lv v, Km k, int32_t* pc) {
  GRID_LOOP(t, (int64_t)v.nchunks * kMaxB) {
    const int ch = (int)(t / kMaxB), c = (int)(t % kMaxB);
    const int node = v.cnode[ch];
    if (v.kk[node] <= 0) continue;
    const int64_t b = v.cbeg[ch];
    int cnt = 0;
    for (int i = 0; i < v.clen[ch]; ++i) cnt += k.asg[b + i] == c;
    pc[t] = cnt;
  }
}

__global__ void part_offsets_kernel(Lv v, Km k, const int32_t* pc, int64_t* off, int32_t* tot) {
  GRID_LOOP(node, v.L) {
    if (v.kk[node] <= 0) continue;
    const int c0 = v.nch0[node], nch = v.nnch[node];
    int64_t o = v.nstart[node];
    for (int c = 0; c < kMaxB; ++c) {
      int64_t t = 0;
      for (int i = 0; i < nch; ++i) {
        off[(int64_t)(c0 + i) * kMaxB + c] = o + t;
        t += c < k.nc[node] ? pc[(int64_t)(c0 + i) * kMaxB + c] : 0;
      }
      tot[(int64_t)node * kMaxB + c] = (int32_t)t;
      o += t;
    }
  }
}

__global__ void part_scatter_kernel(Lv v, Km k, const int64_t* off, int32_t* ids_next) {
  GRID_LOOP(t, (int64_t)v.nchunks * kMaxB) {
    const int ch = (int)(t / kMaxB), c = (int)(t % kMaxB);
    const int node = v.cnode[ch];
    if (v.kk[node] <= 0 || c >= k.nc[node]) continue;
    int64_t o = off[t];
    const int64_t b = v.cbeg[ch];
    for (int i = 0; i < v.clen[ch]; ++i)
      if (k.asg[b + i] == c) ids_next[o++] = v.ids[b + i];
  }
}

struct DevArr {
  void* p = nullptr;
  cudaStream_t s;
  DevArr(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) PSG_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  ~DevArr() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

template <class T>
void up(psg_ctx* ctx, T* dst, const std::vector<T>& v) {
  if (!v.empty())
    PSG_CUDA(cudaMemcpyAsync(dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice,
                             ctx->stream));
}
template <class T>
void down(psg_ctx* ctx, std::vector<T>& v, const T* src, size_t n) {
  v.resize(n);
  if (n)
    PSG_CUDA(cudaMemcpyAsync(v.data(), src, sizeof(T) * n, cudaMemcpyDeviceToHost, ctx->stream));
}

int grid_for(psg_ctx* ctx, int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)ctx->num_sms * 32;
  if (b > cap) b = cap;
  return (int)std::max<int64_t>(b, 1);
}

void launch_assign(psg_ctx* ctx, const Lv& v, const Km& k, int64_t N) {
  const int g = grid_for(ctx, N, 256);
  if (v.d <= 32)
    assign_kernel<32><<<g, 256, 0, ctx->stream>>>(v, k);
  else if (v.d <= 64)
    assign_kernel<64><<<g, 256, 0, ctx->stream>>>(v, k);
  else
    assign_kernel<0><<<g, 256, 0, ctx->stream>>>(v, k);
}

}  // namespace

HostTree build_tree_device(psg_ctx* ctx, const double* P, int64_t N, int d, int branching,
                           int max_depth, int leaf_threshold, uint64_t seed) {
  ProfScope _prof(ctx, K_BUILD);
  if (N < 1) fail(PSG_E_DOMAIN, "cannot build a tree over zero points");
  if (branching < 2) fail(PSG_E_DOMAIN, "tree branching must be >= 2");
  if (branching > kMaxB) fail(PSG_E_DOMAIN, "tree branching > 32 is not supported");
  if (leaf_threshold <= 0) leaf_threshold = branching;
  cudaStream_t st = ctx->stream;
  if (d <= 0) {  // nothing to cluster on: one leaf (km_tree.cpp:174)
    HostTree t;
    t.radius.push_back(0.0);
    t.boxlo.assign(kBoxDims, 0.0);
    t.boxhi.assign(kBoxDims, 0.0);
    t.first_child.push_back(-1);
    t.n_children.push_back(0);
    t.leaf_start.push_back(0);
    t.leaf_count.push_back((int32_t)N);
    t.depth.push_back(0);
    t.n_leaves = 1;
    t.perm.resize((size_t)N);
    for (int64_t i = 0; i < N; ++i) t.perm[i] = (int32_t)i;
    return t;
  }
  const int dd = d;
  const int KB = std::min(d, kBoxDims);
  HostTree t;
  t.perm.resize((size_t)N);

  DevArr ids_a(sizeof(int32_t) * N, st), ids_b(sizeof(int32_t) * N, st);
  DevArr node_of(sizeof(int32_t) * N, st), asg(sizeof(int32_t) * N, st), d2(sizeof(double) * N, st);
  {
    std::vector<int32_t> iota((size_t)N);
    for (int64_t i = 0; i < N; ++i) iota[i] = (int32_t)i;
    up(ctx, ids_a.as<int32_t>(), iota);
  }
  int32_t* ids = ids_a.as<int32_t>();
  int32_t* ids_next = ids_b.as<int32_t>();

  struct HNode {
    int64_t start;
    int32_t count;
    int depth;
  };
  std::vector<HNode> level{{0, (int32_t)N, 0}};

  while (!level.empty()) {
    const int L = (int)level.size();
    const int64_t base = (int64_t)t.radius.size();
    // chunk table
    std::vector<int64_t> nstart(L), cbeg;
    std::vector<int32_t> ncount(L), nch0(L), nnch(L), cnode, clen, kk(L), gid(L);
    for (int i = 0; i < L; ++i) {
      nstart[i] = level[i].start;
      ncount[i] = level[i].count;
      nch0[i] = (int32_t)cnode.size();
      for (int64_t b = 0; b < level[i].count; b += kChunk) {
        cnode.push_back(i);
        cbeg.push_back(level[i].start + b);
        clen.push_back((int32_t)std::min<int64_t>(kChunk, level[i].count - b));
      }
      nnch[i] = (int32_t)cnode.size() - nch0[i];
      const bool can = level[i].count >= leaf_threshold && d > 0 &&
                       (max_depth <= 0 || level[i].depth < max_depth);
      kk[i] = can ? std::min(branching, level[i].count) : 0;
      gid[i] = (int32_t)(base + i);
    }
    const int nchunks = (int)cnode.size();
    DevArr d_nstart(sizeof(int64_t) * L, st), d_ncount(sizeof(int32_t) * L, st);
    DevArr d_nch0(sizeof(int32_t) * L, st), d_nnch(sizeof(int32_t) * L, st);
    DevArr d_kk(sizeof(int32_t) * L, st), d_gid(sizeof(int32_t) * L, st);
    DevArr d_cnode(sizeof(int32_t) * nchunks, st), d_cbeg(sizeof(int64_t) * nchunks, st);
    DevArr d_clen(sizeof(int32_t) * nchunks, st);
    up(ctx, d_nstart.as<int64_t>(), nstart);
    up(ctx, d_ncount.as<int32_t>(), ncount);
    up(ctx, d_nch0.as<int32_t>(), nch0);
    up(ctx, d_nnch.as<int32_t>(), nnch);
    up(ctx, d_kk.as<int32_t>(), kk);
    up(ctx, d_gid.as<int32_t>(), gid);
    up(ctx, d_cnode.as<int32_t>(), cnode);
    up(ctx, d_cbeg.as<int64_t>(), cbeg);
    up(ctx, d_clen.as<int32_t>(), clen);

    Lv v{};
    v.P = P;
    v.d = dd;
    v.KB = KB;
    v.N = N;
    v.ids = ids;
    v.L = L;
    v.nstart = d_nstart.as<int64_t>();
    v.ncount = d_ncount.as<int32_t>();
    v.nch0 = d_nch0.as<int32_t>();
    v.nnch = d_nnch.as<int32_t>();
    v.nchunks = nchunks;
    v.cnode = d_cnode.as<int32_t>();
    v.cbeg = d_cbeg.as<int64_t>();
    v.clen = d_clen.as<int32_t>();
    v.node_of = node_of.as<int32_t>();
    v.kk = d_kk.as<int32_t>();

    // positions of earlier leaves belong to no node of this level (-1)
    PSG_CUDA(cudaMemsetAsync(node_of.p, 0xFF, sizeof(int32_t) * N, st));
    node_of_kernel<<<grid_for(ctx, (int64_t)nchunks * kChunk, 256), 256, 0, st>>>(
        v, node_of.as<int32_t>());
    PSG_LAUNCHED(ctx);
    // ---- statistics ----
    DevArr psum(sizeof(double) * (size_t)nchunks * dd, st);
    DevArr pmin(sizeof(double) * (size_t)nchunks * kBoxDims, st);
    DevArr pmax(sizeof(double) * (size_t)nchunks * kBoxDims, st);
    DevArr cent(sizeof(double) * (size_t)L * dd, st);
    DevArr blo(sizeof(double) * (size_t)L * kBoxDims, st), bhi(sizeof(double) * (size_t)L * kBoxDims, st);
    DevArr rbits(sizeof(unsigned long long) * L, st);
    PSG_CUDA(cudaMemsetAsync(blo.p, 0, sizeof(double) * (size_t)L * kBoxDims, st));
    PSG_CUDA(cudaMemsetAsync(bhi.p, 0, sizeof(double) * (size_t)L * kBoxDims, st));
    PSG_CUDA(cudaMemsetAsync(rbits.p, 0, sizeof(unsigned long long) * L, st));
    stats_part_kernel<<<grid_for(ctx, (int64_t)nchunks * dd, 128), 128, 0, st>>>(
        v, psum.as<double>(), pmin.as<double>(), pmax.as<double>());
    PSG_LAUNCHED(ctx);
    stats_node_kernel<<<grid_for(ctx, (int64_t)L * dd, 128), 128, 0, st>>>(
        v, psum.as<double>(), pmin.as<double>(), pmax.as<double>(), cent.as<double>(),
        blo.as<double>(), bhi.as<double>());
    PSG_LAUNCHED(ctx);
    radius_kernel<<<grid_for(ctx, N, 256), 256, 0, st>>>(v, cent.as<double>(),
                                                         rbits.as<unsigned long long>());
    PSG_LAUNCHED(ctx);

    // ---- clustering of the splittable nodes ----
    const bool any_split = std::any_of(kk.begin(), kk.end(), [](int k) { return k > 0; });
    std::vector<int32_t> tot;
    if (any_split) {
      DevArr centers(sizeof(double) * (size_t)L * kMaxB * dd, st);
      DevArr nc(sizeof(int32_t) * L, st), picking(sizeof(int32_t) * L, st);
      DevArr rng(sizeof(uint64_t) * L, st), done(sizeof(int32_t) * L, st);
      DevArr pd2(sizeof(double) * nchunks, st);
      Km k{};
      k.centers = centers.as<double>();
      k.nc = nc.as<int32_t>();
      k.picking = picking.as<int32_t>();
      k.rng = rng.as<uint64_t>();
      k.done = done.as<int32_t>();
      k.asg = asg.as<int32_t>();
      k.d2 = d2.as<double>();
      k.gid = d_gid.as<int32_t>();
      k.seed = seed;
      const int kmax = *std::max_element(kk.begin(), kk.end());
      kpp_first_kernel<<<grid_for(ctx, L, 128), 128, 0, st>>>(v, k);
      PSG_LAUNCHED(ctx);
      for (int c = 1; c < kmax; ++c) {
        kpp_d2_kernel<<<grid_for(ctx, N, 256), 256, 0, st>>>(v, k, c);
        PSG_LAUNCHED(ctx);
        kpp_part_kernel<<<grid_for(ctx, nchunks, 128), 128, 0, st>>>(v, k, c, pd2.as<double>());
        PSG_LAUNCHED(ctx);
        kpp_pick_kernel<<<grid_for(ctx, (int64_t)L * 32, 128), 128, 0, st>>>(v, k, c,
                                                                          pd2.as<double>());
        PSG_LAUNCHED(ctx);
      }
      DevArr psc(sizeof(double) * (size_t)nchunks * kMaxB * dd, st);
      DevArr pcnt(sizeof(int32_t) * (size_t)nchunks * kMaxB, st);
      DevArr mv2(sizeof(double) * (size_t)L * kMaxB * dd, st);
      DevArr sorted(sizeof(int32_t) * (size_t)N, st);
      DevArr active(sizeof(int), st);
      launch_assign(ctx, v, k, N);
      PSG_LAUNCHED(ctx);
      for (int sweep = 0; sweep < 20; ++sweep) {  // km_tree.cpp:86-111
        lloyd_sort_kernel<<<grid_for(ctx, (int64_t)nchunks * 32, 128), 128, 0, st>>>(
            v, k, sorted.as<int32_t>(), pcnt.as<int32_t>());
        PSG_LAUNCHED(ctx);
        lloyd_part_kernel<<<grid_for(ctx, (int64_t)nchunks * kMaxB * dd, 128), 128, 0, st>>>(
            v, k, sorted.as<int32_t>(), pcnt.as<int32_t>(), psc.as<double>());
        PSG_LAUNCHED(ctx);
        lloyd_update_kernel<<<grid_for(ctx, (int64_t)L * kMaxB * dd, 128), 128, 0, st>>>(
            v, k, psc.as<double>(), pcnt.as<int32_t>(), mv2.as<double>());
        PSG_LAUNCHED(ctx);
        PSG_CUDA(cudaMemsetAsync(active.p, 0, sizeof(int), st));
        lloyd_conv_kernel<<<grid_for(ctx, L, 128), 128, 0, st>>>(v, k, mv2.as<double>(),
                                                                 active.as<int>());
        PSG_LAUNCHED(ctx);
        launch_assign(ctx, v, k, N);
        PSG_LAUNCHED(ctx);
        if (sweep % 4 == 3) {
          int h = 0;
          PSG_CUDA(cudaMemcpyAsync(&h, active.p, sizeof(int), cudaMemcpyDeviceToHost, st));
          PSG_CUDA(cudaStreamSynchronize(st));
          if (h == 0) break;
        }
      }
      DevArr pc(sizeof(int32_t) * (size_t)nchunks * kMaxB, st);
      DevArr off(sizeof(int64_t) * (size_t)nchunks * kMaxB, st);
      DevArr dtot(sizeof(int32_t) * (size_t)L * kMaxB, st);
      part_count_kernel<<<grid_for(ctx, (int64_t)nchunks * kMaxB, 128), 128, 0, st>>>(
          v, k, pc.as<int32_t>());
      PSG_LAUNCHED(ctx);
      part_offsets_kernel<<<grid_for(ctx, L, 128), 128, 0, st>>>(v, k, pc.as<int32_t>(),
                                                                 off.as<int64_t>(),
                                                                 dtot.as<int32_t>());
      PSG_LAUNCHED(ctx);
      PSG_CUDA(cudaMemcpyAsync(ids_next, ids, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st));
      part_scatter_kernel<<<grid_for(ctx, (int64_t)nchunks * kMaxB, 128), 128, 0, st>>>(
          v, k, off.as<int64_t>(), ids_next);
      PSG_LAUNCHED(ctx);
      down(ctx, tot, dtot.as<int32_t>(), (size_t)L * kMaxB);
    }
    std::vector<double> hc, hlo, hhi;
    std::vector<unsigned long long> hr;
    down(ctx, hc, cent.as<double>(), (size_t)L * dd);
    down(ctx, hlo, blo.as<double>(), (size_t)L * kBoxDims);
    down(ctx, hhi, bhi.as<double>(), (size_t)L * kBoxDims);
    down(ctx, hr, rbits.as<unsigned long long>(), (size_t)L);
    PSG_CUDA(cudaStreamSynchronize(st));
    if (any_split) std::swap(ids, ids_next);

    // ---- emit this level; children (non-empty clusters, in order) form the next ----
    std::vector<HNode> next;
    const int64_t first_next = base + L;
    for (int i = 0; i < L; ++i) {
      if (d > 0) t.centroid.insert(t.centroid.end(), hc.begin() + (size_t)i * dd,
                                   hc.begin() + (size_t)(i + 1) * dd);
      double r;
      std::memcpy(&r, &hr[i], sizeof(double));
      t.radius.push_back(r);
      t.boxlo.insert(t.boxlo.end(), hlo.begin() + (size_t)i * kBoxDims, hlo.begin() + (size_t)(i + 1) * kBoxDims);
      t.boxhi.insert(t.boxhi.end(), hhi.begin() + (size_t)i * kBoxDims, hhi.begin() + (size_t)(i + 1) * kBoxDims);
      t.depth.push_back(level[i].depth);
      t.max_depth = std::max(t.max_depth, level[i].depth);
      int nonempty = 0;
      if (kk[i] > 0)
        for (int c = 0; c < kMaxB; ++c) nonempty += tot[(size_t)i * kMaxB + c] > 0;
      if (nonempty >= 2) {  // km_tree.cpp:181-184
        t.first_child.push_back((int32_t)(first_next + next.size()));
        t.n_children.push_back(nonempty);
        t.leaf_start.push_back(0);
        t.leaf_count.push_back(0);
        int64_t s = level[i].start;
        for (int c = 0; c < kMaxB; ++c) {
          const int32_t n = tot[(size_t)i * kMaxB + c];
          if (n > 0) next.push_back(HNode{s, n, level[i].depth + 1});
          s += n;
        }
      } else {
        t.first_child.push_back(-1);
        t.n_children.push_back(0);
        t.leaf_start.push_back((int32_t)level[i].start);
        t.leaf_count.push_back(level[i].count);
        t.n_leaves++;
      }
    }
    level = std::move(next);
  }
  // leaves keep their segments once emitted: the final permutation is the leaf order
  std::vector<int32_t> perm;
  down(ctx, perm, ids, (size_t)N);
  PSG_CUDA(cudaStreamSynchronize(st));
  t.perm = std::move(perm);
  return t;
}

}  // namespace psg
