// k-means tree build (native host runtime, per stage).
//
// Same construction as KmTree::build (km_tree.cpp:141-195): node centroid =
// mean of its points in ascending id order, radius = max distance; a node is
// split with k = min(b, n) k-means++/Lloyd clusters (km_tree.cpp:34-119:
// <= 20 sweeps, stop when the largest centroid move < 1e-6, strict-< reassign,
// empty clusters dropped) when it holds >= leaf_threshold points, is above
// the depth cap (the BASELINE configs' "depth"), and the split yields >= 2
// clusters.  Differences from the reference, none of which changes an exact
// query result (exact search is tree-independent, km_tree.cpp:251-278):
//   * breadth-first node ids with contiguous children (GPU-friendly);
//   * one splitmix64 stream per node instead of one shared mt19937_64 in DFS
//     order, so nodes build in parallel and deterministically;
//   * optional depth cap;
//   * Lloyd sums are accumulated per fixed 4096-point chunk and combined in
//     chunk order, so a large node is clustered by all host threads with a
//     result independent of the thread count.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "psg_internal.h"

namespace psg {
namespace {

// Minimal persistent pool: run(n, fn) calls fn(i) for i in [0, n) on all
// workers (the caller participates) and returns when every index is done.
class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  int size() const { return (int)workers_.size() + 1; }
  void run(int64_t n, const std::function<void(int64_t)>& fn) {
    if (n <= 0) return;
    if (workers_.empty() || n == 1) {
      for (int64_t i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(m_);
    cv_done_.wait(lk, [&] { return done_ == (int)workers_.size(); });
    fn_ = nullptr;
  }

 private:
  Pool() {
    unsigned hw = std::thread::hardware_concurrency();
    if (hw == 0) hw = 1;
    for (unsigned i = 1; i < hw && i < 64; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void work() {
    for (;;) {
      const int64_t i = next_.fetch_add(1);
      if (i >= n_) break;
      (*fn_)(i);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
      {
        std::lock_guard<std::mutex> g(m_);
        ++done_;
      }
      cv_done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, cv_done_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  std::atomic<int64_t> next_{0};
  int64_t n_ = 0;
  int done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

constexpr int64_t kChunk = 4096;

struct SplitMix {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform01() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
};

inline double dist2(const double* a, const double* b, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = a[j] - b[j];
    acc += t * t;
  }
  return acc;
}

// dist2(p, centers[c0 + i]) for i < m <= 8, each accumulated in j order
// exactly like dist2(); the m independent chains hide the add latency.
inline void dist2_block(const double* p, const double* centers, int c0, int m, int d,
                        double* out) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const double* c = centers + (size_t)c0 * d;
  if (m == 8) {
    for (int j = 0; j < d; ++j) {
      const double pj = p[j];
#pragma GCC unroll 8
      for (int i = 0; i < 8; ++i) {
        const double t = pj - c[(size_t)i * d + j];
        acc[i] += t * t;
      }
    }
  } else {
    for (int j = 0; j < d; ++j) {
      const double pj = p[j];
      for (int i = 0; i < m; ++i) {
        const double t = pj - c[(size_t)i * d + j];
        acc[i] += t * t;
      }
    }
  }
  for (int i = 0; i < m; ++i) out[i] = acc[i];
}

// dist2(P[ids[i]], c) for 4 consecutive ids at once (independent chains).
inline void dist2_points4(const double* P, const int32_t* ids, const double* c, int d,
                          double* out) {
  const double* a0 = P + (size_t)ids[0] * d;
  const double* a1 = P + (size_t)ids[1] * d;
  const double* a2 = P + (size_t)ids[2] * d;
  const double* a3 = P + (size_t)ids[3] * d;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int j = 0; j < d; ++j) {
    const double cj = c[j];
    const double t0 = a0[j] - cj, t1 = a1[j] - cj, t2 = a2[j] - cj, t3 = a3[j] - cj;
    s0 += t0 * t0;
    s1 += t1 * t1;
    s2 += t2 * t2;
    s3 += t3 * t3;
  }
  out[0] = s0;
  out[1] = s1;
  out[2] = s2;
  out[3] = s3;
}

struct Job {
  std::vector<int32_t> ids;
  int depth;
};

// fn(chunk, lo, hi) over [0, n) in fixed kChunk pieces, in parallel when
// `parallel` (chunk boundaries do not depend on the thread count).
void for_chunks(int64_t n, bool parallel,
                const std::function<void(int64_t, int64_t, int64_t)>& fn) {
  const int64_t nch = (n + kChunk - 1) / kChunk;
  auto body = [&](int64_t c) { fn(c, c * kChunk, std::min(n, (c + 1) * kChunk)); };
  if (parallel && nch > 1) {
    Pool::get().run(nch, body);
  } else {
    for (int64_t c = 0; c < nch; ++c) body(c);
  }
}

// k-means++ + Lloyd over ids (ascending); returns non-empty clusters with
// ascending ids.
std::vector<std::vector<int32_t>> cluster(const double* P, int d, const std::vector<int32_t>& ids,
                                          int k, uint64_t seed, bool parallel) {
  const int64_t n = (int64_t)ids.size();
  const int64_t nch = (n + kChunk - 1) / kChunk;
  SplitMix rng{seed};
  std::vector<double> centers;
  centers.reserve((size_t)k * d);
  const size_t first = rng.next() % n;
  centers.insert(centers.end(), P + (size_t)ids[first] * d, P + (size_t)ids[first] * d + d);
  std::vector<double> d2(n);
  for_chunks(n, parallel, [&](int64_t, int64_t lo, int64_t hi) {
    int64_t i = lo;
    for (; i + 4 <= hi; i += 4) dist2_points4(P, ids.data() + i, centers.data(), d, &d2[i]);
    for (; i < hi; ++i) d2[i] = dist2(P + (size_t)ids[i] * d, centers.data(), d);
  });
  int nc = 1;
  while (nc < k) {
    double total = 0.0;
    for (double v : d2) total += v;
    if (total <= 0.0) break;
    double r = rng.uniform01() * total;
    int64_t chosen = n - 1;
    for (int64_t i = 0; i < n; ++i) {
      r -= d2[i];
      if (r <= 0.0) {
        chosen = i;
        break;
      }
    }
    const double* c = P + (size_t)ids[chosen] * d;
    centers.insert(centers.end(), c, c + d);
    ++nc;
    for_chunks(n, parallel, [&](int64_t, int64_t lo, int64_t hi) {
      int64_t i = lo;
      double t[4];
      for (; i + 4 <= hi; i += 4) {
        dist2_points4(P, ids.data() + i, c, d, t);
        for (int q = 0; q < 4; ++q) d2[i + q] = std::min(d2[i + q], t[q]);
      }
      for (; i < hi; ++i) d2[i] = std::min(d2[i], dist2(P + (size_t)ids[i] * d, c, d));
    });
  }
  std::vector<int> assign(n);
  auto reassign = [&] {
    for_chunks(n, parallel, [&](int64_t, int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        const double* p = P + (size_t)ids[i] * d;
        int best = 0;
        double bd = 0.0;
        double dd[8];
        for (int c0 = 0; c0 < nc; c0 += 8) {
          const int m = std::min(8, nc - c0);
          dist2_block(p, centers.data(), c0, m, d, dd);
          for (int q = 0; q < m; ++q) {
            if (c0 + q == 0) {
              bd = dd[0];
            } else if (dd[q] < bd) {  // strict <: lowest cluster on ties
              bd = dd[q];
              best = c0 + q;
            }
          }
        }
        assign[i] = best;
      }
    });
  };
  reassign();
  std::vector<double> sums((size_t)nc * d), csum((size_t)nch * nc * d);
  std::vector<int64_t> sizes(nc), csz((size_t)nch * nc);
  for (int sweep = 0; sweep < 20; ++sweep) {
    for_chunks(n, parallel, [&](int64_t ch, int64_t lo, int64_t hi) {
      double* s = csum.data() + (size_t)ch * nc * d;
      int64_t* z = csz.data() + (size_t)ch * nc;
      std::fill(s, s + (size_t)nc * d, 0.0);
      std::fill(z, z + nc, 0);
      for (int64_t i = lo; i < hi; ++i) {
        const double* p = P + (size_t)ids[i] * d;
        double* sc = s + (size_t)assign[i] * d;
        for (int j = 0; j < d; ++j) sc[j] += p[j];
        ++z[assign[i]];
      }
    });
    std::fill(sums.begin(), sums.end(), 0.0);
    std::fill(sizes.begin(), sizes.end(), 0);
    for (int64_t ch = 0; ch < nch; ++ch)  // fixed chunk order: deterministic
      for (int c = 0; c < nc; ++c) {
        sizes[c] += csz[(size_t)ch * nc + c];
        for (int j = 0; j < d; ++j)
          sums[(size_t)c * d + j] += csum[((size_t)ch * nc + c) * d + j];
      }
    double movement = 0.0;
    for (int c = 0; c < nc; ++c) {
      if (sizes[c] == 0) continue;
      double move = 0.0;
      for (int j = 0; j < d; ++j) {
        const double v = sums[(size_t)c * d + j] / (double)sizes[c];
        const double t = v - centers[(size_t)c * d + j];
        move += t * t;
        centers[(size_t)c * d + j] = v;
      }
      movement = std::max(movement, std::sqrt(move));
    }
    if (movement < 1e-6) break;
    reassign();
  }
  std::vector<std::vector<int32_t>> clusters(nc);
  for (int64_t i = 0; i < n; ++i) clusters[assign[i]].push_back(ids[i]);
  clusters.erase(std::remove_if(clusters.begin(), clusters.end(),
                                [](const std::vector<int32_t>& c) { return c.empty(); }),
                 clusters.end());
  return clusters;
}

uint64_t node_seed(uint64_t seed, int64_t node) {
  SplitMix s{seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(node + 1))};
  return s.next();
}

}  // namespace

HostTree build_tree_host(const double* P, int64_t N, int d, int branching, int max_depth,
                         int leaf_threshold, uint64_t seed) {
  if (N < 1) fail(PSG_E_DOMAIN, "cannot build a tree over zero points");
  if (branching < 2) fail(PSG_E_DOMAIN, "tree branching must be >= 2");
  if (leaf_threshold <= 0) leaf_threshold = branching;
  HostTree t;
  std::vector<Job> level(1);
  level[0].ids.resize(N);
  for (int64_t i = 0; i < N; ++i) level[0].ids[i] = (int32_t)i;
  level[0].depth = 0;
  int32_t leaf_cursor = 0;
  t.perm.reserve(N);
  const int threads = Pool::get().size();

  while (!level.empty()) {
    const size_t base = t.radius.size();
    const size_t L = level.size();
    std::vector<std::vector<std::vector<int32_t>>> splits(L);
    std::vector<double> cent(L * (size_t)d), rad(L);
    const int KB = std::min(d, kBoxDims);
    std::vector<double> blo(L * kBoxDims, 0.0), bhi(L * kBoxDims, 0.0);
    // few big nodes: parallel inside each node; many nodes: one node per task
    const bool inner = (int64_t)L < threads;
    auto work = [&](size_t i) {
      const auto& ids = level[i].ids;
      double* c = cent.data() + i * d;
      for (int j = 0; j < d; ++j) c[j] = 0.0;
      for (int32_t id : ids)
        for (int j = 0; j < d; ++j) c[j] += P[(size_t)id * d + j];
      for (int j = 0; j < d; ++j) c[j] /= (double)ids.size();
      double r = 0.0;
      for (int32_t id : ids) r = std::max(r, std::sqrt(dist2(P + (size_t)id * d, c, d)));
      rad[i] = r;
      for (int j = 0; j < KB; ++j) {
        double mn = P[(size_t)ids[0] * d + j], mx = mn;
        for (int32_t id : ids) {
          mn = std::min(mn, P[(size_t)id * d + j]);
          mx = std::max(mx, P[(size_t)id * d + j]);
        }
        blo[i * kBoxDims + j] = mn;
        bhi[i * kBoxDims + j] = mx;
      }
      const bool can = (int64_t)ids.size() >= leaf_threshold && d > 0 &&
                       (max_depth <= 0 || level[i].depth < max_depth);
      if (can) {
        const int k = (int)std::min<size_t>((size_t)branching, ids.size());
        auto cl = cluster(P, d, ids, k, node_seed(seed, (int64_t)(base + i)), inner);
        if (cl.size() >= 2) splits[i] = std::move(cl);
      }
    };
    if (inner) {
      for (size_t i = 0; i < L; ++i) work(i);
    } else {
      Pool::get().run((int64_t)L, [&](int64_t i) { work((size_t)i); });
    }
    // Emit this level's nodes; children go to the next level, contiguous.
    std::vector<Job> next_level;
    const size_t first_next = base + L;
    for (size_t i = 0; i < L; ++i) {
      t.centroid.insert(t.centroid.end(), cent.begin() + i * d, cent.begin() + (i + 1) * d);
      t.radius.push_back(rad[i]);
      t.boxlo.insert(t.boxlo.end(), blo.begin() + i * kBoxDims, blo.begin() + (i + 1) * kBoxDims);
      t.boxhi.insert(t.boxhi.end(), bhi.begin() + i * kBoxDims, bhi.begin() + (i + 1) * kBoxDims);
      t.depth.push_back(level[i].depth);
      t.max_depth = std::max(t.max_depth, level[i].depth);
      if (!splits[i].empty()) {
        t.first_child.push_back((int32_t)(first_next + next_level.size()));
        t.n_children.push_back((int32_t)splits[i].size());
        t.leaf_start.push_back(0);
        t.leaf_count.push_back(0);
        for (auto& c : splits[i]) next_level.push_back(Job{std::move(c), level[i].depth + 1});
      } else {
        t.first_child.push_back(-1);
        t.n_children.push_back(0);
        t.leaf_start.push_back(leaf_cursor);
        t.leaf_count.push_back((int32_t)level[i].ids.size());
        t.perm.insert(t.perm.end(), level[i].ids.begin(), level[i].ids.end());
        leaf_cursor += (int32_t)level[i].ids.size();
        t.n_leaves++;
      }
    }
    level = std::move(next_level);
  }
  return t;
}

// Replay of an externally built tree (the reference's KmTree, recovered from
// its public structure_json() + leaves(), km_tree.cpp:286-318).  Input:
// child counts in pre-order DFS (children in the reference's order) and the
// leaf member lists in DFS order.  Every node's id list is the ascending union
// of its leaves (clusters preserve id order, km_tree.cpp:113-116), so centroid
// and radius are recomputed with the reference's ordered fp64 loops
// (km_tree.cpp:162-171).  The backtrack tie id is the reference's post-order
// node id (km_tree.cpp:159,187-188).  Output layout: breadth-first,
// contiguous children, like build_tree_host.
HostTree import_tree_host(const double* P, int64_t N, int d, const int32_t* n_children_pre,
                          int64_t n_nodes, const int32_t* leaf_sizes, int64_t n_leaves,
                          const int32_t* leaf_ids) {
  if (n_nodes < 1 || n_leaves < 1) fail(PSG_E_SHAPE, "tree import: empty tree");
  struct PNode {
    std::vector<int32_t> kids;  // pre-order indices of the children
    int64_t leaf = -1;          // DFS leaf number
    int32_t post = -1;
    int depth = 0;
  };
  std::vector<PNode> pn((size_t)n_nodes);
  // pre-order parse with an explicit stack of (node, children still expected)
  int64_t leaf_no = 0, post = 0;
  std::vector<std::pair<int64_t, int32_t>> st;
  for (int64_t i = 0; i < n_nodes; ++i) {
    const int32_t nc = n_children_pre[i];
    if (nc < 0) fail(PSG_E_SHAPE, "tree import: negative child count");
    if (i > 0) {
      if (st.empty()) fail(PSG_E_SHAPE, "tree import: more nodes than the structure holds");
      pn[(size_t)st.back().first].kids.push_back((int32_t)i);
      pn[(size_t)i].depth = pn[(size_t)st.back().first].depth + 1;
      --st.back().second;
    }
    if (nc == 0) {
      if (leaf_no >= n_leaves) fail(PSG_E_SHAPE, "tree import: more leaves than leaf lists");
      pn[(size_t)i].leaf = leaf_no++;
      pn[(size_t)i].post = (int32_t)post++;
    } else {
      st.emplace_back(i, nc);
    }
    while (!st.empty() && st.back().second == 0) {  // subtree complete: post-order id
      pn[(size_t)st.back().first].post = (int32_t)post++;
      st.pop_back();
    }
  }
  if (!st.empty() || leaf_no != n_leaves)
    fail(PSG_E_SHAPE, "tree import: structure and leaf lists disagree");
  // leaf lists, ids must form a permutation of [0, N)
  std::vector<int64_t> loff((size_t)n_leaves + 1, 0);
  for (int64_t l = 0; l < n_leaves; ++l) {
    if (leaf_sizes[l] < 1) fail(PSG_E_SHAPE, "tree import: empty leaf");
    loff[(size_t)l + 1] = loff[(size_t)l] + leaf_sizes[l];
  }
  if (loff.back() != N) fail(PSG_E_SHAPE, "tree import: leaves do not hold N points");
  {
    std::vector<char> seen((size_t)N, 0);
    for (int64_t i = 0; i < N; ++i) {
      const int32_t id = leaf_ids[i];
      if (id < 0 || id >= N || seen[(size_t)id]) fail(PSG_E_SHAPE, "tree import: ids are not a permutation");
      seen[(size_t)id] = 1;
    }
  }
  // breadth-first relayout
  std::vector<int64_t> order;  // BFS position -> pre-order index
  order.reserve((size_t)n_nodes);
  order.push_back(0);
  std::vector<int32_t> bfs_of((size_t)n_nodes, -1);
  for (size_t h = 0; h < order.size(); ++h) {
    bfs_of[(size_t)order[h]] = (int32_t)h;
    for (int32_t c : pn[(size_t)order[h]].kids) order.push_back(c);
  }
  // ascending id list per node, bottom-up (reverse BFS: children first)
  std::vector<std::vector<int32_t>> ids((size_t)n_nodes);
  for (int64_t h = n_nodes - 1; h >= 0; --h) {
    const PNode& nd = pn[(size_t)order[(size_t)h]];
    auto& v = ids[(size_t)h];
    if (nd.leaf >= 0) {
      v.assign(leaf_ids + loff[(size_t)nd.leaf], leaf_ids + loff[(size_t)nd.leaf + 1]);
      std::sort(v.begin(), v.end());
    } else {
      for (int32_t c : nd.kids) {
        const auto& cv = ids[(size_t)bfs_of[(size_t)c]];
        v.insert(v.end(), cv.begin(), cv.end());
      }
      std::sort(v.begin(), v.end());
    }
  }
  HostTree t;
  const size_t nn = (size_t)n_nodes;
  t.centroid.assign(nn * (size_t)d, 0.0);
  t.radius.assign(nn, 0.0);
  t.first_child.assign(nn, -1);
  t.n_children.assign(nn, 0);
  t.leaf_start.assign(nn, 0);
  t.leaf_count.assign(nn, 0);
  t.depth.assign(nn, 0);
  t.tie.assign(nn, 0);
  t.boxlo.assign(nn * kBoxDims, 0.0);
  t.boxhi.assign(nn * kBoxDims, 0.0);
  const int KB = std::min(d, kBoxDims);
  for (size_t h = 0; h < nn; ++h) {
    const PNode& nd = pn[(size_t)order[h]];
    const auto& v = ids[h];
    double* c = t.centroid.data() + h * d;
    for (int32_t id : v)
      for (int j = 0; j < d; ++j) c[j] += P[(size_t)id * d + j];
    for (int j = 0; j < d; ++j) c[j] /= (double)v.size();
    double r = 0.0;
    for (int32_t id : v) r = std::max(r, std::sqrt(dist2(P + (size_t)id * d, c, d)));
    t.radius[h] = r;
    for (int j = 0; j < KB; ++j) {
      double mn = P[(size_t)v[0] * d + j], mx = mn;
      for (int32_t id : v) {
        mn = std::min(mn, P[(size_t)id * d + j]);
        mx = std::max(mx, P[(size_t)id * d + j]);
      }
      t.boxlo[h * kBoxDims + j] = mn;
      t.boxhi[h * kBoxDims + j] = mx;
    }
    t.depth[h] = nd.depth;
    t.max_depth = std::max(t.max_depth, nd.depth);
    t.tie[h] = nd.post;
    if (!nd.kids.empty()) {
      t.first_child[h] = bfs_of[(size_t)nd.kids[0]];
      t.n_children[h] = (int32_t)nd.kids.size();
    } else {
      t.leaf_start[h] = (int32_t)t.perm.size();
      t.leaf_count[h] = (int32_t)v.size();
      t.perm.insert(t.perm.end(), v.begin(), v.end());
      t.n_leaves++;
    }
  }
  return t;
}

}  // namespace psg
