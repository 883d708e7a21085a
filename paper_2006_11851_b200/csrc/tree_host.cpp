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
//     order, so levels build in parallel and deterministically;
//   * optional depth cap.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "psg_internal.h"

namespace psg {
namespace {

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

struct Job {
  std::vector<int32_t> ids;
  int depth;
};

// k-means++ + Lloyd over ids (ascending); returns non-empty clusters with
// ascending ids.
std::vector<std::vector<int32_t>> cluster(const double* P, int d, const std::vector<int32_t>& ids,
                                          int k, uint64_t seed) {
  const size_t n = ids.size();
  SplitMix rng{seed};
  std::vector<double> centers;
  centers.reserve((size_t)k * d);
  const size_t first = rng.next() % n;
  centers.insert(centers.end(), P + (size_t)ids[first] * d, P + (size_t)ids[first] * d + d);
  std::vector<double> d2(n);
  for (size_t i = 0; i < n; ++i) d2[i] = dist2(P + (size_t)ids[i] * d, centers.data(), d);
  int nc = 1;
  while (nc < k) {
    double total = 0.0;
    for (double v : d2) total += v;
    if (total <= 0.0) break;
    double r = rng.uniform01() * total;
    size_t chosen = n - 1;
    for (size_t i = 0; i < n; ++i) {
      r -= d2[i];
      if (r <= 0.0) {
        chosen = i;
        break;
      }
    }
    const double* c = P + (size_t)ids[chosen] * d;
    centers.insert(centers.end(), c, c + d);
    ++nc;
    for (size_t i = 0; i < n; ++i)
      d2[i] = std::min(d2[i], dist2(P + (size_t)ids[i] * d, c, d));
  }
  std::vector<int> assign(n);
  auto reassign = [&] {
    for (size_t i = 0; i < n; ++i) {
      const double* p = P + (size_t)ids[i] * d;
      int best = 0;
      double bd = dist2(p, centers.data(), d);
      for (int c = 1; c < nc; ++c) {
        const double dd = dist2(p, centers.data() + (size_t)c * d, d);
        if (dd < bd) {
          bd = dd;
          best = c;
        }
      }
      assign[i] = best;
    }
  };
  reassign();
  std::vector<double> sums((size_t)nc * d);
  std::vector<size_t> sizes(nc);
  for (int sweep = 0; sweep < 20; ++sweep) {
    std::fill(sums.begin(), sums.end(), 0.0);
    std::fill(sizes.begin(), sizes.end(), 0);
    for (size_t i = 0; i < n; ++i) {
      const double* p = P + (size_t)ids[i] * d;
      double* s = sums.data() + (size_t)assign[i] * d;
      for (int j = 0; j < d; ++j) s[j] += p[j];
      ++sizes[assign[i]];
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
  for (size_t i = 0; i < n; ++i) clusters[assign[i]].push_back(ids[i]);
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
  unsigned hw = std::thread::hardware_concurrency();
  if (hw == 0) hw = 1;

  while (!level.empty()) {
    const size_t base = t.radius.size();
    const size_t L = level.size();
    std::vector<std::vector<std::vector<int32_t>>> splits(L);
    std::vector<double> cent(L * (size_t)d), rad(L);
    const int KB = std::min(d, kBoxDims);
    std::vector<double> blo(L * kBoxDims, 0.0), bhi(L * kBoxDims, 0.0);
    auto work = [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
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
          auto cl = cluster(P, d, ids, k, node_seed(seed, (int64_t)(base + i)));
          if (cl.size() >= 2) splits[i] = std::move(cl);
        }
      }
    };
    // Heavy nodes first get their own thread; tail in chunks.
    const size_t nthreads = std::min<size_t>(hw, L);
    if (nthreads <= 1) {
      work(0, L);
    } else {
      std::vector<std::thread> pool;
      std::atomic<size_t> next{0};
      for (size_t th = 0; th < nthreads; ++th)
        pool.emplace_back([&] {
          for (;;) {
            const size_t i = next.fetch_add(1);
            if (i >= L) break;
            work(i, i + 1);
          }
        });
      for (auto& th : pool) th.join();
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

}  // namespace psg
