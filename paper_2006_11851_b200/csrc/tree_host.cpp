// Host side of the k-means tree: import / replay of the reference's own
// tree, and the opt-in replica of KmTree::build that produces it.
//
// The default tree is built on the device (kernels_tree.cu: level-synchronous
// k-means++/Lloyd, one splitmix64 stream per node, optional depth cap).  Exact
// queries do not depend on the tree (km_tree.cpp:251-278), but greedy and
// backtrack(m) answers do; the reference's default budget is backtrack(4)
// (optimizer.hpp:48, persyn_main.cpp:79).  psg_index_cfg.tree_kind =
// PSG_TREE_REFERENCE therefore rebuilds the reference's tree itself:
// KmTree::build (km_tree.cpp:141-195) draws its k-means++ seeds from ONE
// std::mt19937_64 shared by all nodes in the recursion's (pre-)order, with
// libstdc++'s uniform_int / uniform_real distributions.  Every draw depends on
// all draws before it, so the replica is a sequential walk by construction; it
// uses the same engine and distribution types from the same C++ library, the
// same fp64 loops (sequential j, no FMA: -ffp-contract=off) and the same
// tie rules, and emits the tree in the public structure_json() + leaves()
// form that import_tree_host replays (post-order tie ids included).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include <thread>

#include "kmeans_host.h"
#include "psg_internal.h"

namespace psg {
namespace {

inline double dist2(const double* a, const double* b, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = a[j] - b[j];
    acc += t * t;
  }
  return acc;
}

}  // namespace

// KmTree::build(points, d, N, branching, leaf_threshold, seed)
// (km_tree.cpp:141-195) as a pre-order walk: a node holding
// >= leaf_threshold points (and d > 0) is clustered with k = min(b, n), and
// split when >= 2 clusters are non-empty; its children are then built one
// subtree at a time in cluster order -- the recursion's order, hence the
// order in which the shared engine is consumed.
void reference_tree_walk(const double* P, int64_t N, int d, int branching, int leaf_threshold,
                         uint64_t seed, std::vector<int32_t>& n_children,
                         std::vector<int32_t>& leaf_sizes, std::vector<int32_t>& leaf_ids) {
  if (N < 1) fail(PSG_E_DOMAIN, "cannot build a tree over zero points");
  if (branching < 2) fail(PSG_E_DOMAIN, "tree branching must be >= 2");
  if (leaf_threshold <= 0) leaf_threshold = branching;
  std::mt19937_64 rng(seed);
  // the k-means of large nodes runs on a few host threads (kmeans_host.cpp);
  // the walk itself and every RNG draw stay sequential
  const unsigned hw = std::thread::hardware_concurrency();
  HostPool pool(N >= 4096 ? (int)std::min(16u, std::max(1u, hw)) : 1);
  n_children.clear();
  leaf_sizes.clear();
  leaf_ids.clear();
  leaf_ids.reserve((size_t)N);
  std::vector<std::vector<int32_t>> todo(1);
  todo[0].resize((size_t)N);
  for (int64_t i = 0; i < N; ++i) todo[0][(size_t)i] = (int32_t)i;
  while (!todo.empty()) {
    std::vector<int32_t> ids = std::move(todo.back());
    todo.pop_back();
    if ((int64_t)ids.size() >= leaf_threshold && d > 0) {
      const int k = (int)std::min<size_t>((size_t)branching, ids.size());
      auto cl = kmeans_reference(P, d, ids, k, rng, &pool);
      if (cl.size() >= 2) {
        n_children.push_back((int32_t)cl.size());
        for (size_t c = cl.size(); c-- > 0;) todo.push_back(std::move(cl[c]));
        continue;
      }
    }
    n_children.push_back(0);
    leaf_sizes.push_back((int32_t)ids.size());
    leaf_ids.insert(leaf_ids.end(), ids.begin(), ids.end());
  }
}

HostTree build_reference_tree_host(const double* P, int64_t N, int d, int branching,
                                   int leaf_threshold, uint64_t seed) {
  std::vector<int32_t> n_children, leaf_sizes, leaf_ids;
  reference_tree_walk(P, N, d, branching, leaf_threshold, seed, n_children, leaf_sizes, leaf_ids);
  return import_tree_host(P, N, d, n_children.data(), (int64_t)n_children.size(),
                          leaf_sizes.data(), (int64_t)leaf_sizes.size(), leaf_ids.data());
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
