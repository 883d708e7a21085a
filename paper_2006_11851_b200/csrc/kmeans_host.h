// Host k-means of the KmTree::build replica (tree_host.cpp), compiled by the
// host compiler alone (kmeans_host.cpp): SIMD across centres + a small thread
// pool across points, bit-identical to the scalar loops it replaces.
#pragma once
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <random>
#include <vector>

namespace psg {

// Persistent worker threads for the large nodes of one tree build.
class HostPool {
 public:
  explicit HostPool(int threads);
  ~HostPool();
  int threads() const;
  // fn(begin, end) over a partition of [0, n) -- disjoint ranges, any order
  void parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// Clusterer::run (km_tree.cpp:34-119) over ascending ids; see kmeans_host.cpp.
std::vector<std::vector<int32_t>> kmeans_reference(const double* P, int d,
                                                   const std::vector<int32_t>& ids, int k,
                                                   std::mt19937_64& rng, HostPool* pool);

}  // namespace psg
