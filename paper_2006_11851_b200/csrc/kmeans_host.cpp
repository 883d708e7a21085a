// Clusterer::run of the reference's KmTree::build (km_tree.cpp:34-119),
// restated for speed without changing one rounding:
//
//  * every distance is the reference's chain  acc += (p_j - c_j)^2, j
//    ascending, multiply then add (this file is compiled with
//    -ffp-contract=off; no FMA is formed);
//  * the reassign step evaluates 8 centres at a time -- the 8 chains are
//    independent, so running them in the lanes of one vector register changes
//    nothing (target_clones: AVX-512 / AVX2 / baseline picked at load time);
//  * large nodes split their points over a thread pool: per-point results
//    (best centre, D^2) do not depend on other points; the ordered cluster
//    sums are split by cluster (each still adds its points in ascending order);
//  * everything that consumes the shared std::mt19937_64 (the k-means++
//    draws, their prefix scans) stays sequential, in the reference's order.
#include "kmeans_host.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <thread>

namespace psg {

struct HostPool::Impl {
  std::vector<std::thread> workers;
  std::mutex m;
  std::condition_variable cv_work, cv_done;
  const std::function<void(size_t, size_t)>* fn = nullptr;
  size_t n = 0;
  int parts = 0, next = 0, pending = 0;
  uint64_t epoch = 0;
  bool stop = false;

  void run_part(int part) {
    const size_t b = n * (size_t)part / (size_t)parts, e = n * (size_t)(part + 1) / (size_t)parts;
    if (b < e) (*fn)(b, e);
  }
  void worker() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(m);
    for (;;) {
      cv_work.wait(lk, [&] { return stop || (epoch != seen && next < parts); });
      if (stop) return;
      while (next < parts) {
        const int part = next++;
        lk.unlock();
        run_part(part);
        lk.lock();
        if (--pending == 0) cv_done.notify_all();
      }
      seen = epoch;
    }
  }
};

HostPool::HostPool(int threads) : impl_(new Impl) {
  for (int i = 1; i < threads; ++i) impl_->workers.emplace_back([this] { impl_->worker(); });
}

HostPool::~HostPool() {
  {
    std::lock_guard<std::mutex> lk(impl_->m);
    impl_->stop = true;
  }
  impl_->cv_work.notify_all();
  for (auto& t : impl_->workers) t.join();
}

int HostPool::threads() const { return (int)impl_->workers.size() + 1; }

void HostPool::parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn) {
  Impl& p = *impl_;
  if (p.workers.empty() || n < 2) {
    fn(0, n);
    return;
  }
  std::unique_lock<std::mutex> lk(p.m);
  p.fn = &fn;
  p.n = n;
  p.parts = (int)std::min<size_t>(n, p.workers.size() + 1);
  p.next = 0;
  p.pending = p.parts;
  ++p.epoch;
  p.cv_work.notify_all();
  while (p.next < p.parts) {  // the caller works too
    const int part = p.next++;
    lk.unlock();
    p.run_part(part);
    lk.lock();
    --p.pending;
  }
  p.cv_done.wait(lk, [&] { return p.pending == 0; });
}

namespace {

inline double dist2(const double* a, const double* b, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = a[j] - b[j];
    acc += t * t;
  }
  return acc;
}

// Strict-< reassign of points [i0, i1) (km_tree.cpp:72-86: centre 0 first, a
// later centre wins only when strictly nearer).  ctr8: centres in groups of 8,
// group g at ctr8 + g*d*8, element (j, c) at [j*8 + c] (pad lanes zero).
// Four points are in flight at once: one point's 8-centre accumulator is a
// single dependent add chain (4-cycle latency per dim), so independent points
// fill the pipeline.  v8 is GCC's generic 8-double vector (lowered to 2 x
// AVX2 or 4 x SSE2 registers by the narrower clones): lane c is centre c's
// own chain t = p_j - c_j; acc = acc + t * t, separate multiply and add.
typedef double v8 __attribute__((vector_size(64), aligned(8)));

__attribute__((target_clones("default", "avx2", "avx512f"))) void assign_range(
    const double* P, const int32_t* ids, size_t i0, size_t i1, int d, const double* ctr8, int nc,
    int* assign) {
  for (size_t i = i0; i < i1; i += 4) {
    const int m = (int)std::min<size_t>(4, i1 - i);
    const double* p0 = P + (size_t)ids[i] * d;
    const double* p1 = P + (size_t)ids[i + (m > 1 ? 1 : 0)] * d;
    const double* p2 = P + (size_t)ids[i + (m > 2 ? 2 : 0)] * d;
    const double* p3 = P + (size_t)ids[i + (m > 3 ? 3 : 0)] * d;
    int best[4] = {0, 0, 0, 0};
    double bd[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c0 = 0; c0 < nc; c0 += 8) {
      const double* ct = ctr8 + (size_t)(c0 / 8) * d * 8;
      v8 a0 = {0, 0, 0, 0, 0, 0, 0, 0}, a1 = a0, a2 = a0, a3 = a0;
      for (int j = 0; j < d; ++j) {
        const v8 c = *reinterpret_cast<const v8*>(ct + (size_t)j * 8);
        const v8 t0 = p0[j] - c, t1 = p1[j] - c, t2 = p2[j] - c, t3 = p3[j] - c;
        a0 = a0 + t0 * t0;
        a1 = a1 + t1 * t1;
        a2 = a2 + t2 * t2;
        a3 = a3 + t3 * t3;
      }
      const v8 acc[4] = {a0, a1, a2, a3};
      const int lim = std::min(8, nc - c0);
      for (int u = 0; u < 4; ++u)
        for (int c = 0; c < lim; ++c) {
          const double v = acc[u][c];
          if (c0 + c == 0) {
            bd[u] = v;
          } else if (v < bd[u]) {
            bd[u] = v;
            best[u] = c0 + c;
          }
        }
    }
    for (int u = 0; u < m; ++u) assign[i + u] = best[u];
  }
}

}  // namespace

// k-means++ seeding (first centre uniform_int(0, n-1); then D^2 sampling with
// uniform_real(0, total) and the subtract-until-<=0 scan), a strict-<
// reassign (lowest centre wins ties), <= 20 Lloyd sweeps with ordered sums
// (empty clusters keep their centre) stopping when the largest move < 1e-6,
// then the non-empty clusters, each in ascending id order.
std::vector<std::vector<int32_t>> kmeans_reference(const double* P, int d,
                                                   const std::vector<int32_t>& ids, int k,
                                                   std::mt19937_64& rng, HostPool* pool) {
  const size_t n = ids.size();
  auto pt = [&](size_t i) { return P + (size_t)ids[i] * d; };
  // a node is worth the pool's hand-off (~10 us) above ~6e4 coordinates per pass
  const bool par = pool && pool->threads() > 1 && n * (size_t)d >= ((size_t)1 << 16);
  auto over_points = [&](const std::function<void(size_t, size_t)>& fn) {
    if (par) pool->parallel_for(n, fn);
    else fn(0, n);
  };
  std::vector<double> ctr;
  ctr.reserve((size_t)k * d);
  std::uniform_int_distribution<std::size_t> first(0, n - 1);
  {
    const double* c0 = pt(first(rng));
    ctr.insert(ctr.end(), c0, c0 + d);
  }
  std::vector<double> d2(n);
  over_points([&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) d2[i] = dist2(pt(i), ctr.data(), d);
  });
  int nc = 1;
  while (nc < k) {
    double total = 0.0;
    for (double v : d2) total += v;
    if (total <= 0.0) break;
    std::uniform_real_distribution<double> pick(0.0, total);
    double r = pick(rng);
    size_t chosen = n - 1;
    for (size_t i = 0; i < n; ++i) {
      r -= d2[i];
      if (r <= 0.0) {
        chosen = i;
        break;
      }
    }
    const double* c = pt(chosen);
    ctr.insert(ctr.end(), c, c + d);
    const double* cn = ctr.data() + (size_t)nc * d;
    ++nc;
    over_points([&](size_t b, size_t e) {
      for (size_t i = b; i < e; ++i) d2[i] = std::min(d2[i], dist2(pt(i), cn, d));
    });
  }
  std::vector<int> assign(n);
  const int ng = (nc + 7) / 8;
  std::vector<double> ctr8((size_t)ng * d * 8, 0.0);
  auto reassign = [&] {
    for (int c = 0; c < nc; ++c)
      for (int j = 0; j < d; ++j)
        ctr8[((size_t)(c / 8) * d + j) * 8 + (c % 8)] = ctr[(size_t)c * d + j];
    over_points([&](size_t b, size_t e) {
      assign_range(P, ids.data(), b, e, d, ctr8.data(), nc, assign.data());
    });
  };
  reassign();
  std::vector<double> sums((size_t)nc * d);
  std::vector<size_t> sizes((size_t)nc);
  for (int sweep = 0; sweep < 20; ++sweep) {
    std::fill(sums.begin(), sums.end(), 0.0);
    std::fill(sizes.begin(), sizes.end(), 0);
    for (size_t i = 0; i < n; ++i) ++sizes[(size_t)assign[i]];
    // ordered sums: each cluster adds its points in ascending order; the pool
    // splits the CLUSTERS (a thread owns whole rows of `sums`)
    auto add_clusters = [&](size_t c0, size_t c1) {
      for (size_t i = 0; i < n; ++i) {
        const size_t c = (size_t)assign[i];
        if (c < c0 || c >= c1) continue;
        const double* p = pt(i);
        double* s = sums.data() + c * d;
        for (int j = 0; j < d; ++j) s[j] += p[j];
      }
    };
    if (par && nc >= 2) pool->parallel_for((size_t)nc, add_clusters);
    else add_clusters(0, (size_t)nc);
    double movement = 0.0;
    for (int c = 0; c < nc; ++c) {
      if (sizes[(size_t)c] == 0) continue;
      double move = 0.0;
      for (int j = 0; j < d; ++j) {
        const double v = sums[(size_t)c * d + j] / sizes[(size_t)c];
        const double t = v - ctr[(size_t)c * d + j];
        move += t * t;
        ctr[(size_t)c * d + j] = v;
      }
      movement = std::max(movement, std::sqrt(move));
    }
    if (movement < 1e-6) break;
    reassign();
  }
  std::vector<std::vector<int32_t>> out((size_t)nc);
  for (size_t i = 0; i < n; ++i) out[(size_t)assign[i]].push_back(ids[i]);
  out.erase(std::remove_if(out.begin(), out.end(),
                           [](const std::vector<int32_t>& v) { return v.empty(); }),
            out.end());
  return out;
}

}  // namespace psg
