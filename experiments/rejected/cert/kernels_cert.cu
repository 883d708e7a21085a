// Seeded exact search with a database-side certificate.
//
// Reference semantics: KmTree::query(exact) returns the lexicographic minimum
// of (fp64 dist^2 in PCA space, id) over ALL database points
// (km_tree.cpp:251-278, ann_test.cpp:225-245) -- a property of the point set,
// not of the tree.  Any procedure that provably finds that minimum is a
// drop-in for it.
//
// Certificate.  For every database point s keep the points p with
// |s - p| < r(s) (at most K of them, sorted by a rigorous lower bound l(s, p)
// of |s - p|); every unlisted point is at distance >= r(s).  A query q seeded
// with s (its previous assignment) at distance Delta >= |q - s|:
//   * an unlisted p has |q - p| >= |s - p| - Delta >= r(s) - Delta, so when
//     2 Delta < r(s) no unlisted point can reach |q - s|;
//   * a listed p with l(s, p) > 2 Delta has |q - p| > Delta >= |q - s|.
// The exact winner is therefore s or a listed point with l(s, p) <= 2 Delta:
// those are evaluated with the reference's own fp64 chain (dist2, j
// ascending) behind the tile kernel's rigorous fp32 filter, and the
// lexicographic minimum is bit-identical to the full search's.  With the
// tensor-core projection (q^ within qdelta of the exact chain's q) Delta is
// |q^ - s| + qdelta and the band bookkeeping is the tile kernel's
// (kernels_search.cu, approximate-query mode): a winner not separated from
// the runner-up by the band goes to the exact resolve path.
// Anchors whose certificate does not hold are left to the tile search
// (`done` = 0).  On the bench stage the certificate settles ~60-70% of the
// anchors of a converging EM loop with ~50 candidate evaluations each.
//
// Neighbour lists: two brute-force fp32 passes over the database (lanes =
// points s, the other points staged in shared memory and read as broadcasts).
// Pass 1 builds each point's distance histogram (quarter-octave bins of the
// fp32 dist^2 bit pattern), the radius is the upper edge of the last bin whose
// cumulative count is <= K; pass 2 recomputes the same fp32 values and lists
// the points below it; a warp per point then sorts its list.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "numerics.cuh"
#include "psg_internal.h"

namespace psg {

namespace {

constexpr int kKnnBins = 128;    // quarter-octave bins of dist^2: 2^-16 .. 2^16
constexpr int kKnnBase = 444;    // (127 - 16) << 2: dist^2 < 2^-16 -> bin 0
constexpr int kKnnTS = 128;      // staged points per round

template <class T>
T* dalloc(size_t count) {  // index-owned buffers, from the stream-ordered pool
  T* p = nullptr;
  if (count) PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, t_stream));
  return p;
}

// fp32 squared distance of staged point pr to the negated query ns: FADD2 +
// FFMA2 in a fixed order (both passes must produce the same bits).
template <int DP>
__device__ __forceinline__ float knn_d2(const float2 (&ns)[DP / 2], const float4* pr) {
  float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < DP / 4; ++k) {
    const float4 p = pr[k];
    const float2 u0 = __fadd2_rn(ns[2 * k], make_float2(p.x, p.y));
    const float2 u1 = __fadd2_rn(ns[2 * k + 1], make_float2(p.z, p.w));
    sa = __ffma2_rn(u0, u0, sa);
    sb = __ffma2_rn(u1, u1, sb);
  }
  return __fadd_rn(__fadd_rn(sa.x, sa.y), __fadd_rn(sb.x, sb.y));
}

__device__ __forceinline__ int knn_raw_bin(float d2) {
  return (int)(__float_as_uint(d2) >> 21) - kKnnBase;
}

// Rigorous lower bound of the exact |s - p| from the fp32 dist^2 x of the
// fp32-rounded points: |u - (p - s)| <= 2^-24 (|p| + |s| + |u|) per component
// (rounding of p, s and of the difference) and the fp32 sum of <= 64 squares
// is within (DP + 4) 2^-24 of its value; 5e-6 and 4e-7 (pmax + 1) dominate
// both for DP <= 64, and the fp64 chain's own rounding (~1e-14).
__device__ __forceinline__ float knn_lower(float x, float pmax) {
  const double v = sqrt((double)x) * (1.0 - 5e-6) - 4e-7 * ((double)pmax + 1.0);
  return v > 0.0 ? __double2float_rd(v) : 0.f;
}

template <int DP, int PASS>
__global__ void __launch_bounds__(128) knn_pass_kernel(const float* __restrict__ rows, int N, int K,
                                                       int16_t* __restrict__ tbin,
                                                       uint2* __restrict__ list,
                                                       int32_t* __restrict__ cnt) {
  extern __shared__ float4 knn_smem[];
  float4* stage = knn_smem;  // [kKnnTS][DP / 4]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint16_t* hist = reinterpret_cast<uint16_t*>(knn_smem + kKnnTS * (DP / 4)) + warp * kKnnBins * 32;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = s < N;
  float2 ns[DP / 2];
  {
    const float4* r = reinterpret_cast<const float4*>(rows + (size_t)(valid ? s : 0) * DP);
#pragma unroll
    for (int k = 0; k < DP / 4; ++k) {
      const float4 v = r[k];
      ns[2 * k] = make_float2(-v.x, -v.y);
      ns[2 * k + 1] = make_float2(-v.z, -v.w);
    }
  }
  if (PASS == 0) {
    for (int b = 0; b < kKnnBins; ++b) hist[b * 32 + lane] = 0;
  }
  const int tb = (PASS == 1 && valid) ? tbin[s] : -1;
  int c = 0;
  for (int base = 0; base < N; base += kKnnTS) {
    __syncthreads();
    const int n = min(kKnnTS, N - base);
    for (int f = threadIdx.x; f < kKnnTS * (DP / 4); f += blockDim.x) {
      const int i = f / (DP / 4);
      stage[f] = i < n ? reinterpret_cast<const float4*>(rows + (size_t)(base + i) * DP)[f % (DP / 4)]
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    if (PASS == 0) {
      for (int i = 0; i < n; ++i) {
        const float d2 = knn_d2<DP>(ns, stage + i * (DP / 4));
        const int b = min(max(knn_raw_bin(d2), 0), kKnnBins - 1);
        uint16_t* h = hist + b * 32 + lane;
        const uint16_t v = *h;
        *h = (uint16_t)(v + (base + i != s && v != 0xffff ? 1 : 0));
      }
    } else if (tb >= 0) {
      for (int i = 0; i < n; ++i) {
        const float d2 = knn_d2<DP>(ns, stage + i * (DP / 4));
        if (knn_raw_bin(d2) <= tb && base + i != s) {
          if (c < K) list[(size_t)s * K + c] = make_uint2(__float_as_uint(d2), (unsigned)(base + i));
          ++c;
        }
      }
    }
  }
  if (!valid) return;
  if (PASS == 0) {
    int cum = 0, t = -1;
    for (int b = 0; b < kKnnBins; ++b) {
      cum += hist[b * 32 + lane];
      if (cum > K) break;
      t = b;
    }
    tbin[s] = (int16_t)t;
  } else {
    cnt[s] = c;
  }
}

// Warp per point: rank-sort its list by (dist^2 bits, id), store
// (l(s, p) bits, id) and the radius r(s).
__global__ void __launch_bounds__(256) knn_finish_kernel(int N, int K, float pmax,
                                                         const int16_t* __restrict__ tbin,
                                                         const int32_t* __restrict__ cnt,
                                                         const uint2* __restrict__ raw,
                                                         uint2* __restrict__ list,
                                                         float* __restrict__ radius) {
  extern __shared__ unsigned long long knn_keys[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* keys = knn_keys + (size_t)warp * K;
  const int s = blockIdx.x * (blockDim.x >> 5) + warp;
  if (s >= N) return;
  const int t = tbin[s];
  int c = t >= 0 ? cnt[s] : 0;
  float r;
  if (c > K) {  // cannot happen (same fp32 values in both passes); no certificate
    c = 0;
    r = 0.f;
  } else if (t < 0) {
    r = 0.f;
  } else if (t >= kKnnBins - 1) {
    r = __int_as_float(0x7f800000);  // every other point is listed
  } else {
    r = knn_lower(__uint_as_float((unsigned)(kKnnBase + t + 1) << 21), pmax);
  }
  for (int i = lane; i < c; i += 32) {
    const uint2 e = raw[(size_t)s * K + i];
    keys[i] = ((unsigned long long)e.x << 32) | e.y;
  }
  __syncwarp();
  for (int i = lane; i < K; i += 32) {
    if (i < c) {
      const unsigned long long k = keys[i];
      int rank = 0;
      for (int j = 0; j < c; ++j) rank += keys[j] < k;
      list[(size_t)s * K + rank] =
          make_uint2(__float_as_uint(knn_lower(__uint_as_float((unsigned)(k >> 32)), pmax)),
                     (unsigned)(k & 0xffffffffu));
    } else {
      list[(size_t)s * K + i] = make_uint2(0x7f800000u, 0u);  // +inf: ends every prefix
    }
  }
  if (lane == 0) radius[s] = r;
}

__global__ void rows32_kernel(const double* __restrict__ proj, int64_t N, int d, int dp,
                              float* __restrict__ rows) {
  const int64_t n = N * dp;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / dp;
    const int j = (int)(f % dp);
    rows[f] = j < d ? (float)proj[i * d + j] : 0.f;
  }
}

// Reference chain (dist2, km_tree.cpp:15-22): j ascending, sub, mul, add.
__device__ __noinline__ double cert_dist2(const double* __restrict__ q, const double* __restrict__ p,
                                          int d) {
  double acc = 0.0;
  int j = 0;
  if (((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(p)) & 15) == 0) {
    for (; j + 8 <= d; j += 8) {
      double2 qv[4], pv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        qv[u] = __ldg(reinterpret_cast<const double2*>(q + j) + u);
        pv[u] = __ldg(reinterpret_cast<const double2*>(p + j) + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double t = dsub(qv[u].x, pv[u].x);
        acc = dadd(acc, dmul(t, t));
        t = dsub(qv[u].y, pv[u].y);
        acc = dadd(acc, dmul(t, t));
      }
    }
  }
  for (; j < d; ++j) {
    const double t = dsub(q[j], p[j]);
    acc = dadd(acc, dmul(t, t));
  }
  return acc;
}

// Thread per anchor; a warp holds an 8 x 4 anchor tile (the tile kernel's
// shape: neighbouring anchors' seeds are neighbouring windows, whose lists
// overlap in L1).
template <int DP, bool kApprox>
__global__ void __launch_bounds__(128) cert_search_kernel(CertArgs a) {
  const int lane = threadIdx.x & 31;
  const int d = a.d;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const float kInfF = __int_as_float(0x7f800000);
  const int qny = (int)(a.nq / a.qnx);
  const int tnx = (a.qnx + 7) / 8;
  const int64_t n_tiles = (int64_t)tnx * ((qny + 3) / 4);
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = wid; t < n_tiles; t += nw) {
    const int tx = (int)(t % tnx), ty = (int)(t / tnx);
    const int ix = tx * 8 + (lane & 7), iy = ty * 4 + (lane >> 3);
    if (ix >= a.qnx || iy >= qny) continue;
    const int64_t q = (int64_t)iy * a.qnx + ix;
    const int32_t s = a.seed[q];
    const double* qrow = a.q + q * d;
    double best = cert_dist2(qrow, a.proj + (int64_t)s * d, d);
    const float band2 = kApprox ? 2.f * a.qdelta[q] : 0.f;
    const float rs = a.radius[s];
    // Delta >= |q - s| for the exact chain's q (|q^ - q| <= qdelta)
    const double lim = (2.0 * (sqrt(best) * (1.0 + 1e-12) + 0.5 * (double)band2)) * (1.0 + 1e-9);
    const bool cert = !(band2 > 3.0e38f) && lim < (double)rs;
    a.done[q] = cert ? 1 : 0;
    if (!cert) continue;
    int32_t best_id = s;
    float2 q2[DP / 2];
    double qn2 = 0.0;
#pragma unroll
    for (int j = 0; j < DP / 2; ++j) {
      const double v0 = 2 * j < d ? qrow[2 * j] : 0.0;
      const double v1 = 2 * j + 1 < d ? qrow[2 * j + 1] : 0.0;
      q2[j] = make_float2(-(float)v0, -(float)v1);
      qn2 += v0 * v0 + v1 * v1;
    }
    const float qn = __double2float_ru(sqrt(qn2) * (1.0 + 1e-12));
    // the tile kernel's float thresholds (kernels_search.cu, search_tile_kernel)
    auto infl = [&](double b) -> float {
      if (!kApprox || !(b > 0.0) || b == kInf) return __double2float_ru(b);
      const double r = sqrt(b) * (1.0 + 1e-12) + (double)band2;
      return __double2float_ru(r * r * (1.0 + 1e-15));
    };
    auto thr_of = [&](float bu) {
      return bu * (1.f + 1e-4f) + 1.01e-6f * (qn + a.pnorm_max) * (sqrtf(2.f * bu + 1.f) + 1e-3f) +
             1e-30f;
    };
    float best_up = infl(best);
    float thr = thr_of(best_up);
    float sec = kInfF, thi = kInfF;
    int32_t sid = -1;
    auto push = [&](double v, int32_t id) {
      if (!kApprox || id == sid) return;
      const float vf = __double2float_rd(v);
      if (vf < sec) {
        thi = sec;
        sec = vf;
        sid = id;
      } else {
        thi = fminf(thi, vf);
      }
    };
    int64_t scanned = 1, exact = 1;
    const uint2* L = a.list + (int64_t)s * a.K;
    for (int j = 0; j < a.K; ++j) {
      const uint2 e = __ldg(L + j);
      if ((double)__uint_as_float(e.x) > lim) break;  // sorted: the rest is farther
      ++scanned;
      const int32_t p = (int32_t)e.y;
      const float4* pr = reinterpret_cast<const float4*>(a.rows32 + (int64_t)p * DP);
      // 8 leading (highest variance) dims first: a partial sum above thr
      // already rules the point out (rounded sums of squares only grow)
      float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
      {
        const float4 p0 = __ldg(pr), p1 = __ldg(pr + 1);
        const float2 u0 = __fadd2_rn(q2[0], make_float2(p0.x, p0.y));
        const float2 u1 = __fadd2_rn(q2[1], make_float2(p0.z, p0.w));
        const float2 u2 = __fadd2_rn(q2[2], make_float2(p1.x, p1.y));
        const float2 u3 = __fadd2_rn(q2[3], make_float2(p1.z, p1.w));
        sa = __ffma2_rn(u0, u0, sa);
        sb = __ffma2_rn(u1, u1, sb);
        sa = __ffma2_rn(u2, u2, sa);
        sb = __ffma2_rn(u3, u3, sb);
      }
      if ((sa.x + sa.y) + (sb.x + sb.y) > thr) continue;
#pragma unroll
      for (int k = 2; k < DP / 4; ++k) {
        const float4 pv = __ldg(pr + k);
        const float2 u0 = __fadd2_rn(q2[2 * k], make_float2(pv.x, pv.y));
        const float2 u1 = __fadd2_rn(q2[2 * k + 1], make_float2(pv.z, pv.w));
        sa = __ffma2_rn(u0, u0, sa);
        sb = __ffma2_rn(u1, u1, sb);
      }
      const float sv = (sa.x + sa.y) + (sb.x + sb.y);
      if (sv > thr) continue;
      const float eps = 2.5e-7f * (float)(d + 4) * sv + 1.0e-6f * (qn + a.pnorm_max) * (sqrtf(sv) + 1e-3f) +
                        1e-30f;
      if (sv - eps > best_up) continue;
      const double d2 = cert_dist2(qrow, a.proj + (int64_t)p * d, d);
      ++exact;
      if (d2 < best || (d2 == best && p < best_id)) {
        push(best, best_id);
        best = d2;
        best_id = p;
        best_up = infl(best);
        thr = thr_of(best_up);
      } else {
        push(d2, p);
      }
    }
    if (kApprox) {
      const double r = sqrt(best) * (1.0 + 1e-12) + (double)band2;
      const double band = r * r * (1.0 + 1e-15);
      if ((double)sec <= band) {
        const bool pair = (double)thi > band;  // exactly {best, second} in the band
        const int slot = atomicAdd(a.amb_count, 1);
        a.amb_list[slot] = (int32_t)q;
        a.amb_c0[slot] = best_id;
        a.amb_c1[slot] = pair ? sid : -1;
      }
    }
    a.out_idx[q] = best_id;
    a.out_d2[q] = best;
    if (a.out_scanned) a.out_scanned[q] = scanned;
    if (a.out_exact) a.out_exact[q] = exact;
    if (a.out_visited) a.out_visited[q] = 0;
  }
}

}  // namespace

bool knn_supported(const Index& ix) { return ix.d > 0 && ix.d <= 64 && ix.N >= 2; }

void knn_prepare(psg_ctx* ctx, const Index& ixc, int K) {
  Index& ix = const_cast<Index&>(ixc);  // lazily built, owned by the index
  if (ix.knn_list && ix.knn_k == K) return;
  if (!knn_supported(ix)) fail(PSG_E_LOGIC, "certificate lists need 0 < d <= 64");
  for (void* p : {(void*)ix.knn_list, (void*)ix.knn_r, (void*)ix.rows32})
    if (p) cudaFreeAsync(p, ctx->stream);
  const int dp = ix.d <= 32 ? 32 : 64;
  const int N = (int)ix.N;
  ix.knn_k = K;
  ix.knn_dp = dp;
  ix.rows32 = dalloc<float>((size_t)N * dp);
  ix.knn_list = dalloc<uint2>((size_t)N * K);
  ix.knn_r = dalloc<float>(N);
  {
    ProfScope _prof(ctx, K_BUILD);
    rows32_kernel<<<std::max(1, std::min(ctx->num_sms * 8, (int)(((int64_t)N * dp + 255) / 256))), 256, 0,
                    ctx->stream>>>(ix.proj, ix.N, ix.d, dp, ix.rows32);
    PSG_LAUNCHED(ctx);
  }
  DBuf<int16_t> tbin(N);
  DBuf<int32_t> cnt(N);
  DBuf<uint2> raw((size_t)N * K);
  const int blocks = (N + 127) / 128;
  const size_t sm0 = sizeof(float4) * kKnnTS * (dp / 4) + sizeof(uint16_t) * 4 * kKnnBins * 32;
  const size_t sm1 = sizeof(float4) * kKnnTS * (dp / 4);
  {
    ProfScope _prof(ctx, K_BUILD);
    if (dp == 32) {
      PSG_CUDA(cudaFuncSetAttribute(knn_pass_kernel<32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0));
      knn_pass_kernel<32, 0><<<blocks, 128, sm0, ctx->stream>>>(ix.rows32, N, K, tbin.p, raw.p, cnt.p);
      PSG_LAUNCHED(ctx);
      knn_pass_kernel<32, 1><<<blocks, 128, sm1, ctx->stream>>>(ix.rows32, N, K, tbin.p, raw.p, cnt.p);
    } else {
      PSG_CUDA(cudaFuncSetAttribute(knn_pass_kernel<64, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm0));
      knn_pass_kernel<64, 0><<<blocks, 128, sm0, ctx->stream>>>(ix.rows32, N, K, tbin.p, raw.p, cnt.p);
      PSG_LAUNCHED(ctx);
      knn_pass_kernel<64, 1><<<blocks, 128, sm1, ctx->stream>>>(ix.rows32, N, K, tbin.p, raw.p, cnt.p);
    }
    PSG_LAUNCHED(ctx);
  }
  {
    ProfScope _prof(ctx, K_BUILD);
    const size_t smf = sizeof(unsigned long long) * 8 * K;
    PSG_CUDA(cudaFuncSetAttribute(knn_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf));
    knn_finish_kernel<<<(N + 7) / 8, 256, smf, ctx->stream>>>(N, K, ix.pnorm_max, tbin.p, cnt.p, raw.p,
                                                              ix.knn_list, ix.knn_r);
    PSG_LAUNCHED(ctx);
  }
}

void launch_cert_search(psg_ctx* ctx, const CertArgs& a, bool approx) {
  ProfScope _prof(ctx, K_CERT);
  if (a.nq <= 0) return;
  const int64_t tiles = ((a.qnx + 7) / 8) * (((a.nq / a.qnx) + 3) / 4);
  int64_t blocks = (tiles + 3) / 4;
  const int64_t cap = (int64_t)ctx->num_sms * 16;
  if (blocks > cap) blocks = cap;
  if (a.dp == 32)
    (approx ? cert_search_kernel<32, true> : cert_search_kernel<32, false>)<<<(int)blocks, 128, 0, ctx->stream>>>(a);
  else
    (approx ? cert_search_kernel<64, true> : cert_search_kernel<64, false>)<<<(int)blocks, 128, 0, ctx->stream>>>(a);
  PSG_LAUNCHED(ctx);
}

struct Unsettled {
  const uint8_t* done;
  __device__ __forceinline__ bool operator()(const int32_t q) const { return !done[q]; }
};

size_t compact_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceSelect::If(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr, (int*)nullptr, (int)n,
                        Unsettled{nullptr});
  return bytes;
}

void launch_compact_unsettled(psg_ctx* ctx, const int32_t* order, const uint8_t* done, int64_t n,
                              int32_t* out, int* count, void* temp, size_t temp_bytes) {
  ProfScope _prof(ctx, K_SCHED);
  PSG_CUDA(cub::DeviceSelect::If(temp, temp_bytes, order, out, count, (int)n, Unsettled{done}, ctx->stream));
  PSG_LAUNCHED(ctx);
}

}  // namespace psg
