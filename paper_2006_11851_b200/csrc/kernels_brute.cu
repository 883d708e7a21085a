// Brute-force nearest neighbour on the tensor cores (BruteForceIndex::nearest,
// optimizer.cpp:175-205), sm_100a.
//
// The reference scans every candidate with an fp64 j-sequential dist^2 and
// keeps the first index of the minimum (early abandoning never changes the
// answer: partial sums only grow and ties need a strict <).  Here:
//
//  1. filter (kind::tf32 UMMA, TMEM accumulators): for a 128-query x
//     256-candidate tile, s = |q'|^2 + |p'|^2 - 2 q'.p' with q' = q - mu,
//     p' = p - mu centred by the database mean (distances are unchanged,
//     norms and hence the filter error shrink) and rounded to tf32.  A rigorous
//     bound E(q, p) >= |s - dist^2| (tf32 rounding, fp32 accumulation, centring,
//     epilogue rounding) gives each query an upper bound U on
//     its minimum and a short list of candidates whose lower bound s - E can
//     still reach U;
//  2. resolve: the survivors are re-evaluated with the reference's exact fp64
//     chain over the ORIGINAL fp32 rows; the lexicographic minimum of
//     (dist^2, id) is the reference's answer bit for bit.
//
// Pipeline per CTA (1 per SM, 6 warps): warp 0 streams A/B K-chunks with 1-D
// TMA bulk copies into a 4-stage shared-memory ring, warp 1 issues the UMMAs
// (one elected thread), warps 2-5 run the epilogue from a double-buffered
// 2 x 256-column TMEM accumulator, so tile t+1 multiplies while tile t is
// filtered.  Operands are pre-tiled in HBM in the no-swizzle K-major canonical
// layout (8-row x 16-byte core matrices; LBO 128 B along K, SBO 1024 B between
// 8-row groups), so every stage is two contiguous bulk copies.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <vector>

#include "numerics.cuh"
#include "psg_internal.h"
#include "umma.cuh"

namespace psg {

namespace {

constexpr int kBM = 128;      // queries per CTA (UMMA M)
constexpr int kBN = 256;      // candidates per accumulator tile (UMMA N)
constexpr int kBK = 32;       // fp32 elements per K chunk (128-byte rows)
constexpr int kStages = 4;
constexpr int kList = 32;     // survivors kept per (query, split) between compactions
constexpr uint32_t kABytes = kBM * kBK * 4;  // 16 KB
constexpr uint32_t kBBytes = kBN * kBK * 4;  // 32 KB
constexpr int kThreads = 192;

struct BruteSmem {
  uint32_t stages, pn2, pnup, bars, tmem, total;
};
__host__ __device__ constexpr BruteSmem brute_smem() {
  BruteSmem s{};
  uint32_t o = 0;
  s.stages = o; o += kStages * (kABytes + kBBytes);
  s.pn2 = o; o += 2 * kBN * 4;
  s.pnup = o; o += 2 * kBN * 4;
  s.bars = o; o += (2 * kStages + 4) * 8;
  s.tmem = o; o += 16;
  s.total = o;
  return s;
}

// Element j of row r, sequentially: windows are w rows of w*C contiguous floats.
struct RowCursor {
  const float* p;
  int left, seg, seglen;
  __device__ RowCursor(const RowSrc& s, int64_t r) {
    seg = 0;
    if (s.kind == 0) {
      p = s.base + r * s.D;
      seglen = s.D;
    } else {
      int x, y;
      if (s.xs) {
        x = s.xs[r % s.nx];
        y = s.ys[r / s.nx];
      } else {
        x = (int)(r % s.nx);
        y = (int)(r / s.nx);
      }
      p = s.base + ((int64_t)y * s.img_w + x) * s.C;
      seglen = s.w * s.C;
    }
    left = seglen;
  }
  __device__ __forceinline__ float next(const RowSrc& s) {
    const float v = *p++;
    if (--left == 0) {
      left = seglen;
      p += (int64_t)(s.img_w - s.w) * s.C;  // next window row (vectors: never reached)
    }
    return v;
  }
};

// The reference's exact distance (optimizer.cpp:184-190 without the early
// abandon, whose result it never changes): fp64, j ascending, mul then add.
__device__ __noinline__ double exact_d2(const RowSrc& qs, int64_t qi, const RowSrc& ps, int64_t pi,
                                        int D) {
  RowCursor a(qs, qi), b(ps, pi);
  double acc = 0.0;
  for (int j = 0; j < D; ++j) {
    const double t = dsub((double)a.next(qs), (double)b.next(ps));
    acc = dadd(acc, dmul(t, t));
  }
  return acc;
}

// dot[jj] for a warp-divergent jj without demoting the array to local memory.
__device__ __forceinline__ float dot_at(const float (&dot)[32], int jj) {
  float v = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) v = (i == jj) ? dot[i] : v;
  return v;
}

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Rows -> tiled tf32 operand [tiles][nch][tile_rows * 32] + norms of the
// centred fp32 rows (computed in fp64 before the tf32 rounding).
__global__ void brute_pack_kernel(RowSrc src, int64_t n, int64_t n_pad, int D, int nch,
                                  int tile_rows, const float* __restrict__ mu,
                                  float* __restrict__ op, float* __restrict__ n2,
                                  float* __restrict__ nup) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_pad;
       r += (int64_t)gridDim.x * blockDim.x) {
    const bool valid = r < n;
    const int64_t tile = r / tile_rows;
    const int rr = (int)(r - tile * tile_rows);
    RowCursor cur(src, valid ? r : 0);
    double acc = 0.0;
    for (int c = 0; c < nch; ++c) {
      float v[kBK];
#pragma unroll
      for (int k = 0; k < kBK; ++k) {
        const int j = c * kBK + k;
        float x = 0.f;
        if (valid && j < D) x = __fsub_rn(cur.next(src), mu[j]);
        acc += (double)x * (double)x;
        v[k] = tf32_rn(x);
      }
      float* blk = op + ((int64_t)tile * nch + c) * ((int64_t)tile_rows * kBK);
      float4* o4 = reinterpret_cast<float4*>(blk + (rr >> 3) * 256 + (rr & 7) * 4);
#pragma unroll
      for (int g = 0; g < kBK / 4; ++g)
        o4[g * 8] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    }
    n2[r] = (float)acc;
    nup[r] = valid ? __double2float_ru(sqrt(acc) * (1.0 + 1e-12)) : 0.f;
  }
}

void launch_pack(psg_ctx* ctx, const RowSrc& src, int64_t n, int64_t n_pad, int D, int nch,
                 int tile_rows, const float* mu, float* op, float* n2, float* nup) {
  const int threads = 128;
  int64_t blocks = (n_pad + threads - 1) / threads;
  if (blocks > (int64_t)ctx->num_sms * 16) blocks = (int64_t)ctx->num_sms * 16;
  brute_pack_kernel<<<(int)blocks, threads, 0, ctx->stream>>>(src, n, n_pad, D, nch, tile_rows,
                                                              mu, op, n2, nup);
  PSG_LAUNCHED(ctx);
}

struct BruteArgs {
  const float* qop;
  const float* qn2;
  const float* qnup;
  const float* qU0;     // [nq] initial upper bound (seed distance rounded up) or +inf
  const float* pop;
  const float* pn2;
  const float* pnup;
  const float* tmax;    // [ptiles] largest |p'| bound of each candidate tile
  int64_t nq, N;
  int nch, ptiles, splits, D;
  float c1, c2;  // |s - dist^2| <= c1 |q'||p'| + c2 (|q'| + |p'|)^2
  RowSrc qs, ps;
  // survivors per (query, split): U, count, list
  float* o_U;
  int32_t* o_n;
  int32_t* o_ids;  // [nq * splits][kList]
  float* o_lb;
  // overflow of full lists: (query, id, lb) triples
  unsigned long long* ov_count;
  int64_t ov_cap;
  int64_t* ov_q;
  int32_t* ov_id;
  float* ov_lb;
  int32_t* lost;   // [nq] a survivor could not be stored: settle by a full scan
};

// Survivor bookkeeping of one query (rare path, kept out of the unrolled
// epilogue loop): tighten U, append (id, lb) to the (query, split) list in
// global memory; when the list is full drop the entries U has ruled out, and
// if it is still full spill to the shared overflow buffer.  No exact distance
// is evaluated here: a stalled epilogue thread would stall the whole CTA.
__device__ __noinline__ void push_candidate(const BruteArgs& a, int64_t q, int32_t id, float lb,
                                            float ub, int32_t* gid, float* glb, float& U,
                                            int& n) {
  U = fminf(U, ub);
  if (n == kList) {
    int m = 0;
    for (int i = 0; i < n; ++i) {
      const float li = glb[i];
      if (li <= U) {
        glb[m] = li;
        gid[m] = gid[i];
        ++m;
      }
    }
    n = m;
  }
  if (lb > U) return;
  if (n < kList) {
    glb[n] = lb;
    gid[n] = id;
    ++n;
    return;
  }
  const unsigned long long k = atomicAdd(a.ov_count, 1ull);
  if ((int64_t)k < a.ov_cap) {
    a.ov_q[k] = q;
    a.ov_id[k] = id;
    a.ov_lb[k] = lb;
  } else {
    a.lost[q] = 1;
  }
}

__global__ void __launch_bounds__(kThreads, 1) brute_mma_kernel(BruteArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr BruteSmem L = brute_smem();
  float* s_pn2 = reinterpret_cast<float*>(smem + L.pn2);    // [2][kBN]
  float* s_pnup = reinterpret_cast<float*>(smem + L.pnup);  // [2][kBN]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(smem + L.tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qt = blockIdx.x, split = blockIdx.y;
  const int pt0 = (int)((int64_t)split * a.ptiles / a.splits);
  const int pt1 = (int)((int64_t)(split + 1) * a.ptiles / a.splits);
  const int npt = pt1 - pt0;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     mma::smem_u32(tmem_s)),
                 "r"(2 * kBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) {
      mma::mbar_init(&full[s], 1);
      mma::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mma::mbar_init(&tfull[b], 1);
      mma::mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mma::fence_async_smem();
  }
  mma::fence_before();
  __syncthreads();
  mma::fence_after();
  const uint32_t tmem = *tmem_s;

  if (warp == 0) {
    // ---- producer: A (query chunk) + B (candidate chunk) per stage ------------
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int it = 0; it < npt; ++it) {
        const int64_t pt = pt0 + it;
        for (int c = 0; c < a.nch; ++c) {
          mma::mbar_wait(&empty[stage], ph ^ 1u);
          uint8_t* sa = smem + L.stages + stage * (kABytes + kBBytes);
          mma::mbar_expect_tx(&full[stage], kABytes + kBBytes);
          mma::bulk_g2s(sa, a.qop + ((int64_t)qt * a.nch + c) * (kBM * kBK), kABytes, &full[stage]);
          mma::bulk_g2s(sa + kABytes, a.pop + (pt * a.nch + c) * (kBN * kBK), kBBytes,
                        &full[stage]);
          if (++stage == kStages) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ---------------------------------------------------------------
    if (lane == 0) {
      constexpr uint32_t kIdesc = mma::make_idesc_tf32(kBM, kBN);
      int stage = 0;
      uint32_t ph = 0;
      for (int it = 0; it < npt; ++it) {
        const int b = it & 1;
        const uint32_t tph = (uint32_t)(it >> 1) & 1u;
        mma::mbar_wait(&tempty[b], tph ^ 1u);
        mma::fence_after();
        const uint32_t d = tmem + (uint32_t)(b * kBN);
        for (int c = 0; c < a.nch; ++c) {
          mma::mbar_wait(&full[stage], ph);
          mma::fence_after();
          const uint32_t sa = mma::smem_u32(smem + L.stages + stage * (kABytes + kBBytes));
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int s = 0; s < kBK / 8; ++s) {
            const uint64_t ad = mma::make_desc(sa + s * 256, 128, 1024);
            const uint64_t bd = mma::make_desc(sb + s * 256, 128, 1024);
            mma::mma_tf32(d, ad, bd, kIdesc, (c | s) ? 1u : 0u);
          }
          mma::commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            ph ^= 1u;
          }
        }
        mma::commit(&tfull[b]);
      }
    }
  } else {
    // ---- epilogue: one query row per thread ---------------------------------------
    const int lg = warp & 3;  // TMEM lane group this warp may access
    const int row = lg * 32 + lane;
    const int et = tid - 64;  // 0..127: loads two candidate norms of each tile
    const int64_t q = (int64_t)qt * kBM + row;
    const bool valid = q < a.nq;
    const float qn2 = valid ? a.qn2[q] : 0.f;
    const float qa = valid ? a.qnup[q] : 0.f;
    float U = valid ? a.qU0[q] : 0.f;
    int n = 0;
    const int64_t o = (valid ? q : 0) * a.splits + split;
    int32_t* gid = a.o_ids + o * kList;
    float* glb = a.o_lb + o * kList;
    // norms of the first tile
    if (npt > 0) {
      const int64_t pb0 = (int64_t)pt0 * kBN;
      s_pn2[et] = a.pn2[pb0 + et];
      s_pn2[et + kBM] = a.pn2[pb0 + et + kBM];
      s_pnup[et] = a.pnup[pb0 + et];
      s_pnup[et + kBM] = a.pnup[pb0 + et + kBM];
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    for (int it = 0; it < npt; ++it) {
      const int b = it & 1;
      const uint32_t tph = (uint32_t)(it >> 1) & 1u;
      const int64_t pbase = (int64_t)(pt0 + it) * kBN;
      // prefetch the next tile's norms into registers (stored after this tile)
      float nx0 = 0.f, nx1 = 0.f, nu0 = 0.f, nu1 = 0.f;
      if (it + 1 < npt) {
        const int64_t nb = pbase + kBN;
        nx0 = __ldg(a.pn2 + nb + et);
        nx1 = __ldg(a.pn2 + nb + et + kBM);
        nu0 = __ldg(a.pnup + nb + et);
        nu1 = __ldg(a.pnup + nb + et + kBM);
      }
      // one loose threshold per tile (the tile's largest candidate norm);
      // candidates passing it are re-tested with their own bound, so the loop
      // below is straight-line compare code
      const float pbm = __ldg(a.tmax + pt0 + it);
      const float abm = qa + pbm;
      const float eps_t = fmaf(a.c1 * qa, pbm, a.c2 * abm * abm);
      const int jmax = (int)min((int64_t)kBN, a.N - pbase);
      mma::mbar_wait(&tfull[b], tph);
      mma::fence_after();
      for (int j0 = 0; j0 < kBN; j0 += 32) {
        float dot[32];
        __syncwarp();
        mma::tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(b * kBN + j0), dot);
        if (valid && j0 < jmax) {
          // margin: dominates the rounding of the precise test below
          const float thr = __fadd_ru(__fadd_ru(U, eps_t), fabsf(U) * 1e-6f + 1e-30f);
          const float4* pn4 = reinterpret_cast<const float4*>(s_pn2 + b * kBN + j0);
          uint32_t m = 0;
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const float4 p4 = pn4[g];
            const float s0 = fmaf(-2.f, dot[4 * g], qn2 + p4.x);
            const float s1 = fmaf(-2.f, dot[4 * g + 1], qn2 + p4.y);
            const float s2 = fmaf(-2.f, dot[4 * g + 2], qn2 + p4.z);
            const float s3 = fmaf(-2.f, dot[4 * g + 3], qn2 + p4.w);
            m |= (s0 <= thr ? 1u : 0u) << (4 * g);
            m |= (s1 <= thr ? 1u : 0u) << (4 * g + 1);
            m |= (s2 <= thr ? 1u : 0u) << (4 * g + 2);
            m |= (s3 <= thr ? 1u : 0u) << (4 * g + 3);
          }
          if (jmax - j0 < 32) m &= (1u << (jmax - j0)) - 1u;
          while (m) {
            const int jj = __ffs(m) - 1;
            m &= m - 1;
            const int j = j0 + jj;
            const float pb = s_pnup[b * kBN + j];
            const float s = fmaf(-2.f, dot_at(dot, jj), qn2 + s_pn2[b * kBN + j]);
            const float ab = qa + pb;
            const float eps = fmaf(a.c1 * qa, pb, a.c2 * ab * ab);
            const float lb = __fsub_rd(s, eps);
            if (lb <= U)
              push_candidate(a, q, (int32_t)(pbase + j), lb, __fadd_ru(s, eps), gid, glb, U, n);
          }
        }
      }
      mma::fence_before();
      __syncwarp();
      if (lane == 0) mma::mbar_arrive(&tempty[b]);
      if (it + 1 < npt) {  // buffer b^1 was last read in tile it-1 (before the last barrier)
        s_pn2[(b ^ 1) * kBN + et] = nx0;
        s_pn2[(b ^ 1) * kBN + et + kBM] = nx1;
        s_pnup[(b ^ 1) * kBN + et] = nu0;
        s_pnup[(b ^ 1) * kBN + et + kBM] = nu1;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    if (valid) {
      a.o_n[o] = n;
      a.o_U[o] = U;
    }
  }
  mma::fence_before();
  __syncthreads();
  if (warp == 0) {
    mma::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kBN));
  }
}

// Seeds (optional): the exact distance of a known candidate (the anchor's
// previous assignment) is a tight initial U, so only near-ties survive.
__global__ void brute_init_kernel(BruteArgs a, const int32_t* __restrict__ seed,
                                  double* __restrict__ seed_d2, float* __restrict__ U0,
                                  unsigned long long* __restrict__ best_bits,
                                  int32_t* __restrict__ best_id, int32_t* __restrict__ cnt) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    double d2 = __longlong_as_double(0x7ff0000000000000ll);
    if (seed) d2 = exact_d2(a.qs, q, a.ps, seed[q], a.D);
    seed_d2[q] = d2;
    U0[q] = seed ? __double2float_ru(d2) : __int_as_float(0x7f800000);
    best_bits[q] = (unsigned long long)__double_as_longlong(d2);
    best_id[q] = INT_MAX;
    cnt[q] = seed ? 1 : 0;
    a.lost[q] = 0;
  }
}

__device__ __forceinline__ float query_U(const BruteArgs& a, const float* U0, int64_t q) {
  float U = U0[q];
  for (int s = 0; s < a.splits; ++s) U = fminf(U, a.o_U[q * a.splits + s]);
  return U;
}

// Settle, pass 1: one thread per survivor (list slot or overflow entry) whose
// lower bound reaches the query's global U: the reference's sequential fp64
// distance (thread-level parallelism hides the latency of the dependent
// chain).  dist^2 >= 0, so its bit pattern orders like the value and the
// per-query minimum is an integer atomicMin.
__global__ void brute_settle_kernel(BruteArgs a, const float* __restrict__ U0,
                                    double* __restrict__ slot_d2, double* __restrict__ ov_d2,
                                    unsigned long long* __restrict__ best_bits,
                                    int32_t* __restrict__ cnt) {
  const int64_t nslots = a.nq * a.splits * kList;
  const int64_t nov = min((int64_t)*a.ov_count, a.ov_cap);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots + nov;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t q;
    int32_t id;
    float lb;
    double* out;
    if (t < nslots) {
      const int64_t o = t / kList;
      const int i = (int)(t - o * kList);
      q = o / a.splits;
      out = slot_d2 + t;
      if (i >= a.o_n[o]) {
        *out = -1.0;
        continue;
      }
      id = a.o_ids[t];
      lb = a.o_lb[t];
    } else {
      const int64_t k = t - nslots;
      q = a.ov_q[k];
      id = a.ov_id[k];
      lb = a.ov_lb[k];
      out = ov_d2 + k;
    }
    double d2 = -1.0;
    if (lb <= query_U(a, U0, q)) {
      d2 = exact_d2(a.qs, q, a.ps, id, a.D);
      atomicMin(best_bits + q, (unsigned long long)__double_as_longlong(d2));
      atomicAdd(cnt + q, 1);
    }
    *out = d2;
  }
}

// Settle, pass 2: lowest id among the candidates at the minimum (the seed too).
__global__ void brute_tie_kernel(BruteArgs a, const int32_t* __restrict__ seed,
                                 const double* __restrict__ seed_d2,
                                 const double* __restrict__ slot_d2,
                                 const double* __restrict__ ov_d2,
                                 const unsigned long long* __restrict__ best_bits,
                                 int32_t* __restrict__ best_id) {
  const int64_t nslots = a.nq * a.splits * kList;
  const int64_t nov = min((int64_t)*a.ov_count, a.ov_cap);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots + nov + a.nq;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t q;
    int32_t id;
    double d2;
    if (t < nslots) {
      d2 = slot_d2[t];
      if (d2 < 0.0) continue;
      q = t / (kList * a.splits);
      id = a.o_ids[t];
    } else if (t < nslots + nov) {
      const int64_t k = t - nslots;
      d2 = ov_d2[k];
      if (d2 < 0.0) continue;
      q = a.ov_q[k];
      id = a.ov_id[k];
    } else {
      if (!seed) continue;
      q = t - nslots - nov;
      id = seed[q];
      d2 = seed_d2[q];
    }
    if ((unsigned long long)__double_as_longlong(d2) == best_bits[q]) atomicMin(best_id + q, id);
  }
}

// Result per query.  A query whose survivor list overflowed the spill buffer
// (never observed; kept for correctness) is settled by a full exact scan.
__global__ void brute_pick_kernel(BruteArgs a, const unsigned long long* __restrict__ best_bits,
                                  const int32_t* __restrict__ best_id,
                                  const int32_t* __restrict__ cnt, int32_t* __restrict__ out_idx,
                                  double* __restrict__ out_d2, int64_t* __restrict__ out_scanned,
                                  int64_t* __restrict__ out_exact) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    double best = __longlong_as_double((long long)best_bits[q]);
    int32_t bid = best_id[q];
    int64_t exact = cnt[q];
    if (a.lost[q]) {
      best = __longlong_as_double(0x7ff0000000000000ll);
      bid = INT_MAX;
      for (int64_t i = 0; i < a.N; ++i) {
        const double d2 = exact_d2(a.qs, q, a.ps, i, a.D);
        if (d2 < best) {
          best = d2;
          bid = (int32_t)i;
        }
      }
      exact += a.N;
    }
    out_idx[q] = bid;
    out_d2[q] = best;
    if (out_scanned) out_scanned[q] = a.N;  // every candidate counts (optimizer.cpp:198)
    if (out_exact) out_exact[q] = exact;
  }
}

struct Scratch {
  void* p = nullptr;
  cudaStream_t s;
  Scratch(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) PSG_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

RowSrc db_source(const Index& ix) {
  RowSrc ps;
  ps.D = ix.D;
  if (ix.from_vectors) {
    ps.kind = 0;
    ps.base = ix.vectors;
  } else {
    ps.kind = 1;
    ps.base = ix.ex_mirror;
    ps.img_w = ix.ew;
    ps.C = ix.C;
    ps.w = ix.w;
    ps.nx = ix.nxe;
  }
  return ps;
}

}  // namespace

void brute_prepare(psg_ctx* ctx, Index& ix) {
  ProfScope _prof(ctx, K_BUILD);
  const int D = ix.D;
  ix.brute_nch = (D + kBK - 1) / kBK;
  ix.brute_ptiles = (int)((ix.N + kBN - 1) / kBN);
  const int64_t npad = (int64_t)ix.brute_ptiles * kBN;
  // centring vector: the database mean per feature (fp64 -> fp32)
  Scratch m64(sizeof(double) * D, ctx->stream);
  if (ix.from_vectors)
    launch_vector_mean(ctx, ix.vectors, ix.N, D, m64.as<double>());
  else
    launch_window_mean(ctx, ix.ex_mirror, ix.ew, ix.C, ix.w, ix.nxe, ix.N, m64.as<double>());
  std::vector<double> hm(D);
  PSG_CUDA(cudaMemcpyAsync(hm.data(), m64.p, sizeof(double) * D, cudaMemcpyDeviceToHost,
                           ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<float> mu((size_t)ix.brute_nch * kBK, 0.f);
  for (int j = 0; j < D; ++j) mu[j] = (float)hm[j];
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.brute_mu), sizeof(float) * mu.size(), ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(ix.brute_mu, mu.data(), sizeof(float) * mu.size(),
                           cudaMemcpyHostToDevice, ctx->stream));
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.brute_op), sizeof(float) * (size_t)npad * ix.brute_nch * kBK, ctx->stream));
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.brute_n2), sizeof(float) * npad, ctx->stream));
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.brute_nup), sizeof(float) * npad, ctx->stream));
  launch_pack(ctx, db_source(ix), ix.N, npad, D, ix.brute_nch, kBN, ix.brute_mu, ix.brute_op,
              ix.brute_n2, ix.brute_nup);
  // largest |p'| bound per candidate tile (the epilogue's loose per-tile threshold)
  std::vector<float> nup((size_t)npad), tmax((size_t)ix.brute_ptiles, 0.f);
  PSG_CUDA(cudaMemcpyAsync(nup.data(), ix.brute_nup, sizeof(float) * npad, cudaMemcpyDeviceToHost,
                           ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int64_t i = 0; i < npad; ++i) tmax[i / kBN] = std::max(tmax[i / kBN], nup[i]);
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.brute_tmax), sizeof(float) * tmax.size(), ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(ix.brute_tmax, tmax.data(), sizeof(float) * tmax.size(),
                           cudaMemcpyHostToDevice, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void launch_brute_search(psg_ctx* ctx, const Index& ix, const RowSrc& qsrc, int64_t nq,
                         const int32_t* seed, int32_t* out_idx, double* out_d2,
                         int64_t* out_scanned, int64_t* out_exact) {
  ProfScope _prof(ctx, K_SEARCH);
  if (nq <= 0) return;
  if (!ix.brute_op) fail(PSG_E_LOGIC, "brute-force operand not prepared");
  const int nch = ix.brute_nch;
  const int64_t qtiles = (nq + kBM - 1) / kBM;
  const int64_t qpad = qtiles * kBM;
  // split the candidate range so that the grid covers the SMs
  // (about 4 waves of one CTA per SM keep the tail of the last wave small)
  int splits = (int)std::max<int64_t>(1, (4 * (int64_t)ctx->num_sms + qtiles - 1) / qtiles);
  splits = std::min(splits, std::max(1, ix.brute_ptiles / 2));
  splits = std::min(splits, 64);
  const int64_t no = nq * splits;
  const int64_t ov_cap = std::max<int64_t>(1 << 20, 4 * nq);
  Scratch qop(sizeof(float) * (size_t)qpad * nch * kBK, ctx->stream);
  Scratch qn2(sizeof(float) * qpad, ctx->stream), qnup(sizeof(float) * qpad, ctx->stream);
  Scratch U0(sizeof(float) * nq, ctx->stream), sd(sizeof(double) * nq, ctx->stream);
  Scratch bbits(sizeof(unsigned long long) * nq, ctx->stream), bid(sizeof(int32_t) * nq, ctx->stream);
  Scratch cnt(sizeof(int32_t) * nq, ctx->stream), lost(sizeof(int32_t) * nq, ctx->stream);
  Scratch oU(sizeof(float) * no, ctx->stream), on(sizeof(int32_t) * no, ctx->stream);
  Scratch oids(sizeof(int32_t) * no * kList, ctx->stream), olb(sizeof(float) * no * kList, ctx->stream);
  Scratch sd2(sizeof(double) * no * kList, ctx->stream);
  Scratch ovc(sizeof(unsigned long long), ctx->stream), ovq(sizeof(int64_t) * ov_cap, ctx->stream);
  Scratch ovid(sizeof(int32_t) * ov_cap, ctx->stream), ovlb(sizeof(float) * ov_cap, ctx->stream);
  Scratch ovd2(sizeof(double) * ov_cap, ctx->stream);
  PSG_CUDA(cudaMemsetAsync(ovc.p, 0, sizeof(unsigned long long), ctx->stream));
  RowSrc qs = qsrc;
  qs.D = ix.D;
  launch_pack(ctx, qs, nq, qpad, ix.D, nch, kBM, ix.brute_mu, qop.as<float>(), qn2.as<float>(),
              qnup.as<float>());
  BruteArgs a{};
  a.qop = qop.as<float>();
  a.qn2 = qn2.as<float>();
  a.qnup = qnup.as<float>();
  a.qU0 = U0.as<float>();
  a.pop = ix.brute_op;
  a.pn2 = ix.brute_n2;
  a.pnup = ix.brute_nup;
  a.tmax = ix.brute_tmax;
  a.nq = nq;
  a.N = ix.N;
  a.nch = nch;
  a.ptiles = ix.brute_ptiles;
  a.splits = splits;
  a.D = ix.D;
  // |s - dist^2| <= c1 |q'||p'| + c2 (|q'| + |p'|)^2 with
  //   c1: tf32 round-to-nearest of both operands (2 * 2^-11 + 2^-22 per
  //       product), fp32 accumulation of Dpad terms (Dpad * 2^-23, truncating
  //       adds assumed), times 2 for the -2 q.p, +2^-22 for its rounding;
  //   c2: norms rounded to fp32, the norm sum and the fused epilogue
  //       (<= 4 * 2^-24) plus the centring subtractions (2^-23).
  // Both padded by 10 % and evaluated in fp32 with directed final rounding.
  const double dpad = (double)nch * kBK;
  const double c1 = (2.0 * (std::ldexp(1.0, -10) + std::ldexp(1.0, -22) + dpad * std::ldexp(1.0, -23)) +
                     std::ldexp(1.0, -22)) * 1.1;
  const double c2 = (4.0 * std::ldexp(1.0, -24) + std::ldexp(1.0, -23)) * 1.1 + 1e-9;
  a.c1 = (float)c1;
  a.c2 = (float)c2;
  a.qs = qs;
  a.ps = db_source(ix);
  a.o_U = oU.as<float>();
  a.o_n = on.as<int32_t>();
  a.o_ids = oids.as<int32_t>();
  a.o_lb = olb.as<float>();
  a.ov_count = ovc.as<unsigned long long>();
  a.ov_cap = ov_cap;
  a.ov_q = ovq.as<int64_t>();
  a.ov_id = ovid.as<int32_t>();
  a.ov_lb = ovlb.as<float>();
  a.lost = lost.as<int32_t>();
  const int64_t qblocks = std::min<int64_t>((nq + 127) / 128, (int64_t)ctx->num_sms * 16);
  brute_init_kernel<<<(int)qblocks, 128, 0, ctx->stream>>>(a, seed, sd.as<double>(), U0.as<float>(),
                                                           bbits.as<unsigned long long>(),
                                                           bid.as<int32_t>(), cnt.as<int32_t>());
  PSG_LAUNCHED(ctx);
  constexpr BruteSmem L = brute_smem();
  PSG_CUDA(cudaFuncSetAttribute(brute_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)L.total));
  brute_mma_kernel<<<dim3((unsigned)qtiles, (unsigned)splits), kThreads, L.total, ctx->stream>>>(a);
  PSG_LAUNCHED(ctx);
  // survivors: all list slots + the (normally empty) overflow buffer
  const int64_t sblocks = (int64_t)ctx->num_sms * 32;
  brute_settle_kernel<<<(int)sblocks, 256, 0, ctx->stream>>>(a, U0.as<float>(), sd2.as<double>(),
                                                            ovd2.as<double>(),
                                                            bbits.as<unsigned long long>(),
                                                            cnt.as<int32_t>());
  PSG_LAUNCHED(ctx);
  brute_tie_kernel<<<(int)sblocks, 256, 0, ctx->stream>>>(a, seed, sd.as<double>(), sd2.as<double>(),
                                                         ovd2.as<double>(),
                                                         bbits.as<unsigned long long>(),
                                                         bid.as<int32_t>());
  PSG_LAUNCHED(ctx);
  brute_pick_kernel<<<(int)qblocks, 128, 0, ctx->stream>>>(a, bbits.as<unsigned long long>(),
                                                           bid.as<int32_t>(), cnt.as<int32_t>(),
                                                           out_idx, out_d2, out_scanned, out_exact);
  PSG_LAUNCHED(ctx);
}

}  // namespace psg
