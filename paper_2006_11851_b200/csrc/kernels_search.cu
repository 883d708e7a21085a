// E-step kernels: window gather + exact fp64 PCA projection, exact k-means
// tree search with warp-cooperative leaf scans, and full-D rescoring.
//
// Reference semantics (paths under /root/reference/proj/core/src):
//   extract_window   neighborhood.cpp:120-137  fp32 = (float) fp64 state
//   PcaModel::project pca.cpp:27-41            acc += (v_j - mean_j) * b_kj, j asc
//   KmTree::query    km_tree.cpp:197-284       greedy / backtrack(m) / exact
//   scan_leaf        km_tree.cpp:128-139       lexicographic min (dist^2, id)
//   full_distance    optimizer.cpp:117-124     sqrt sum (a_j - b_j)^2, j asc
#include <cuda_runtime.h>
#include <float.h>

#include <cuda_bf16.h>
#include <cub/cub.cuh>

#include "numerics.cuh"
#include "psg_internal.h"

// d <= 32 tile kernel: 4 CTAs x 4 warps per SM = 16 warps, a 128-register cap
// (the bf16 stack bounds keep a 4-warp CTA under 48 KB of static shared
// memory).  Measured per search on the bench stage: 3 warps x 5 CTAs 1.78 ms
// (36 B spill), uncapped 165 registers at 4 x 3 warps 1.87 ms, 4 x 4 warps
// 1.71 ms.  Exact-recheck load batch in double2 (4 = 8 dims).
#ifndef TILE_MIN_CTAS
#define TILE_MIN_CTAS 4
#endif
#ifndef TILE64_MIN_CTAS
#define TILE64_MIN_CTAS 6  // d in (32, 64]: 6 CTAs x 2 warps (168 registers): cfg4 finest search 31 -> 27 ms
#endif
// leading PCA dims of the branch-free first filter phase (measured on the
// bench stage: 4 -> 1.41 ms, 8 -> 1.50, 12 -> 1.75)
#define P1_DIMS 4
// phase-1 chunk: 8 staged points (4: same speed, 16: 3% slower, 32 = the
// whole staging buffer: 6% slower -- short batches filtered stale rows)
#define P1_CHUNK 8
// image query tiles: kTW x kTH anchors per warp (lane = query).  Measured on
// the bench stage: 8 x 4 1.39 ms, 4 x 8 1.40, 16 x 2 1.46.
constexpr int kTW = 8, kTH = 32 / kTW;
// phase 2: the dims after the first DP / P2_SPLIT_DEN (difference form, then
// an early exit) in expanded form |q~|^2 + |p~|^2 - 2 q~.p~ (one FFMA2 per two
// dims; rounding covered by exp_slack).  Measured on the bench stage: all
// difference form 1.41 ms; split 16 | 16 1.39; 8 | 24 1.38; 4 | 28 1.58;
// all expanded (no early exit) 1.52.
#ifndef P2_SPLIT_DEN
#define P2_SPLIT_DEN 4
#endif
// dims in difference form: DP / P2_SPLIT_DEN rounded down to whole float4
// groups (the per-point half norms pp32.y use the same split)
__host__ __device__ constexpr int p2_split(int dp) { return (dp / P2_SPLIT_DEN) & ~3; }
#ifndef RECHECK_BATCH
#define RECHECK_BATCH 4
#endif

namespace psg {

// ----------------------------------------------------------------------------
// planes [C][H][W] fp64 -> mirror [H][W][C] fp32 (the layout the gathers read)
__global__ void make_mirror_kernel(const double* __restrict__ planes, int C, int64_t P,
                                   float* __restrict__ mirror) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < C; ++c) mirror[i * C + c] = (float)planes[c * P + i];
  }
}

// planes -> [H][W][8] fp32, channels zero-padded to 8 (32-byte pixels): the
// candidate side of the rescoring reads a window row as 16-byte vectors.
__global__ void make_mirror8_kernel(const double* __restrict__ planes, int C, int64_t P,
                                    float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = c < C ? (float)planes[c * P + i] : 0.f;
    float4* o = reinterpret_cast<float4*>(out + i * 8);
    o[0] = make_float4(v[0], v[1], v[2], v[3]);
    o[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

void launch_make_mirror8(psg_ctx* ctx, const double* planes, int C, int W, int H, float* out) {
  ProfScope _prof(ctx, K_MIRROR);
  const int64_t P = (int64_t)W * H;
  int blocks = (int)std::min<int64_t>((P + 255) / 256, (int64_t)ctx->num_sms * 16);
  make_mirror8_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(planes, C, P, out);
  PSG_LAUNCHED(ctx);
}

void launch_make_mirror(psg_ctx* ctx, const double* planes, int C, int W, int H, float* mirror) {
  ProfScope _prof(ctx, K_MIRROR);
  const int64_t P = (int64_t)W * H;
  const int threads = 256;
  int blocks = (int)((P + threads - 1) / threads);
  if (blocks > ctx->num_sms * 16) blocks = ctx->num_sms * 16;
  if (blocks < 1) blocks = 1;
  make_mirror_kernel<<<blocks, threads, 0, ctx->stream>>>(planes, C, P, mirror);
  PSG_LAUNCHED(ctx);
}

// ----------------------------------------------------------------------------
// Exact projection.  A CTA of 8 warps owns TQ = 8*RQ queries; lane owns
// components k = lane + 32*kk.  The feature axis j is walked in order in
// chunks of one window row (JC = w*C features) staged in shared memory:
//   cen[q][jj] = (double)v - mean[j]      (one rounding, as the reference)
//   bas[jj][k] = basis[k][j]              (from the transposed basis)
//   acc[q][k]  = acc + cen * bas          (separate mul + add, j ascending)
// Each (q, k) accumulator is a sequential chain, so the result is bit-equal
// to pca.cpp:35-38; parallelism comes from the Q x d independent chains.
template <int KPT, int RQ, bool kWindows>
__global__ void __launch_bounds__(256) project_kernel(
    const float* __restrict__ src, int img_w, int C, int w,  // windows: mirror image
    const int32_t* __restrict__ xs, const int32_t* __restrict__ ys, int nx,
    int64_t n, int D, int JC,                                // vectors: src = X[n][D]
    const double* __restrict__ mean, const double* __restrict__ basisT,  // [D][32*KPT]
    int d, double* __restrict__ out) {
  constexpr int KP = 32 * KPT;
  constexpr int TQ = 8 * RQ;
  extern __shared__ double smem[];
  const int JCp = JC | 1;  // odd stride: conflict-free per-q row fills
  double* cen = smem;               // [TQ][JCp]
  double* bas = smem + TQ * JCp;    // [JC][KP]
  __shared__ int64_t base_s[TQ];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t q0 = (int64_t)blockIdx.x * TQ;
  if (tid < TQ) {
    const int64_t qi = q0 + tid;
    int64_t b = -1;
    if (qi < n) {
      if (kWindows) {
        const int ax = xs[qi % nx], ay = ys[qi / nx];
        b = ((int64_t)ay * img_w + ax) * C;
      } else {
        b = qi * (int64_t)D;
      }
    }
    base_s[tid] = b;
  }

  double acc[RQ][KPT];
#pragma unroll
  for (int r = 0; r < RQ; ++r)
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk) acc[r][kk] = 0.0;

  const int n_chunks = (D + JC - 1) / JC;
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int j0 = ch * JC;
    const int jc = min(JC, D - j0);
    // windows: chunk j0 is window row j0 / R at offset j0 % R (R = w * C)
    const int64_t roff = kWindows ? (int64_t)(j0 / (w * C)) * img_w * C + j0 % (w * C) : 0;
    __syncthreads();
    for (int f = tid; f < TQ * jc; f += 256) {
      const int q = f / jc, jj = f - q * jc;
      const int64_t b = base_s[q];
      double v = 0.0;
      if (b >= 0) {
        float x;
        if (kWindows) {
          // window row ch (= dy) of anchor q: contiguous w*C floats
          x = src[b + roff + jj];
        } else {
          x = src[b + j0 + jj];
        }
        v = dsub((double)x, mean[j0 + jj]);
      }
      cen[q * JCp + jj] = v;
    }
    for (int f = tid; f < jc * KP; f += 256) bas[f] = basisT[(int64_t)j0 * KP + f];
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < jc; ++jj) {
      double b[KPT];
#pragma unroll
      for (int kk = 0; kk < KPT; ++kk) b[kk] = bas[jj * KP + lane + 32 * kk];
#pragma unroll
      for (int r = 0; r < RQ; ++r) {
        const double c = cen[(warp * RQ + r) * JCp + jj];
#pragma unroll
        for (int kk = 0; kk < KPT; ++kk) acc[r][kk] = dadd(acc[r][kk], dmul(c, b[kk]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RQ; ++r) {
    const int64_t qi = q0 + warp * RQ + r;
    if (qi >= n) continue;
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk) {
      const int k = lane + 32 * kk;
      if (k < d) out[qi * d + k] = acc[r][kk];
    }
  }
}

// d <= 32: lane = (anchor group g2, k pair kp): each thread accumulates 2
// consecutive k for RQ anchors, so one double2 basis load and RQ broadcast
// double2 loads of the centred window feed 4 * RQ fp64 ops per 2 j (the
// per-(anchor, k) order over j is unchanged: bit-identical to project_kernel).
template <int RQ, bool kWindows, int JCT>
__global__ void __launch_bounds__(256, 3) project2_kernel(
    const float* __restrict__ src, int img_w, int C, int w, const int32_t* __restrict__ xs,
    const int32_t* __restrict__ ys, int nx, int64_t n, int D, int JC_,
    const double* __restrict__ mean, const double* __restrict__ basisT,  // [D][32]
    int d, double* __restrict__ out) {
  constexpr int TQ = 8 * 2 * RQ;  // anchors per block: 8 warps x 2 groups x RQ
  const int JC = JCT > 0 ? JCT : JC_;  // JCT > 0: window chunks are always full (JC | w*C)
  extern __shared__ __align__(16) double smem2[];
  const int JCp = JC + 2;  // even (double2 aligned), breaks the power-of-two stride
  double* cen = smem2;             // [TQ][JCp]
  double* bas = smem2 + TQ * JCp;  // [JC][32]
  __shared__ int64_t base_s[TQ];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g2 = lane >> 4, kp = lane & 15;
  const int64_t q0 = (int64_t)blockIdx.x * TQ;
  if (tid < TQ) {
    const int64_t qi = q0 + tid;
    int64_t b = -1;
    if (qi < n) {
      if (kWindows) {
        const int ax = xs[qi % nx], ay = ys[qi / nx];
        b = ((int64_t)ay * img_w + ax) * C;
      } else {
        b = qi * (int64_t)D;
      }
    }
    base_s[tid] = b;
  }
  double acc0[RQ], acc1[RQ];
#pragma unroll
  for (int r = 0; r < RQ; ++r) acc0[r] = acc1[r] = 0.0;
  const int qb = (warp * 2 + g2) * RQ;  // first anchor (block-local) of this thread
  const int n_chunks = (D + JC - 1) / JC;
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int j0 = ch * JC;
    const int jc = JCT > 0 ? JCT : min(JC, D - j0);
    // windows: chunk j0 is window row j0 / R at offset j0 % R (R = w * C)
    const int64_t roff = kWindows ? (int64_t)(j0 / (w * C)) * img_w * C + j0 % (w * C) : 0;
    __syncthreads();
    if constexpr (JCT > 0) {
      // fixed trip count: loads batched 4 deep (one latency per 4 elements)
      constexpr int PER = (TQ * JCT + 255) / 256, H = 4;
#pragma unroll
      for (int h = 0; h < PER; h += H) {
        float xv[H];
        double mv[H];
#pragma unroll
        for (int k = 0; k < H; ++k) {
          const int f = tid + 256 * (h + k);
          const int q = f / JCT, jj = f - q * JCT;
          xv[k] = 0.f;
          mv[k] = 0.0;
          if (h + k < PER && f < TQ * JCT && base_s[q] >= 0) {
            xv[k] = __ldg(src + base_s[q] + roff + jj);
            mv[k] = __ldg(mean + j0 + jj);
          }
        }
#pragma unroll
        for (int k = 0; k < H; ++k) {
          const int f = tid + 256 * (h + k);
          const int q = f / JCT, jj = f - q * JCT;
          if (h + k < PER && f < TQ * JCT)
            cen[q * JCp + jj] = base_s[q] >= 0 ? dsub((double)xv[k], mv[k]) : 0.0;
        }
      }
    } else {
      for (int f = tid; f < TQ * jc; f += 256) {
        const int q = f / jc, jj = f - q * jc;
        const int64_t b = base_s[q];
        double v = 0.0;
        if (b >= 0) {
          const float x = kWindows ? src[b + roff + jj] : src[b + j0 + jj];
          v = dsub((double)x, mean[j0 + jj]);
        }
        cen[q * JCp + jj] = v;
      }
    }
    if (jc & 1)  // odd chunk: zero pad column so the double2 loop can read it
      for (int q = tid; q < TQ; q += 256) cen[q * JCp + jc] = 0.0;
    for (int f = tid; f < jc * 32; f += 256) bas[f] = basisT[(int64_t)j0 * 32 + f];
    if (jc & 1)
      for (int f = tid; f < 32; f += 256) bas[jc * 32 + f] = 0.0;
    __syncthreads();
    const int jc2 = jc & ~1;
#pragma unroll 2
    for (int jj = 0; jj < jc2; jj += 2) {
      const double2 b0 = *reinterpret_cast<const double2*>(bas + jj * 32 + 2 * kp);
      const double2 b1 = *reinterpret_cast<const double2*>(bas + (jj + 1) * 32 + 2 * kp);
#pragma unroll
      for (int r = 0; r < RQ; ++r) {
        const double2 c = *reinterpret_cast<const double2*>(cen + (qb + r) * JCp + jj);
        acc0[r] = dadd(acc0[r], dmul(c.x, b0.x));
        acc1[r] = dadd(acc1[r], dmul(c.x, b0.y));
        acc0[r] = dadd(acc0[r], dmul(c.y, b1.x));
        acc1[r] = dadd(acc1[r], dmul(c.y, b1.y));
      }
    }
    if (jc & 1) {  // last odd column
      const int jj = jc - 1;
      const double2 b0 = *reinterpret_cast<const double2*>(bas + jj * 32 + 2 * kp);
#pragma unroll
      for (int r = 0; r < RQ; ++r) {
        const double c = cen[(qb + r) * JCp + jj];
        acc0[r] = dadd(acc0[r], dmul(c, b0.x));
        acc1[r] = dadd(acc1[r], dmul(c, b0.y));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RQ; ++r) {
    const int64_t qi = q0 + qb + r;
    if (qi >= n) continue;
    if (2 * kp < d) out[qi * d + 2 * kp] = acc0[r];
    if (2 * kp + 1 < d) out[qi * d + 2 * kp + 1] = acc1[r];
  }
}

// 32 < d <= 48 (cfg4: d = 48) windows: lane (g2, kp) accumulates THREE
// consecutive k (3 kp .. 3 kp + 2) for RQ anchors, so 16 lanes cover 48
// components (the KPT = 2 kernel leaves 16 of its 64 lanes idle at d = 48).
// Same per-(anchor, k) j-sequential chains: bit-identical.  basisT is
// [D][64] (zero-padded).
template <int RQ, int JCT>
__global__ void __launch_bounds__(256, 2) project48_kernel(
    const float* __restrict__ src, int img_w, int C, int w, const int32_t* __restrict__ xs,
    const int32_t* __restrict__ ys, int nx, int64_t n, int D,
    const double* __restrict__ mean, const double* __restrict__ basisT,  // [D][64]
    int d, double* __restrict__ out) {
  constexpr int TQ = 8 * 2 * RQ, JC = JCT, JCp = JC + 2, BS = 64;
  extern __shared__ __align__(16) double smem48[];
  double* cen = smem48;             // [TQ][JCp]
  double* bas = smem48 + TQ * JCp;  // [JC][64]
  __shared__ int64_t base_s[TQ];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g2 = lane >> 4, kp = lane & 15;
  const int64_t q0 = (int64_t)blockIdx.x * TQ;
  if (tid < TQ) {
    const int64_t qi = q0 + tid;
    int64_t b = -1;
    if (qi < n) b = ((int64_t)ys[qi / nx] * img_w + xs[qi % nx]) * C;
    base_s[tid] = b;
  }
  double acc[3][RQ];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int r = 0; r < RQ; ++r) acc[i][r] = 0.0;
  const int qb = (warp * 2 + g2) * RQ;
  const int n_chunks = D / JC;  // JC | w * C
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int j0 = ch * JC;
    const int64_t roff = (int64_t)(j0 / (w * C)) * img_w * C + j0 % (w * C);
    __syncthreads();
    constexpr int PER = (TQ * JC + 255) / 256, H = 4;
#pragma unroll
    for (int h = 0; h < PER; h += H) {
      float xv[H];
      double mv[H];
#pragma unroll
      for (int k = 0; k < H; ++k) {
        const int f = tid + 256 * (h + k);
        const int q = f / JC, jj = f - q * JC;
        xv[k] = 0.f;
        mv[k] = 0.0;
        if (h + k < PER && f < TQ * JC && base_s[q] >= 0) {
          xv[k] = __ldg(src + base_s[q] + roff + jj);
          mv[k] = __ldg(mean + j0 + jj);
        }
      }
#pragma unroll
      for (int k = 0; k < H; ++k) {
        const int f = tid + 256 * (h + k);
        const int q = f / JC, jj = f - q * JC;
        if (h + k < PER && f < TQ * JC)
          cen[q * JCp + jj] = base_s[q] >= 0 ? dsub((double)xv[k], mv[k]) : 0.0;
      }
    }
    for (int f = tid; f < JC * BS / 2; f += 256)
      reinterpret_cast<double2*>(bas)[f] =
          __ldg(reinterpret_cast<const double2*>(basisT + (int64_t)j0 * BS) + f);
    __syncthreads();
#pragma unroll 2
    for (int jj = 0; jj < JC; jj += 2) {
      double b0[3], b1[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        b0[i] = bas[jj * BS + 3 * kp + i];
        b1[i] = bas[(jj + 1) * BS + 3 * kp + i];
      }
#pragma unroll
      for (int r = 0; r < RQ; ++r) {
        const double2 c = *reinterpret_cast<const double2*>(cen + (qb + r) * JCp + jj);
#pragma unroll
        for (int i = 0; i < 3; ++i) acc[i][r] = dadd(acc[i][r], dmul(c.x, b0[i]));
#pragma unroll
        for (int i = 0; i < 3; ++i) acc[i][r] = dadd(acc[i][r], dmul(c.y, b1[i]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RQ; ++r) {
    const int64_t qi = q0 + qb + r;
    if (qi >= n) continue;
#pragma unroll
    for (int i = 0; i < 3; ++i)
      if (3 * kp + i < d) out[qi * d + 3 * kp + i] = acc[i][r];
  }
}

template <bool kWindows>
static void launch_project(psg_ctx* ctx, const float* src, int img_w, int C, int w,
                           const int32_t* xs, const int32_t* ys, int nx, int64_t n, int D, int JC,
                           const double* mean, const double* basisT, int d, double* out) {
  ProfScope _prof(ctx, K_PROJECT);
  if (n <= 0 || d <= 0) return;
  constexpr int RQ = 8;
  const int TQ = 8 * RQ;
  const int JCp = JC | 1;
  const int blocks = (int)((n + TQ - 1) / TQ);
  if (d <= 32 && kWindows && (JC == 32 || JC == 40)) {
    // compile-time chunk width: immediate shared-memory offsets in the
    // multiply loop, multiply-shift staging indices
    constexpr int TQ2 = 8 * 2 * RQ;
    const size_t sm = sizeof(double) * ((size_t)TQ2 * (JC + 2) + (size_t)(JC + 1) * 32);
    auto k = JC == 32 ? project2_kernel<RQ, kWindows, 32> : project2_kernel<RQ, kWindows, 40>;
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int blocks2 = (int)((n + TQ2 - 1) / TQ2);
    k<<<blocks2, 256, sm, ctx->stream>>>(src, img_w, C, w, xs, ys, nx, n, D, JC, mean, basisT, d,
                                          out);
  } else if (d <= 32) {
    constexpr int TQ2 = 8 * 2 * RQ;
    const size_t sm = sizeof(double) * ((size_t)TQ2 * (JC + 2) + (size_t)(JC + 1) * 32);
    auto k = project2_kernel<RQ, kWindows, 0>;
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int blocks2 = (int)((n + TQ2 - 1) / TQ2);
    k<<<blocks2, 256, sm, ctx->stream>>>(src, img_w, C, w, xs, ys, nx, n, D, JC, mean, basisT, d,
                                          out);
  } else if (d <= 48 && kWindows && (JC == 32 || JC == 40) && !ctx->knobs.project_kpt2) {
    constexpr int TQ2 = 8 * 2 * RQ;
    const size_t sm = sizeof(double) * ((size_t)TQ2 * (JC + 2) + (size_t)JC * 64);
    auto k = JC == 32 ? project48_kernel<RQ, 32> : project48_kernel<RQ, 40>;
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int blocks2 = (int)((n + TQ2 - 1) / TQ2);
    k<<<blocks2, 256, sm, ctx->stream>>>(src, img_w, C, w, xs, ys, nx, n, D, mean, basisT, d, out);
  } else if (d <= 64) {
    const size_t sm = sizeof(double) * ((size_t)TQ * JCp + (size_t)JC * 64);
    auto k = project_kernel<2, RQ, kWindows>;
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k<<<blocks, 256, sm, ctx->stream>>>(src, img_w, C, w, xs, ys, nx, n, D, JC, mean, basisT, d,
                                         out);
  } else if (d <= kMaxDP) {
    const size_t sm = sizeof(double) * ((size_t)TQ * JCp + (size_t)JC * 128);
    auto k = project_kernel<4, RQ, kWindows>;
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k<<<blocks, 256, sm, ctx->stream>>>(src, img_w, C, w, xs, ys, nx, n, D, JC, mean, basisT, d,
                                         out);
  } else {
    fail(PSG_E_DOMAIN, "retained PCA dimension > 128 is not supported");
  }
  PSG_LAUNCHED(ctx);
}

void launch_project_windows(psg_ctx* ctx, const float* mirror, int img_w, int C, int w,
                            AnchorSet anchors, const double* mean, const double* basisT, int d,
                            double* out) {
  // chunk = the largest divisor of a window row (w * C floats) <= 48 (bounded
  // shared memory; chunk j0 is row j0 / R, offset j0 % R)
  const int R = w * C;
  int JC = 1;
  for (int c = 1; c <= 48 && c <= R; ++c)  // small chunks: several blocks per SM
    if (R % c == 0) JC = c;
  launch_project<true>(ctx, mirror, img_w, C, w, anchors.xs, anchors.ys, anchors.nx,
                       anchors.count, w * w * C, JC, mean, basisT, d, out);
}

void launch_project_vectors(psg_ctx* ctx, const float* X, int64_t n, int D, const double* mean,
                            const double* basisT, int d, double* out) {
  const int JC = D < 128 ? D : 128;
  launch_project<false>(ctx, X, 0, 0, 0, nullptr, nullptr, 1, n, D, JC, mean, basisT, d, out);
}

// ----------------------------------------------------------------------------
// Tree search: one warp per query (persistent grid-stride over queries).
constexpr int kSearchWarps = 4;
#ifndef PSG_KSTACK
#define PSG_KSTACK 512
#endif
constexpr int kStack = PSG_KSTACK;  // warp-per-query kernel (deep imported trees, backtrack frontier; spills to global scratch)
constexpr int kStackX = 256;  // search_exact_kernel
constexpr int kMaxD = kMaxDP;  // the warp kernels; the tile kernel takes d <= 64

struct WarpLexMin {
  double d2;
  int32_t id;
};

__device__ __forceinline__ bool lex_less(double a, int32_t ia, double b, int32_t ib) {
  return a < b || (a == b && ia < ib);
}

__device__ __forceinline__ WarpLexMin warp_lexmin(double d2, int32_t id) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, d2, off);
    const int32_t oi = __shfl_xor_sync(0xffffffffu, id, off);
    if (lex_less(od, oi, d2, id)) {
      d2 = od;
      id = oi;
    }
  }
  return {d2, id};
}

// dist^2 to a centroid, j ascending (km_tree.cpp:15-22) — the reference's
// exact key for greedy/backtrack ordering.
__device__ __forceinline__ double dist2_seq(const double* __restrict__ q,
                                            const double* __restrict__ p, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = dsub(q[j], p[j]);
    acc = dadd(acc, dmul(t, t));
  }
  return acc;
}

// Out-of-line copy for rarely executed call sites (seeds, filter survivors):
// keeps the hot loops of the tile kernel small enough for the I-cache.
// Loads are issued 8 at a time (16-byte vectors when the rows are 16-byte
// aligned) ahead of the sequential chain: one memory latency per 8 dims
// instead of one per dim.  Same j-ascending sub, mul, add.
constexpr int kRB = RECHECK_BATCH;  // double2 per batch
__device__ __noinline__ double dist2_seq_cold(const double* __restrict__ q,
                                             const double* __restrict__ p, int d) {
  double acc = 0.0;
  int j = 0;
  if (((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(p)) & 15) == 0) {
    for (; j + 2 * kRB <= d; j += 2 * kRB) {
      double2 qv[kRB], pv[kRB];
#pragma unroll
      for (int u = 0; u < kRB; ++u) {
        qv[u] = __ldg(reinterpret_cast<const double2*>(q + j) + u);
        pv[u] = __ldg(reinterpret_cast<const double2*>(p + j) + u);
      }
#pragma unroll
      for (int u = 0; u < kRB; ++u) {
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

// Scan one leaf: lanes over points, exact dist^2 per lane, warp lexmin.
__device__ __forceinline__ void scan_leaf(const SearchArgs& a, const double* __restrict__ qs,
                                          int node, int lane, double& best, int32_t& best_id,
                                          int64_t& scanned) {
  const int32_t s = a.tree.leaf_start[node];
  const int32_t cnt = a.tree.leaf_count[node];
  for (int base = 0; base < cnt; base += 32) {
    const int i = base + lane;
    double d2 = DBL_MAX * 2;  // +inf
    int32_t id = 0x7fffffff;
    if (i < cnt) {
      const int64_t pos = (int64_t)s + i;
      id = a.perm[pos];
      double acc = 0.0;
      const double* col = a.proj_soa + pos;
      for (int j = 0; j < a.d; ++j) {
        const double t = dsub(qs[j], col[(int64_t)j * a.N]);
        acc = dadd(acc, dmul(t, t));
      }
      d2 = acc;
    }
    const WarpLexMin m = warp_lexmin(d2, id);
    if (lex_less(m.d2, m.id, best, best_id)) {
      best = m.d2;
      best_id = m.id;
    }
  }
  scanned += cnt;
}

// Greedy / backtrack(m) with one thread per query (km_tree.cpp:213-250): the
// reference's fp64 keys dist^2(q, centroid) (j ascending), best-first frontier
// as a binary min-heap on (key, tie id) in thread-local memory, leaves scanned
// with the exact fp64 chain against the row-major projected database;
// lexicographic (dist^2, id) minimum (km_tree.cpp:134).  Budget queries touch
// ~m leaves, so a query per thread keeps every lane busy (the warp-per-query
// search_kernel leaves most lanes idle on ~15-point leaves).
constexpr int kHeapCap = 384;

template <int DP>
__global__ void __launch_bounds__(128) search_budget_kernel(SearchArgs a) {
  const int d = a.d;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    double qs[DP];
#pragma unroll
    for (int j = 0; j < DP; ++j) qs[j] = j < d ? a.q[q * d + j] : 0.0;
    auto key_of = [&](int node) {
      const double* c = a.tree.centroid + (int64_t)node * d;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < DP; ++j)
        if (j < d) {
          const double t = dsub(qs[j], c[j]);
          acc = dadd(acc, dmul(t, t));
        }
      return acc;
    };
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int32_t best_id = 0x7fffffff;
    int64_t scanned = 0;
    int32_t visited = 0;
    auto scan = [&](int node) {
      const int32_t s0 = a.tree.leaf_start[node], cnt = a.tree.leaf_count[node];
      for (int i = 0; i < cnt; ++i) {
        const int32_t id = a.perm[s0 + i];
        const double* p = a.proj + (int64_t)id * d;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < DP; ++j)
          if (j < d) {
            const double t = dsub(qs[j], p[j]);
            acc = dadd(acc, dmul(t, t));
          }
        if (acc < best || (acc == best && id < best_id)) {
          best = acc;
          best_id = id;
        }
      }
      scanned += cnt;
    };
    if (a.mode == PSG_GREEDY) {
      int node = 0;
      ++visited;
      while (a.tree.n_children[node] > 0) {
        const int fc = a.tree.first_child[node], nc = a.tree.n_children[node];
        double bd = __longlong_as_double(0x7ff0000000000000ll);
        int next = fc;
        for (int c = 0; c < nc; ++c) {
          const double k = key_of(fc + c);
          if (k < bd) {  // strict: the first child in order wins ties
            bd = k;
            next = fc + c;
          }
        }
        node = next;
        ++visited;
      }
      scan(node);
    } else {
      double hk[kHeapCap];
      int32_t hn[kHeapCap], ht[kHeapCap];
      int size = 0;
      auto less = [](const double* k, const int32_t* t, int i, int j) {
        return k[i] < k[j] || (k[i] == k[j] && t[i] < t[j]);
      };
      auto push = [&](double k, int32_t node) {
        if (size == kHeapCap) {
          atomicOr(a.flags, FLAG_STACK_OVERFLOW);
          return;
        }
        int i = size++;
        hk[i] = k;
        hn[i] = node;
        ht[i] = a.tree.tie ? a.tree.tie[node] : node;
        while (i > 0) {
          const int par = (i - 1) >> 1;
          if (!less(hk, ht, i, par)) break;
          const double tk = hk[i];
          hk[i] = hk[par];
          hk[par] = tk;
          const int32_t tn = hn[i];
          hn[i] = hn[par];
          hn[par] = tn;
          const int32_t tt = ht[i];
          ht[i] = ht[par];
          ht[par] = tt;
          i = par;
        }
      };
      push(0.0, 0);
      int leaves = 0;
      while (size > 0 && leaves < a.max_leaves) {
        const int node = hn[0];
        --size;
        hk[0] = hk[size];
        hn[0] = hn[size];
        ht[0] = ht[size];
        for (int i = 0;;) {  // sift down
          const int l = 2 * i + 1, r = l + 1;
          int m = i;
          if (l < size && less(hk, ht, l, m)) m = l;
          if (r < size && less(hk, ht, r, m)) m = r;
          if (m == i) break;
          const double tk = hk[i];
          hk[i] = hk[m];
          hk[m] = tk;
          const int32_t tn = hn[i];
          hn[i] = hn[m];
          hn[m] = tn;
          const int32_t tt = ht[i];
          ht[i] = ht[m];
          ht[m] = tt;
          i = m;
        }
        ++visited;
        const int nc = a.tree.n_children[node];
        if (nc == 0) {
          scan(node);
          ++leaves;
        } else {
          const int fc = a.tree.first_child[node];
          for (int c = 0; c < nc; ++c) push(key_of(fc + c), fc + c);
        }
      }
    }
    a.out_idx[q] = best_id;
    a.out_d2[q] = best;
    if (a.out_scanned) a.out_scanned[q] = scanned;
    if (a.out_exact) a.out_exact[q] = scanned;
    if (a.out_visited) a.out_visited[q] = visited;
  }
}

__global__ void __launch_bounds__(32 * kSearchWarps) search_kernel(SearchArgs a) {
  __shared__ double qs_all[kSearchWarps][kMaxD];
  __shared__ int32_t st_node[kSearchWarps][kStack];
  __shared__ double st_key[kSearchWarps][kStack];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* qs = qs_all[warp];
  int32_t* sn = st_node[warp];
  double* sk = st_key[warp];
  const int d = a.d;

  const int64_t nlist = a.ovf_list ? (int64_t)*a.ovf_count : a.nq;
  for (int64_t i = (int64_t)blockIdx.x * kSearchWarps + warp; i < nlist;
       i += (int64_t)gridDim.x * kSearchWarps) {
    const int64_t q = a.ovf_list ? (int64_t)a.ovf_list[i] : i;  // list mode: the pool overflows
    for (int j = lane; j < d; j += 32) qs[j] = a.q[q * d + j];
    __syncwarp();
    double best = DBL_MAX * 2;
    int32_t best_id = 0x7fffffff;
    int64_t scanned = 0;
    if (a.seed_idx) {
      const int32_t pid = a.seed_idx[q];
      double d2 = 0.0;
      if (lane == 0) d2 = dist2_seq(qs, a.proj + (int64_t)pid * d, d);
      best = __shfl_sync(0xffffffffu, d2, 0);
      best_id = pid;
      scanned += 1;
    }

    if (a.mode == PSG_EXACT) {
      int top = 0;
      if (lane == 0) {
        sn[0] = 0;  // root is node 0 (breadth-first layout)
        sk[0] = 0.0;
      }
      top = 1;
      __syncwarp();
      while (top > 0) {
        --top;
        const int node = sn[top];
        const double key = sk[top];
        __syncwarp();
        if (key > best) continue;  // km_tree.cpp:265 prune
        const int nc = a.tree.n_children[node];
        if (nc == 0) {
          scan_leaf(a, qs, node, lane, best, best_id, scanned);
          continue;
        }
        const int fc = a.tree.first_child[node];
        for (int cb = 0; cb < nc; cb += 32) {
          const int c = cb + lane;
          double lb2 = DBL_MAX * 2;
          bool keep = false;
          if (c < nc) {
            const int cid = fc + c;
            // lower_bound2 (km_tree.cpp:255-260): (|q-c| - radius - slack)+^2
            const double dc = sqrt(dist2_seq(qs, a.tree.centroid + (int64_t)cid * d, d));
            const double rad = a.tree.radius[cid];
            const double slack = 1e-9 * (1.0 + dc + rad);
            const double lb = dc - rad - slack;
            lb2 = lb > 0.0 ? lb * lb : 0.0;
            keep = lb2 <= best;
          }
          const unsigned km = __ballot_sync(0xffffffffu, keep);
          const int nkeep = __popc(km);
          // rank among kept children by (lb2, child) ascending
          int rank = 0;
          for (int o = 0; o < 32; ++o) {
            const double ol = __shfl_sync(0xffffffffu, lb2, o);
            if (((km >> o) & 1u) && (ol < lb2 || (ol == lb2 && o < lane))) ++rank;
          }
          if (top + nkeep > kStack) {
            if (lane == 0) atomicOr(a.flags, FLAG_STACK_OVERFLOW);
            break;
          }
          if (keep) {
            const int slot = top + nkeep - 1 - rank;  // nearest popped first
            sn[slot] = fc + c;
            sk[slot] = lb2;
          }
          top += nkeep;
          __syncwarp();
        }
      }
    } else if (a.mode == PSG_GREEDY) {
      // km_tree.cpp:213-231: descend to the nearest child (strict <, lowest wins)
      int node = 0;
      int nc = a.tree.n_children[node];
      while (nc > 0) {
        const int fc = a.tree.first_child[node];
        double bd = DBL_MAX * 2;
        int32_t bi = 0x7fffffff;
        for (int cb = 0; cb < nc; cb += 32) {
          const int c = cb + lane;
          double dc2 = DBL_MAX * 2;
          if (c < nc) dc2 = dist2_seq(qs, a.tree.centroid + (int64_t)(fc + c) * d, d);
          const WarpLexMin m = warp_lexmin(dc2, c < nc ? c : 0x7fffffff);
          if (lex_less(m.d2, m.id, bd, bi)) {
            bd = m.d2;
            bi = m.id;
          }
        }
        node = fc + bi;
        nc = a.tree.n_children[node];
      }
      scan_leaf(a, qs, node, lane, best, best_id, scanned);
    } else {
      // backtrack(m), km_tree.cpp:232-250: best-first on (dist^2 to centroid,
      // node id); frontier kept as an unsorted pool, min found by the warp.
      // The node id of the tie-break is the tree's tie id (the reference's
      // post-order id for an imported tree, km_tree.cpp:159,187-188).
      int size = 1, cap = kStack;
      sn = st_node[warp];  // (a previous query may have moved its frontier to the global scratch)
      sk = st_key[warp];
      if (lane == 0) {
        sn[0] = 0;
        sk[0] = 0.0;
      }
      __syncwarp();
      int leaves = 0;
      while (size > 0 && leaves < a.max_leaves) {
        double bk = DBL_MAX * 2;
        int32_t bn = 0x7fffffff;
        int bslot = -1;
        for (int s0 = 0; s0 < size; s0 += 32) {
          const int s = s0 + lane;
          double k = DBL_MAX * 2;
          int32_t nid = 0x7fffffff;
          if (s < size) {
            k = sk[s];
            nid = a.tree.tie ? a.tree.tie[sn[s]] : sn[s];
          }
          const WarpLexMin m = warp_lexmin(k, nid);
          if (lex_less(m.d2, m.id, bk, bn)) {
            bk = m.d2;
            bn = m.id;
          }
        }
        // locate the slot of the winner and remove it (swap with last)
        for (int s0 = 0; s0 < size; s0 += 32) {
          const int s = s0 + lane;
          const bool hit =
              s < size && sk[s] == bk && (a.tree.tie ? a.tree.tie[sn[s]] : sn[s]) == bn;
          const unsigned hm = __ballot_sync(0xffffffffu, hit);
          if (hm && bslot < 0) bslot = s0 + __ffs(hm) - 1;
        }
        const int node = sn[bslot];
        __syncwarp();
        if (lane == 0) {
          sn[bslot] = sn[size - 1];
          sk[bslot] = sk[size - 1];
        }
        --size;
        __syncwarp();
        const int nc = a.tree.n_children[node];
        if (nc == 0) {
          scan_leaf(a, qs, node, lane, best, best_id, scanned);
          ++leaves;
        } else {
          const int fc = a.tree.first_child[node];
          if (size + nc > cap) {
            // frontier past the shared-memory pool: move it to this warp's
            // global scratch (the reference's priority queue is unbounded,
            // km_tree.cpp:206-208) and go on there
            if (cap == kStack && a.deep_key && size + nc <= a.deep_cap) {
              const int64_t w0 = ((int64_t)blockIdx.x * kSearchWarps + warp) * a.deep_cap;
              double* gk = a.deep_key + w0;
              int32_t* gn = a.deep_node + w0;
              for (int s = lane; s < size; s += 32) {
                gk[s] = sk[s];
                gn[s] = sn[s];
              }
              __syncwarp();
              sk = gk;
              sn = gn;
              cap = a.deep_cap;
            } else {
              if (lane == 0) atomicOr(a.flags, FLAG_STACK_OVERFLOW);
              break;
            }
          }
          for (int cb = 0; cb < nc; cb += 32) {
            const int c = cb + lane;
            if (c < nc) {
              sn[size + c] = fc + c;
              sk[size + c] = dist2_seq(qs, a.tree.centroid + (int64_t)(fc + c) * d, d);
            }
          }
          size += nc;
          __syncwarp();
        }
      }
    }
    if (lane == 0) {
      // a listed query of a mapped re-run: results go to its output slot
      const int64_t o = (a.ovf_list && a.out_map) ? (int64_t)a.out_map[q] : q;
      a.out_idx[o] = best_id;
      if (a.out_d2) a.out_d2[o] = best;
      if (a.out_scanned) a.out_scanned[o] = scanned;
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// backtrack(m) with one warp per query (km_tree.cpp:232-250), m > 2: the
// best-first frontier is an unsorted pool in shared memory holding (key,
// node, tie id, node meta); a pop is one warp-wide lexicographic min over
// (key, tie) carrying the slot, and the popped entry already holds the node's
// children range or leaf range (no dependent metadata load).  An expansion
// stages the children's centroid rows (contiguous in the breadth-first
// layout), metas and tie ids with one round of independent coalesced loads;
// lane c forms child c's key dist^2(q, centroid) with the reference's
// j-ascending fp64 chain from shared memory.  A leaf stages its points
// (leaf-ordered [d][N] columns) the same way and lane i scans point i
// (lexicographic (dist^2, id) minimum, km_tree.cpp:128-139).
constexpr int kBtWarps = 4, kBtCap = 192;

template <int DP>
__global__ void __launch_bounds__(32 * kBtWarps) search_backtrack_kernel(SearchArgs a) {
  constexpr int CH = 8;  // rows staged per round (children or leaf points)
  __shared__ double qs_all[kBtWarps][DP];
  __shared__ double pk_all[kBtWarps][kBtCap];
  __shared__ int4 pn_all[kBtWarps][kBtCap];  // (node, tie id, meta.x, meta.y)
  // rows padded to an odd number of doubles: lane r reading row r, dim j is
  // free of bank conflicts (a DP-double stride put 16 lanes on one bank)
  constexpr int RP = DP + 1;
  __shared__ double cs_all[kBtWarps][CH][RP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* qs = qs_all[warp];
  double* pk = pk_all[warp];
  int4* pn = pn_all[warp];
  double(*cs)[RP] = cs_all[warp];
  const int d = a.d;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const int2 root = a.tree.meta[0];
  const int32_t root_tie = a.tree.tie ? a.tree.tie[0] : 0;
  // dims d..DP-1 are zero on both sides: their terms add an exact +0.0 to a
  // non-negative accumulator, so the full DP-step chain equals the d-step one
  auto chain = [&](const double* r) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      const double t = dsub(qs[j], r[j]);
      acc = dadd(acc, dmul(t, t));
    }
    return acc;
  };
  for (int64_t q = (int64_t)blockIdx.x * kBtWarps + warp; q < a.nq;
       q += (int64_t)gridDim.x * kBtWarps) {
    for (int j = lane; j < DP; j += 32) qs[j] = j < d ? a.q[q * d + j] : 0.0;
    if (lane == 0) {
      pk[0] = 0.0;
      pn[0] = make_int4(0, root_tie, root.x, root.y);
    }
    __syncwarp();
    double best = kInf;
    int32_t best_id = 0x7fffffff;
    int64_t scanned = 0;
    int32_t visited = 0;
    int size = 1, leaves = 0;
    bool overflow = false;
    while (size > 0 && leaves < a.max_leaves) {
      // pop the lexicographic minimum (key, tie)
      double bk = kInf;
      int32_t bt = 0x7fffffff, bs = -1;
      for (int s0 = lane; s0 < size; s0 += 32) {
        const double k = pk[s0];
        const int32_t t = pn[s0].y;
        if (k < bk || (k == bk && t < bt)) {
          bk = k;
          bt = t;
          bs = s0;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, bk, off);
        const int32_t ot = __shfl_xor_sync(0xffffffffu, bt, off);
        const int32_t os = __shfl_xor_sync(0xffffffffu, bs, off);
        if (ok < bk || (ok == bk && ot < bt)) {
          bk = ok;
          bt = ot;
          bs = os;
        }
      }
      const int4 e = pn[bs];
      __syncwarp();
      if (lane == 0) {
        pk[bs] = pk[size - 1];
        pn[bs] = pn[size - 1];
      }
      --size;
      ++visited;
      __syncwarp();
      if (e.w >= 0) {  // leaf: points [e.z, e.z + e.w) of the leaf order
        for (int base = 0; base < e.w; base += CH) {
          const int cn = min(CH, e.w - base);
          const int64_t p0 = (int64_t)e.z + base;
          // the leaf's rows are contiguous in the leaf-ordered row copy
          const double* src = a.proj_leaf + p0 * d;
          for (int f = lane; f < cn * DP; f += 32) {
            const int i = f / DP, j = f - i * DP;
            cs[i][j] = j < d ? __ldg(src + (int64_t)i * d + j) : 0.0;
          }
          const int32_t id = lane < cn ? __ldg(a.perm + p0 + lane) : 0x7fffffff;
          __syncwarp();
          const double d2 = lane < cn ? chain(cs[lane]) : kInf;
          const WarpLexMin m = warp_lexmin(d2, id);
          if (lex_less(m.d2, m.id, best, best_id)) {
            best = m.d2;
            best_id = m.id;
          }
          __syncwarp();
        }
        scanned += e.w;
        ++leaves;
        continue;
      }
      const int nc = -e.w, fc = e.z;
      if (size + nc > kBtCap) {  // frontier too wide for the pool: the query
        overflow = true;         // is re-run by the deep-stack warp kernel
        break;
      }
      for (int cb = 0; cb < nc; cb += CH) {
        const int cn = min(CH, nc - cb);
        // children's centroid rows are contiguous: coalesced staging
        const double* src = a.tree.centroid + (int64_t)(fc + cb) * d;
        for (int f = lane; f < cn * DP; f += 32) {
          const int c = f / DP, j = f - c * DP;
          cs[c][j] = j < d ? __ldg(src + (int64_t)c * d + j) : 0.0;
        }
        int2 cm = make_int2(0, 0);
        int32_t ct = 0;
        if (lane < cn) {
          const int child = fc + cb + lane;
          cm = __ldg(a.tree.meta + child);
          ct = a.tree.tie ? __ldg(a.tree.tie + child) : child;
        }
        __syncwarp();
        if (lane < cn) {
          pk[size + lane] = chain(cs[lane]);
          pn[size + lane] = make_int4(fc + cb + lane, ct, cm.x, cm.y);
        }
        size += cn;
        __syncwarp();
      }
    }
    if (lane == 0) {
      if (overflow) {
        a.ovf_list[atomicAdd(a.ovf_count, 1)] = (int32_t)q;
      } else {
        a.out_idx[q] = best_id;
        a.out_d2[q] = best;
        if (a.out_scanned) a.out_scanned[q] = scanned;
        if (a.out_exact) a.out_exact[q] = scanned;
        if (a.out_visited) a.out_visited[q] = visited;
      }
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// backtrack(m), m > 2, with a GROUP of G lanes per query (G = 8 or 16 >= the
// tree's branching; 32 / G queries per warp).  The warp-per-query kernel above
// is issue-bound with 8 of its 32 lanes forming keys; here lane c of a group
// forms child c's key (or scans leaf point c) and every lane is busy.
//
//  * rows come straight from global memory into registers: the children of a
//    node (contiguous in the breadth-first layout) and the points of a leaf
//    are stored PAIR-INTERLEAVED per block -- element (row i, dim j) of a
//    block of n rows starting at row s sits at s*DP + (j/2)*(2n) + 2i + (j&1)
//    (DP = the fp32 layouts' width class of d, pad dims zero) -- so the G
//    lanes' 16-byte loads of one dim pair are one contiguous segment: no
//    shared-memory staging, no barrier between the loads and the chains, and
//    the loads are unpredicated (idle lanes re-read a valid row);
//  * the frontier is the same unsorted pool of (key, tie id, node meta) in
//    shared memory, CAP entries per query; a pop is a group-wide lexicographic
//    min; a query whose frontier would outgrow the pool is listed and re-run
//    by the deep-stack kernel (same answers);
//  * the loop body is the same for leaves and inner nodes (evaluate <= G rows,
//    then either fold into the best or append to the pool), so the groups of
//    a warp stay converged; every shuffle uses the full-warp mask with xor
//    offsets < G.
// Keys and leaf distances are the reference's fp64 j-ascending chains
// (km_tree.cpp:15-22, 128-139, 232-250); dims d..DP-1 add an exact +0.0.
#ifndef PSG_BG_CAP
#define PSG_BG_CAP 96
#endif
#ifndef PSG_BG_MINB
#define PSG_BG_MINB 4
#endif
constexpr int kBgWarps = 4, kBgCap = PSG_BG_CAP;
// 16-lane groups (branching 9..16): a frontier grows by up to 15 per expansion
constexpr int kBgCap16 = 224;

//
// Approximate queries (AP, tensor-core projection): a.q holds q^ with
// |q^ - q|_2 <= delta = a.qdelta[query] (q = the reference's fp64 projection).
// For any row p, |sqrt(D^(p)) - sqrt(D(p))| <= delta (D = real dist^2), and a
// chain's rounding is <= (d + 3) 2^-53 relative.  A decision "key a is the
// strict minimum" made on the q^ keys is the reference's decision whenever
// every other key exceeds T(a) = (sqrt(K^_a) + 2 delta)^2 inflated by 1e-11
// (which dominates both chains' rounding): the kernel tracks the second
// smallest key of every pop and of all scanned points -- as the HIGH WORD of
// the non-negative double (an ordered integer; hi(k2) > hi(T) implies k2 > T,
// one 32-bit min / shuffle instead of fp64 ones) -- and a query with any
// decision inside its band (or whose frontier outgrows the pool) is listed in
// a.amb_list and re-run with its exact projection (AP = false, device-counted
// list, results written through a.out_map).
template <int DP, int G, int CAP, bool AP, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, (DP <= 32 && WARPS == kBgWarps ? PSG_BG_MINB : 2))
search_backtrack_group_kernel(SearchArgs a) {
  constexpr int QPW = 32 / G, QPC = WARPS * QPW;
  constexpr int QS = DP + 4;  // q rows 32 bytes apart modulo the banks: the groups' 16-byte reads spread
  __shared__ __align__(16) double qs_all[QPC][QS];
  __shared__ double pk_all[QPC][CAP];
  __shared__ int32_t pt_all[QPC][CAP];
  __shared__ int2 pm_all[QPC][CAP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = lane % G, slot = warp * QPW + lane / G;
  double* qs = qs_all[slot];
  double* pk = pk_all[slot];
  int32_t* pt = pt_all[slot];
  int2* pm = pm_all[slot];
  const int d = a.d;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const int2 root = a.tree.meta[0];
  const int32_t root_tie = a.tree.tie ? a.tree.tie[0] : 0;
  const unsigned kFull = 0xffffffffu;
  const int64_t nq = a.nq_dev ? (int64_t)*a.nq_dev : a.nq;
  // greedy (km_tree.cpp:213-229): the frontier holds the current node's children
  // only, ties go to the first child, one leaf
  const bool greedy = a.mode == PSG_GREEDY;
  const int max_leaves = greedy ? 1 : a.max_leaves;
  // smallest key another entry must exceed for `k` to be the robust minimum
  auto band_top = [](double k, double dl2) {
    const double s = (double)__fsqrt_ru(__double2float_ru(k));
    return (k + dl2 * (2.0 * s + dl2)) * (1.0 + 1e-11);
  };
  for (int64_t q0 = (int64_t)blockIdx.x * QPC; q0 < nq; q0 += (int64_t)gridDim.x * QPC) {
    const bool live = q0 + slot < nq;
    // listed queries (the pool overflows of a previous pass): item -> query id
    const int64_t q = !live ? 0 : (a.q_list ? (int64_t)a.q_list[q0 + slot] : q0 + slot);
    for (int j = l; j < DP; j += G) qs[j] = (live && j < d) ? a.q[q * d + j] : 0.0;
    if (l == 0) {
      pk[0] = 0.0;
      pt[0] = root_tie;
      pm[0] = root;
    }
    __syncwarp();
    double best = kInf;
    int32_t second = 0x7ff00000;  // high word of the second smallest scanned key
    int32_t best_id = 0x7fffffff;
    int32_t scanned = 0, visited = 0;
    int size = live ? 1 : 0, leaves = 0;
    bool overflow = false;  // the frontier outgrew the pool
    bool ambig = false;     // AP: a decision fell inside the band
    double dl2 = 0.0;       // 2 delta (slightly inflated)
    if (AP && live) {
      const float dl = a.qdelta[q];
      if (!(dl < 3.0e38f)) ambig = true;  // no bound for this query: exact re-run
      dl2 = 2.0 * (double)dl * (1.0 + 1e-6);
    }
    for (;;) {
      const bool act = size > 0 && leaves < max_leaves && !overflow && !ambig;
      if (!__any_sync(kFull, act)) break;
      // ---- pop the lexicographic minimum (key, tie) of the group's pool ----
      double bk = kInf;
      int32_t k2 = 0x7ff00000;  // high word of the second smallest key
      int32_t bt = 0x7fffffff, bs = 0;
      const int n = act ? size : 0;
      for (int s = l; s < n; s += G) {
        const double k = pk[s];
        const int32_t t = pt[s];
        if (k < bk || (k == bk && t < bt)) {
          if (AP) k2 = __double2hiint(bk);
          bk = k;
          bt = t;
          bs = s;
        } else if (AP) {
          k2 = min(k2, __double2hiint(k));
        }
      }
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) {
        const double ok = __shfl_xor_sync(kFull, bk, off);
        const int32_t ot = __shfl_xor_sync(kFull, bt, off);
        const int32_t os = __shfl_xor_sync(kFull, bs, off);
        if (AP) {
          const int32_t o2 = __shfl_xor_sync(kFull, k2, off);
          k2 = min(min(k2, o2), max(__double2hiint(bk), __double2hiint(ok)));
        }
        if (ok < bk || (ok == bk && ot < bt)) {
          bk = ok;
          bt = ot;
          bs = os;
        }
      }
      const int2 e = pm[bs];
      __syncwarp();
      if (act) {
        if (l == 0) {
          pk[bs] = pk[size - 1];
          pt[bs] = pt[size - 1];
          pm[bs] = pm[size - 1];
        }
        --size;
        if (greedy) size = 0;  // the siblings are dropped
        ++visited;
      }
      __syncwarp();
      // ---- the popped node's rows: leaf points or children's centroids ----
      const bool leaf = e.y >= 0;
      int cnt = act ? (leaf ? e.y : -e.y) : 0;
      if (act && !leaf && size + cnt > CAP) {
        overflow = true;  // re-run by the deep-stack kernel
        cnt = 0;
      }
      if (AP && act && !(k2 > __double2hiint(band_top(bk, dl2)))) {
        ambig = true;  // the pop order is not certain: exact re-run
        cnt = 0;
      }
      // idle groups / lanes read row 0 of a one-row block (always valid)
      const int cl = cnt > 0 ? cnt : 1;
      const double* blk = cnt > 0 ? (leaf ? a.proj_leaf_il : a.tree.centroid_il) + (int64_t)e.x * DP
                                  : a.tree.centroid_il;
      for (int base = 0; __any_sync(kFull, base < cnt); base += G) {
        const int i = base + l;
        const bool on = i < cnt;
        double2 r[DP / 2];
        {
          const double2* p = reinterpret_cast<const double2*>(blk) + (on ? i : 0);
#pragma unroll
          for (int jp = 0; jp < DP / 2; ++jp) r[jp] = __ldg(p + (int64_t)jp * cl);
        }
        int2 cm = make_int2(0, 0);
        int32_t ct = 0x7fffffff;
        if (on) {
          if (leaf) {
            ct = __ldg(a.perm + e.x + i);
          } else {
            cm = __ldg(a.tree.meta + e.x + i);
            ct = (a.tree.tie && !greedy) ? __ldg(a.tree.tie + e.x + i) : e.x + i;
          }
        }
        double acc = 0.0;
#pragma unroll
        for (int jp = 0; jp < DP / 2; ++jp) {
          const double2 qq = *reinterpret_cast<const double2*>(qs + 2 * jp);
          const double t0 = dsub(qq.x, r[jp].x);
          acc = dadd(acc, dmul(t0, t0));
          const double t1 = dsub(qq.y, r[jp].y);
          acc = dadd(acc, dmul(t1, t1));
        }
        if (on && !leaf) {
          pk[size + i] = acc;
          pt[size + i] = ct;
          pm[size + i] = cm;
        }
        // leaf rows: group-wide lexicographic (dist^2, id) minimum (inner-node
        // groups and idle lanes carry +inf and change nothing)
        if (__any_sync(kFull, on && leaf)) {
          double md = (on && leaf) ? acc : kInf;
          int32_t m2 = 0x7ff00000;
          int32_t mi = (on && leaf) ? ct : 0x7fffffff;
#pragma unroll
          for (int off = G / 2; off > 0; off >>= 1) {
            const double od = __shfl_xor_sync(kFull, md, off);
            const int32_t oi = __shfl_xor_sync(kFull, mi, off);
            if (AP) {
              const int32_t o2 = __shfl_xor_sync(kFull, m2, off);
              m2 = min(min(m2, o2), max(__double2hiint(md), __double2hiint(od)));
            }
            if (lex_less(od, oi, md, mi)) {
              md = od;
              mi = oi;
            }
          }
          if (AP) second = min(min(second, m2), max(__double2hiint(best), __double2hiint(md)));
          if (lex_less(md, mi, best, best_id)) {
            best = md;
            best_id = mi;
          }
        }
      }
      if (act && !overflow && !ambig) {
        if (leaf) {
          scanned += cnt;
          ++leaves;
        } else {
          size += cnt;
        }
      }
      __syncwarp();
    }
    if (AP && live && !overflow && !ambig && !(second > __double2hiint(band_top(best, dl2))))
      ambig = true;
    if (live && l == 0) {
      if (overflow && a.ovf_list) {  // next pass: the larger pool, then the deep stack
        a.ovf_list[atomicAdd(a.ovf_count, 1)] = (int32_t)q;
      } else if (overflow || ambig) {
        if (AP) {
          const int s = atomicAdd(a.amb_count, 1);
          a.amb_list[s] = (int32_t)q;
          a.amb_c0[s] = 0;
          a.amb_c1[s] = -1;  // resolve: exact projection only, then the re-run
        } else {
          atomicOr(a.flags, FLAG_STACK_OVERFLOW);  // no list to hand the query to
        }
      } else {
        const int64_t o = a.out_map ? (int64_t)a.out_map[q] : q;
        a.out_idx[o] = best_id;
        if (a.out_d2) a.out_d2[o] = best;
        if (a.out_scanned) a.out_scanned[o] = scanned;
        if (a.out_exact) a.out_exact[o] = scanned;
        if (a.out_visited) a.out_visited[o] = visited;
      }
    }
    __syncwarp();
  }
}

// Pair-interleaved copy of row blocks (see search_backtrack_group_kernel): one
// warp per tree node; inner nodes interleave their children's centroid rows,
// leaves their points' rows (leaf order); dE = the padded block width.  `out`
// is zeroed by the caller (the pad dims).
__global__ void interleave_blocks_kernel(const double* __restrict__ rows,
                                         const int2* __restrict__ meta, int n_nodes, int d,
                                         int dE, int want_leaves, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t node = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; node < n_nodes;
       node += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int2 m = meta[node];
    const bool leaf = m.y >= 0;
    if (leaf != (want_leaves != 0)) continue;
    const int cnt = leaf ? m.y : -m.y;
    const int64_t s = m.x;
    for (int f = lane; f < cnt * d; f += 32) {
      const int i = f / d, j = f - i * d;
      out[s * dE + (int64_t)(j >> 1) * 2 * cnt + 2 * i + (j & 1)] = rows[(s + i) * d + j];
    }
  }
}

// ----------------------------------------------------------------------------
// Exact search (the bit-parity mode, km_tree.cpp:251-278 semantics: the
// lexicographic minimum of (fp64 dist^2, id) over ALL database points).
//
//  * upper bound first: the query's previous assignment and its four lattice
//    neighbours' assignments shifted by the anchor offset (texture coherence)
//    are evaluated exactly; the smallest is the starting (best, best_id);
//  * traversal: depth-first, nearest child first, one warp per query.  Child
//    bounds max(ball, box) are computed in fp32 from outward-rounded data with
//    a slack dominating every fp32 rounding term, so a bound never exceeds the
//    true distance and pruning stays exact;
//  * leaves: consecutive leaf entries on the stack are scanned together (up to
//    32 points per warp pass); each lane evaluates an fp32 dist^2 with a
//    rigorous error bound and only points that can still be <= best are
//    re-evaluated with the reference's exact fp64 j-sequential chain; ties go
//    to the lowest id (km_tree.cpp:134).
template <int DP>
__global__ void __launch_bounds__(256) search_exact_kernel(SearchArgs a) {
  constexpr int W = 8;
  __shared__ double qs_all[W][DP];
  __shared__ __align__(16) float q32_all[W][DP];
  __shared__ int2 st_meta[W][kStackX];   // node meta: {first child | leaf start, -children | count}
  __shared__ float st_key[W][kStackX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* qs = qs_all[warp];
  float* q32 = q32_all[warp];
  int2* sm_ = st_meta[warp];
  float* sk = st_key[warp];
  const int d = a.d;
  const int N = (int)a.N;
  const int nn = a.tree.n_nodes;
  const int KB = d < kBoxDims ? d : kBoxDims;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);

  const int64_t nq = a.nq_dev ? (int64_t)*a.nq_dev : a.nq;
  for (int64_t q = (int64_t)blockIdx.x * W + warp; q < nq; q += (int64_t)gridDim.x * W) {
    double qn2 = 0.0;
    for (int j = lane; j < DP; j += 32) {
      const double v = j < d ? a.q[q * d + j] : 0.0;
      qs[j] = v;
      q32[j] = (float)v;
      qn2 += v * v;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) qn2 += __shfl_xor_sync(0xffffffffu, qn2, off);
    const float qn = __double2float_ru(sqrt(qn2) * (1.0 + 1e-12));
    __syncwarp();
    double best = kInf;
    int32_t best_id = 0x7fffffff;
    int64_t scanned = 0, exact_evals = 0;
    int32_t visited = 0;

    // ---- coherence seeds: exact dist^2 of up to 5 candidates, one per lane ----
    if (a.seed_idx) {
      int32_t cand = -1;
      if (lane == 0) {
        cand = a.seed_idx[q];
      } else if (lane <= 4 && a.qxs) {
        const int qix = (int)(q % a.qnx), qiy = (int)(q / a.qnx);
        const int qny = (int)(nq / a.qnx);
        const int nix = qix + (lane == 1 ? -1 : lane == 2 ? 1 : 0);
        const int niy = qiy + (lane == 3 ? -1 : lane == 4 ? 1 : 0);
        if (nix >= 0 && nix < a.qnx && niy >= 0 && niy < qny) {
          const int32_t e = a.seed_idx[(int64_t)niy * a.qnx + nix];
          const int ex = e % a.nxe + (a.qxs[qix] - a.qxs[nix]);
          const int ey = e / a.nxe + (a.qys[qiy] - a.qys[niy]);
          if (ex >= 0 && ex < a.nxe && ey >= 0 && ey < a.nye) cand = ey * a.nxe + ex;
        }
      }
      double d2 = kInf;
      if (cand >= 0) d2 = dist2_seq(qs, a.proj + (int64_t)cand * d, d);
      const WarpLexMin m = warp_lexmin(d2, cand >= 0 ? cand : 0x7fffffff);
      best = m.d2;
      best_id = m.id;
      const int ns = __popc(__ballot_sync(0xffffffffu, cand >= 0));
      scanned += ns;
      exact_evals += ns;
    }
    if (lane == 0) {
      sm_[0] = a.tree.meta[0];
      sk[0] = 0.f;
    }
    int top = 1;
    __syncwarp();
    while (top > 0) {
      // ---- gather a batch of leaves from the stack top (warp-uniform) ----------
      int bstart[4], bcnt[4];
      int nb = 0, tot = 0;
      int2 node = make_int2(0, 0);
      while (top > 0) {
        const int2 md = sm_[top - 1];
        const float key = sk[top - 1];
        if ((double)key > best) {  // km_tree.cpp:265 prune
          --top;
          continue;
        }
        if (md.y < 0) {
          if (nb == 0) {
            node = md;
            --top;
          }
          break;
        }
        const int cnt = md.y;
        if (nb > 0 && (tot + cnt > 32 || nb == 4)) break;
        --top;
        bstart[nb] = md.x;
        bcnt[nb] = cnt;
        ++nb;
        tot += cnt;
        if (tot >= 32) break;
      }
      __syncwarp();
      if (nb > 0) {
        for (int b = 0; b < nb; ++b) scanned += bcnt[b];
        visited += nb;
        const int chunks = (tot + 31) / 32;
        for (int ck = 0; ck < chunks; ++ck) {
          int i = ck * 32 + lane;
          int pos = -1;
          if (i < tot) {
            int b = 0;
#pragma unroll
            for (int t = 0; t < 3; ++t)
              if (b < nb - 1 && i >= bcnt[b]) i -= bcnt[b++];
            pos = bstart[b] + i;
          }
          float s = 0.f, eps = 0.f;
          if (pos >= 0) {
            // [dp/4][N] float4 groups: lanes read consecutive points -> coalesced
            const float4* col = reinterpret_cast<const float4*>(a.proj32_q4) + pos;
            float4 p[DP / 4];
#pragma unroll
            for (int k = 0; k < DP / 4; ++k)
              p[k] = (4 * k < d) ? __ldg(col + (int64_t)k * N) : make_float4(0, 0, 0, 0);
            const float4* qv = reinterpret_cast<const float4*>(q32);
#pragma unroll
            for (int k = 0; k < DP / 4; ++k) {
              const float4 qq = qv[k];
              float t = qq.x - p[k].x;
              s = fmaf(t, t, s);
              t = qq.y - p[k].y;
              s = fmaf(t, t, s);
              t = qq.z - p[k].z;
              s = fmaf(t, t, s);
              t = qq.w - p[k].w;
              s = fmaf(t, t, s);
            }
            const float pn = a.pnorm32[pos];
            eps = 2.5e-7f * (float)(d + 4) * s + 1.0e-6f * (qn + pn) * (sqrtf(s) + 1e-3f) + 1e-30f;
          }
          // (the current best is exact already: never re-evaluated)
          const int32_t pid = pos >= 0 ? a.perm[pos] : -1;
          const bool surv = pos >= 0 && (double)s - (double)eps <= best && pid != best_id;
          const unsigned smask = __ballot_sync(0xffffffffu, surv);
          if (!smask) continue;
          double d2 = kInf;
          int32_t id = 0x7fffffff;
          if (surv) {
            id = pid;
            const double* col = a.proj_soa + pos;
            double acc = 0.0;
#pragma unroll
            for (int j0 = 0; j0 < DP; j0 += 16) {
              if (j0 < d) {
                double p[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) p[jj] = (j0 + jj < d) ? col[(int64_t)(j0 + jj) * N] : 0.0;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                  if (j0 + jj < d) {
                    const double t = dsub(qs[j0 + jj], p[jj]);
                    acc = dadd(acc, dmul(t, t));
                  }
                }
              }
            }
            d2 = acc;
          }
          exact_evals += __popc(smask);
          const WarpLexMin m = warp_lexmin(d2, id);
          if (lex_less(m.d2, m.id, best, best_id)) {
            best = m.d2;
            best_id = m.id;
          }
        }
        continue;
      }
      if (node.y >= 0) break;
      // ---- expand an internal node: lanes (child, dim-group) -------------------
      const int nc = -node.y;
      ++visited;
      const int fc = node.x;
      for (int cb = 0; cb < nc; cb += 32) {
        const int ncb = min(32, nc - cb);
        // lanes per child: largest power of two with ncp * lpc <= 32
        const int ncp = ncb <= 1 ? 1 : ncb <= 2 ? 2 : ncb <= 4 ? 4 : ncb <= 8 ? 8 : ncb <= 16 ? 16 : 32;
        const int lpc = 32 / ncp;
        const int c = lane % ncp, g = lane / ncp;
        const bool valid = c < ncb;
        const int cid = fc + cb + (valid ? c : 0);
        const int2 cm = (valid && g == 0) ? a.tree.meta[cid] : make_int2(0, 0);
        float s = 0.f, bx = 0.f;
        // all loads of a block issued before use: one L2 round trip per 8 dims
        for (int j0 = g; j0 < d; j0 += 8 * lpc) {
          float cv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int j = j0 + k * lpc;
            cv[k] = j < d ? __ldg(a.tree.centroid32T + (int64_t)j * nn + cid) : 0.f;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int j = j0 + k * lpc;
            const float t = (j < d ? q32[j] : 0.f) - cv[k];
            s = fmaf(t, t, s);
          }
        }
        {
          float lov[kBoxDims], hiv[kBoxDims];
#pragma unroll
          for (int k = 0; k < kBoxDims; ++k) {
            const int j = g + k * lpc;
            lov[k] = j < KB ? __ldg(a.tree.boxlo + (int64_t)j * nn + cid) : 0.f;
            hiv[k] = j < KB ? __ldg(a.tree.boxhi + (int64_t)j * nn + cid) : 0.f;
          }
#pragma unroll
          for (int k = 0; k < kBoxDims; ++k) {
            const int j = g + k * lpc;
            if (j < KB) {
              const float qj = q32[j];
              float gap = fmaxf(lov[k] - qj, qj - hiv[k]) -
                          2.4e-7f * (fabsf(qj) + fabsf(lov[k]) + fabsf(hiv[k]));
              gap = fmaxf(gap, 0.f);
              bx = fmaf(gap, gap, bx);
            }
          }
        }
        for (int off = ncp; off < 32; off <<= 1) {
          s += __shfl_xor_sync(0xffffffffu, s, off);
          bx += __shfl_xor_sync(0xffffffffu, bx, off);
        }
        float lb2 = __int_as_float(0x7f800000);
        bool keep = false;
        if (valid) {
          const float dc = sqrtf(s);
          const float rad = a.tree.radius32[cid];
          const float slack = 2e-5f * (1.f + dc + rad + qn + a.tree.cnorm32[cid]);
          const float lb = dc - rad - slack;
          lb2 = lb > 0.f ? lb * lb * (1.f - 1e-6f) : 0.f;
          lb2 = fmaxf(lb2, bx * (1.f - 1e-5f));
          keep = (double)lb2 <= best;
        }
        // one representative lane (g == 0) per child
        const unsigned km = __ballot_sync(0xffffffffu, keep && g == 0);
        const int nkeep = __popc(km);
        int rank = 0;
        for (int o = 0; o < ncb; ++o) {
          const float ol = __shfl_sync(0xffffffffu, lb2, o);
          if (((km >> o) & 1u) && (ol < lb2 || (ol == lb2 && o < c))) ++rank;
        }
        if (top + nkeep > kStackX) {
          if (lane == 0) atomicOr(a.flags, FLAG_STACK_OVERFLOW);
          break;
        }
        if (keep && g == 0) {
          const int slot = top + nkeep - 1 - rank;  // nearest child popped first
          sm_[slot] = cm;
          sk[slot] = lb2;
        }
        top += nkeep;
        __syncwarp();
      }
    }
    if (lane == 0) {
      if (a.out_map) {  // a listed query: results go to its anchor, counters add
        const int32_t qa = a.out_map[q];
        a.out_idx[qa] = best_id;
        if (a.out_scanned) a.out_scanned[qa] += scanned;
        if (a.out_exact) a.out_exact[qa] += exact_evals;
      } else {
        a.out_idx[q] = best_id;
        a.out_d2[q] = best;
        if (a.out_scanned) a.out_scanned[q] = scanned;
        if (a.out_exact) a.out_exact[q] = exact_evals;
        if (a.out_visited) a.out_visited[q] = visited;
      }
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// Tile search (exact mode, default): one warp owns 32 consecutive queries,
// one query per lane, and the 32 queries share ONE depth-first traversal.
// A node is expanded / a leaf scanned when at least one lane's conservative
// bound is <= that lane's own best; every lane then evaluates its own query
// against the node's children or the leaf's points, which are staged once in
// shared memory and read as broadcasts.  This turns the irregular per-query
// traversal into dense, divergence-free fp32 work (lanes = queries, like a
// GEMM tile of queries x points), while each lane keeps its own exact
// lexicographic (fp64 dist^2, id) minimum.  Spatially consecutive anchors have
// overlapping windows and hence overlapping candidate sets, so the shared
// traversal visits little more than each query alone.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool full) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(full ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}

// three-input max (FMNMX3 on sm_100)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

constexpr int kTileStack = 48;
constexpr int kTileMaxB = 16;

template <int DP, int kTileWarps, bool kApprox>
__global__ void __launch_bounds__(32 * kTileWarps, DP <= 32 ? TILE_MIN_CTAS : TILE64_MIN_CTAS) search_tile_kernel(SearchArgs a) {
  constexpr int RS = DP + 4;  // padded staging row (floats): conflict-free 16 B accesses
  __shared__ int2 st_meta[kTileWarps][kTileStack];
  // per-lane node bounds of the stack as bf16 rounded DOWN: still valid lower
  // bounds (pruning only loosens by < 2^-7 = 0.78%), half the largest shared array
  __shared__ __nv_bfloat16 st_lb[kTileWarps][kTileStack][32];
  __shared__ __align__(16) float stage_all[kTileWarps][32 * RS];
  // staged points' (|p~|^2, |p~_B|^2); |p| <= sqrt(|p~|^2) (1 + 1e-6)
  __shared__ float2 pp_all[kTileWarps][32];
  float2* ppst = pp_all[threadIdx.x >> 5];
  __shared__ int2 cmeta_all[kTileWarps][kTileMaxB];
  __shared__ __align__(16) float box_all[kTileWarps][kTileMaxB][2 * kBoxDims];
  __shared__ int32_t pid_all[kTileWarps][32];
  __shared__ float tlb_all[kTileWarps][kTileMaxB][32];
  __shared__ unsigned tkey_all[kTileWarps][kTileMaxB];
  // approximate-query bookkeeping, per lane (touched only on exact
  // evaluations and at the end: kept out of the register file)
  __shared__ float band2_all[kTileWarps][32], sec_all[kTileWarps][32], thi_all[kTileWarps][32];
  __shared__ int32_t sid_all[kTileWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int2* sm_ = st_meta[warp];
  __nv_bfloat16(*slb)[32] = st_lb[warp];
  float* stage = stage_all[warp];
  int2* cmeta = cmeta_all[warp];
  float(*boxs)[2 * kBoxDims] = box_all[warp];
  int32_t* pid = pid_all[warp];
  float(*tlb)[32] = tlb_all[warp];
  unsigned* tkey = tkey_all[warp];
  const int d = a.d;
  const int N = (int)a.N;
  const int nn = a.tree.n_nodes;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const float kInfF = __int_as_float(0x7f800000);
  const int64_t nq = a.nq_dev ? (int64_t)*a.nq_dev : a.nq;
  // approximate queries (tensor-core projection): every comparison uses the
  // best distance inflated by the query's error band, (sqrt(best) + 2 delta)^2,
  // so every point that can be the exact winner is evaluated; `second` keeps
  // the smallest other evaluated distance (kernels_project_tc.cu)
  constexpr bool approx = kApprox;  // a.qdelta != nullptr
  // image queries: 8 x 4 anchor tiles (overlapping windows share candidates);
  // vector queries: 32 consecutive rows
  const int qny = a.qxs ? (int)(nq / a.qnx) : 0;
  const int tnx = a.qxs ? (a.qnx + kTW - 1) / kTW : 0;
  const int64_t n_tiles = a.qxs ? (int64_t)tnx * ((qny + kTH - 1) / kTH) : (nq + 31) / 32;

  // persistent warps fetch tiles from a global ticket: tile costs vary ~4x,
  // and a fast warp must not idle until its CTA's slowest warp finishes
  for (;;) {
    int64_t t = 0;
    if (lane == 0) t = atomicAdd(reinterpret_cast<unsigned long long*>(a.sched), 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n_tiles) break;
    if (a.tile_order) t = a.tile_order[t];  // costliest tiles first (previous search)
    int64_t q;
    bool valid;
    if (a.qxs) {
      const int tx = (int)(t % tnx), ty = (int)(t / tnx);
      const int ix = tx * kTW + (lane % kTW), iy = ty * kTH + (lane / kTW);
      valid = ix < a.qnx && iy < qny;
      q = valid ? (int64_t)iy * a.qnx + ix : 0;
    } else {
      q = t * 32 + lane;
      valid = q < nq;
    }
    const double* qrow = a.q + (valid ? q : 0) * d;
    bool trav = valid;
    if (approx) {
      const float twod = valid ? 2.f * a.qdelta[q] : 0.f;
      trav = valid && !(twod > 3.0e38f);  // delta = inf: exact fallback only
      band2_all[warp][lane] = twod;
      sec_all[warp][lane] = kInfF;
      thi_all[warp][lane] = kInfF;
      sid_all[warp][lane] = -1;
    }
    // float threshold for a best distance: the best itself, or its band
    auto infl = [&](double b) -> float {
      if (!approx || !(b > 0.0) || b == kInf) return __double2float_ru(b);
      const double r = sqrt(b) * (1.0 + 1e-12) + (double)band2_all[warp][lane];
      return __double2float_ru(r * r * (1.0 + 1e-15));
    };
    // the two smallest other evaluated distances (rounded down: lower bounds)
    // and the closer one's id: an ambiguous query with only one other point
    // in its band is settled by two exact evaluations, no re-search
    auto push = [&](double v, int32_t id) {
      if (!approx || id == sid_all[warp][lane]) return;
      const float vf = __double2float_rd(v);
      const float sv = sec_all[warp][lane];
      if (vf < sv) {
        thi_all[warp][lane] = sv;
        sec_all[warp][lane] = vf;
        sid_all[warp][lane] = id;
      } else {
        thi_all[warp][lane] = fminf(thi_all[warp][lane], vf);
      }
    };
    float2 q2[DP / 2];
    double qn2 = 0.0;
#pragma unroll
    for (int j = 0; j < DP / 2; ++j) {
      const double v0 = (valid && 2 * j < d) ? qrow[2 * j] : 0.0;
      const double v1 = (valid && 2 * j + 1 < d) ? qrow[2 * j + 1] : 0.0;
      // held negated: u = p + (-q) is one FADD2 against plainly staged rows
      q2[j] = make_float2(-(float)v0, -(float)v1);
      qn2 += v0 * v0 + v1 * v1;
    }
    const float qn = __double2float_ru(sqrt(qn2) * (1.0 + 1e-12));
    // |q~_B|^2 of the fp32 query (B = the dims after the first DP / P2_SPLIT_DEN), and the
    // rigorous bound of the expanded form's rounding: |fl(qq + pp - 2 q.p) -
    // |q~ - p~|^2| <= (n + 4) 2^-24 (qq + pp + 2 |q.p|) <= (n + 4) 2^-24 (|q| + |p|)^2
    // for n = the dims in expanded form (x1.5 margin for the rounded norms)
    float qqx;
    {
      double t = 0.0;
#pragma unroll
      for (int j = p2_split(DP) / 2; j < DP / 2; ++j) {
        t += (double)q2[j].x * (double)q2[j].x;
        t += (double)q2[j].y * (double)q2[j].y;
      }
      qqx = (float)t;
    }
    const float exp_slack = 1.5f * (float)(DP - p2_split(DP) + 4) * 5.9604645e-8f *
                            (qn + a.pnorm_max) * (qn + a.pnorm_max);
    // box margin: >= |float(q_j) - q_j| + the rounding of (-q_j -/+ margin)
    const float qdelta2 = 2.4e-7f * qn;
    // invalid lanes hold best = -1: every bound (>= 0) prunes them
    double best = trav ? kInf : -1.0;
    int32_t best_id = 0x7fffffff;
    int64_t scanned = 0, exact_evals = 0;
    int32_t visited = 0;

    // ---- seed (exact fp64): the query's previous assignment is the initial
    // upper bound.  (Lattice neighbours' shifted assignments were tried too: on
    // the bench stage they cost more exact evaluations than they save.)
    if (a.seed_idx && trav) {
      const int32_t cand = a.seed_idx[q];
      best = dist2_seq_cold(qrow, a.proj + (int64_t)cand * d, d);
      best_id = cand;
      ++scanned;
      ++exact_evals;
    }

    // best rounded up to float: float compares against it can only keep more
    float bestf = infl(best);
    if (lane == 0) sm_[0] = a.tree.meta[0];
    slb[0][lane] = __float2bfloat16_rd(0.f);
    int top = 1;
    __syncwarp();
    while (top > 0) {
      // ---- pop: drop entries no lane still wants; batch consecutive leaves ------
      int bstart[4], bcnt[4];
      int nb = 0, tot = 0;
      int2 node = make_int2(0, 0);
      while (top > 0) {
        const int2 md = sm_[top - 1];
        const bool want = __bfloat162float(slb[top - 1][lane]) <= bestf;
        if (!__any_sync(0xffffffffu, want)) {  // km_tree.cpp:265 prune, per lane
          --top;
          continue;
        }
        if (md.y < 0) {
          if (nb == 0) {
            node = md;
            --top;
          }
          break;
        }
        if (nb > 0 && (tot + md.y > 32 || nb == 4)) break;
        --top;
        bstart[nb] = md.x;
        bcnt[nb] = md.y;
        ++nb;
        tot += md.y;
        if (tot >= 32) break;
      }
      if (nb > 0) {
        visited += nb;
        scanned += tot;
        for (int c0 = 0; c0 < tot; c0 += 32) {
          const int cn = min(32, tot - c0);
          // stage <= 32 points: lane i loads point c0 + i (coalesced float4 groups)
          __syncwarp();
          if (lane < cn) {
            int i = c0 + lane, b = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k)
              if (b < nb - 1 && i >= bcnt[b]) i -= bcnt[b++];
            const int pos = bstart[b] + i;
            const float4* col = reinterpret_cast<const float4*>(a.proj32_q4) + pos;
            float4* dst = reinterpret_cast<float4*>(stage + lane * RS);
            // asynchronous global -> shared copies (LDGSTS): no staging
            // registers; dims >= d are zero-filled (src-size 0)
#pragma unroll
            for (int k = 0; k < DP / 4; ++k) cp_async16(dst + k, col + (int64_t)k * N, 4 * k < d);
            cp_async4(pid + lane, a.perm + pos);
            cp_async8(ppst + lane, a.pp32 + pos);
          }
          asm volatile("cp.async.wait_all;" ::: "memory");
          __syncwarp();
          // best rounded up to float: a float compare can only keep more points.
          // thr >= s for every point that can pass the precise test below
          // (eps is increasing in s and |p| <= pnorm_max)
          float best_up = bestf;
          float thr = (best_up + exp_slack) * (1.f + 1e-4f) +
                      1.01e-6f * (qn + a.pnorm_max) * (sqrtf(2.f * (best_up + exp_slack) + 1.f) + 1e-3f) + 1e-30f;
          // phase 1, branch-free over the batch: the P1_DIMS leading (highest
          // variance) PCA dims of every staged point against the batch-start
          // threshold; rounded sums of non-negative terms only grow, so a
          // partial sum above thr already rules the point out for this lane
          uint32_t pass = 0;
          // in chunks of P1_CHUNK staged points (a batch holds cn <= 32 of them)
#pragma unroll
          for (int i0 = 0; i0 < 32; i0 += P1_CHUNK) {
            if (i0 >= cn) break;
#pragma unroll
            for (int i = i0; i < i0 + P1_CHUNK; ++i) {
              const float4* pr = reinterpret_cast<const float4*>(stage + i * RS);
              float2 sa = make_float2(0.f, 0.f);
#pragma unroll
              for (int k = 0; k < P1_DIMS / 4; ++k) {
                const float4 p = pr[k];
                const float2 u0 = __fadd2_rn(q2[2 * k], make_float2(p.x, p.y));
                const float2 u1 = __fadd2_rn(q2[2 * k + 1], make_float2(p.z, p.w));
                sa = __ffma2_rn(u0, u0, sa);
                sa = __ffma2_rn(u1, u1, sa);
              }
              if (sa.x + sa.y <= thr) pass |= 1u << i;
            }
          }
          if (cn < 32) pass &= (1u << cn) - 1u;
          uint32_t todo = __reduce_or_sync(0xffffffffu, pass);
          // phase 2: the points some lane still wants, all dims, in batch order
          while (todo) {
            const int i = __ffs(todo) - 1;
            todo &= todo - 1;
            const float4* pr = reinterpret_cast<const float4*>(stage + i * RS);
            // packed fp32x2 (FADD2/FFMA2); partial sums in any order: the filter
            // bound covers it
            float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < p2_split(DP) / 4; ++k) {
              const float4 p = pr[k];
              const float2 u0 = __fadd2_rn(q2[2 * k], make_float2(p.x, p.y));
              const float2 u1 = __fadd2_rn(q2[2 * k + 1], make_float2(p.z, p.w));
              sa = __ffma2_rn(u0, u0, sa);
              sb = __ffma2_rn(u1, u1, sb);
            }
            // early exit after the leading (highest-variance) PCA dims: rounded
            // sums of non-negative terms only grow, so a partial sum above thr
            // already rules the point out for this lane
            if (!__any_sync(0xffffffffu, (sa.x + sa.y) + (sb.x + sb.y) <= thr)) continue;
            // the remaining dims B in expanded form: |q~_B|^2 + |p~_B|^2 - 2 q~_B.p~_B
            float2 ta = make_float2(0.f, 0.f), tb = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = p2_split(DP) / 4; k < DP / 4; ++k) {
              const float4 p = pr[k];
              ta = __ffma2_rn(q2[2 * k], make_float2(p.x, p.y), ta);
              tb = __ffma2_rn(q2[2 * k + 1], make_float2(p.z, p.w), tb);
            }
            const float s = ((sa.x + sa.y) + (sb.x + sb.y)) +
                            fmaf(2.f, (ta.x + ta.y) + (tb.x + tb.y), qqx + ppst[i].y);
            bool surv = s <= thr;
            if (surv) {
              const float sp = fmaxf(s, 0.f);
              const float eps = 2.5e-7f * (float)(d + 4) * sp +
                                1.0e-6f * (qn + (sqrtf(ppst[i].x) * 1.000001f)) * (sqrtf(sp) + 1e-3f) + 1e-30f + exp_slack;
              // the current best (usually the seed, met again in its leaf) is
              // exact already: re-evaluating it cannot change anything
              surv = s - eps <= best_up && pid[i] != best_id;
            }
            if (__any_sync(0xffffffffu, surv)) {
              if (surv) {
                const int32_t id = pid[i];
                const double d2 = dist2_seq_cold(qrow, a.proj + (int64_t)id * d, d);
                ++exact_evals;
                if (lex_less(d2, id, best, best_id)) {
                  if (best_id != id && best_id != 0x7fffffff) push(best, best_id);
                  best = d2;
                  best_id = id;
                  best_up = infl(best);
                  bestf = best_up;
                  thr = (best_up + exp_slack) * (1.f + 1e-4f) +
                        1.01e-6f * (qn + a.pnorm_max) * (sqrtf(2.f * (best_up + exp_slack) + 1.f) + 1e-3f) + 1e-30f;
                } else if (id != best_id) {
                  push(d2, id);
                }
              }
            }
          }
        }
        continue;
      }
      if (node.y >= 0) break;
      // ---- expand an internal node: stage children, every lane bounds them -----------
      ++visited;
      const int nc = -node.y;
      const int fc = node.x;
      __syncwarp();
      // the children's metas and (lo, -hi) boxes (64 contiguous bytes per
      // child in the tree's box2 layout; dims >= d hold [0, 0]) copied
      // global -> shared asynchronously
      if (lane < nc) cp_async8(cmeta + lane, a.tree.meta + fc + lane);
      for (int f = lane; f < nc * (kBoxDims / 2); f += 32)
        cp_async16(reinterpret_cast<float4*>(&boxs[0][0]) + f,
                   reinterpret_cast<const float4*>(a.tree.box2) + (int64_t)fc * (kBoxDims / 2) + f, true);
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
      // phase 1: box bound of every child (8 leading dims):
      // gap_j = max(lo_j - q_j - m, q_j - hi_j - m, 0) as one FADD2 + FMNMX3.
      // The box is rounded outward; the fp32 query differs from the fp64 one by
      // <= 2^-24 |q_j| and (-q_j - m), (q_j - m) round by <= 2^-24 (|q_j| + m):
      // m = qdelta2 = 2.4e-7 |q| covers both.  The remaining roundings are
      // relative to the results, covered by the final factor.  For j >= d the
      // box ([0, 0]) and q_j (0) are zero-padded: the gap is 0.
      float2 tq[kBoxDims];
#pragma unroll
      for (int j = 0; j < kBoxDims; ++j) {
        const float nq = (j & 1) ? q2[j >> 1].y : q2[j >> 1].x;  // -q_j
        tq[j] = make_float2(nq - qdelta2, -nq - qdelta2);
      }
      uint32_t boxpass = 0;
#pragma unroll 2
      for (int c = 0; c < nc; ++c) {
        float bx = 0.f;
        const float4* bc = reinterpret_cast<const float4*>(boxs[c]);
#pragma unroll
        for (int j2 = 0; j2 < kBoxDims / 2; ++j2) {
          const float4 bb = bc[j2];
          const float2 u0 = __fadd2_rn(make_float2(bb.x, bb.y), tq[2 * j2]);
          const float2 u1 = __fadd2_rn(make_float2(bb.z, bb.w), tq[2 * j2 + 1]);
          const float g0 = fmax3(u0.x, u0.y, 0.f), g1 = fmax3(u1.x, u1.y, 0.f);
          bx = fmaf(g0, g0, bx);
          bx = fmaf(g1, g1, bx);
        }
        bx *= 1.f - 1e-5f;
        tlb[c][lane] = bx;
        boxpass |= (bx <= bestf ? 1u : 0u) << c;
      }
      const uint32_t todo = __reduce_or_sync(0xffffffffu, boxpass);  // else pruned for all lanes
      if (lane < nc && !((todo >> lane) & 1u)) tkey[lane] = 0xffffffffu;
      // The box bound alone orders and prunes the children: the ball bound
      // (|q - c| - radius)+ of the wanted children (centroid rows staged, a
      // full-d distance per lane) cost more than it pruned -- measured on the
      // bench stage: search 1.69 -> 1.46 ms without it, points staged per
      // tile 2118 -> 2158.
      for (uint32_t m = todo; m; m &= m - 1) {
        const int c = __ffs(m) - 1;
        const float lb2 = tlb[c][lane];
        // non-negative floats order like their bit patterns
        const unsigned key = __reduce_min_sync(0xffffffffu, lb2 <= bestf ? __float_as_uint(lb2) : 0xffffffffu);
        if (lane == 0) tkey[c] = key;
      }
      __syncwarp();
      const unsigned mykey = lane < nc ? tkey[lane] : 0xffffffffu;
      const bool kept = mykey != 0xffffffffu;
      const unsigned keepmask = __ballot_sync(0xffffffffu, kept);
      const int nkeep = __popc(keepmask);
      if (top + nkeep > kTileStack) {
        if (lane == 0) atomicOr(a.flags, FLAG_STACK_OVERFLOW);
        break;
      }
      // lane c ranks child c among the kept ones (nearest popped first)
      int myslot = -1;
      if (kept) {
        int rank = 0;
        for (uint32_t m = keepmask; m; m &= m - 1) {
          const int o = __ffs(m) - 1;
          const unsigned ko = tkey[o];
          if (ko < mykey || (ko == mykey && o < lane)) ++rank;
        }
        myslot = top + nkeep - 1 - rank;
        sm_[myslot] = cmeta[lane];
      }
#pragma unroll 1
      for (uint32_t m = keepmask; m; m &= m - 1) {
        const int c = __ffs(m) - 1;
        slb[__shfl_sync(0xffffffffu, myslot, c)][lane] = __float2bfloat16_rd(tlb[c][lane]);
      }
      top += nkeep;
      __syncwarp();
    }
    if (valid) {
      if (approx) {
        // unique within the band -> it is the exact chain's winner; otherwise
        // (near-tie, or no usable band) the exact fallback re-searches it
        bool amb = !trav, pair = false;
        if (trav) {
          const double r = sqrt(best) * (1.0 + 1e-12) + (double)band2_all[warp][lane];
          const double band = r * r * (1.0 + 1e-15);
          amb = (double)sec_all[warp][lane] <= band;
          pair = amb && (double)thi_all[warp][lane] > band;  // exactly {best, second} in the band
        }
        if (amb) {
          if (best_id == 0x7fffffff) best_id = a.seed_idx ? a.seed_idx[q] : 0;
          const int slot = atomicAdd(a.amb_count, 1);
          a.amb_list[slot] = (int32_t)q;
          a.amb_c0[slot] = best_id;
          a.amb_c1[slot] = pair ? sid_all[warp][lane] : -1;
        }
      }
      a.out_idx[q] = best_id;
      a.out_d2[q] = best;
      if (a.out_scanned) a.out_scanned[q] = scanned;
      if (a.out_exact) a.out_exact[q] = exact_evals;
      if (a.out_visited) a.out_visited[q] = visited;
    }
    __syncwarp();
  }
  // the last warp out re-arms the ticket for the next launch on the stream
  if (lane == 0) {
    __threadfence();
    const unsigned long long total = (unsigned long long)gridDim.x * kTileWarps;
    unsigned long long* s = reinterpret_cast<unsigned long long*>(a.sched);
    if (atomicAdd(s + 1, 1ull) == total - 1) {
      s[0] = 0;
      s[1] = 0;
      __threadfence();
    }
  }
}

template <int DP, int W>
static int tile_resident_ctas(psg_ctx* ctx) {
  static int per_sm = 0;
  if (!per_sm) {
    PSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, search_tile_kernel<DP, W, false>,
                                                           32 * W, 0));
    if (per_sm < 1) per_sm = 1;
  }
  return per_sm * ctx->num_sms;
}

// Image searches with few queries leave most of the GPU idle on 32-query
// tiles (one warp per tile): below ~6 tiles per SM the warp-per-query kernel
// wins (measured: cfg3 finest w = 32, 15,625 anchors: tiles 4.06 ms vs
// 2.79 ms; w = 16, 64,009 anchors: 2.54 vs 7.07).
static bool enough_tiles(psg_ctx* ctx, int64_t nq) { return nq >= (int64_t)32 * 6 * ctx->num_sms; }

bool search_uses_tiles(psg_ctx* ctx, const DevTree& tree, int d, bool exact, int64_t nq) {
  return exact && d <= 64 && tree.centroid32 && !ctx->knobs.legacy_search &&
         tree.max_children <= kTileMaxB && 1 + tree.max_depth * (tree.max_children - 1) <= kTileStack &&
         (nq < 0 || enough_tiles(ctx, nq));
}

bool search_uses_groups(psg_ctx* ctx, const Index& ix, const psg_budget& budget) {
  const bool small = budget.mode == PSG_GREEDY || budget.max_leaves <= 2;
  return budget.mode != PSG_EXACT && ix.d > 0 && ix.d <= 64 && ix.proj_leaf_il &&
         ix.tree.centroid_il && ix.tree.max_children <= 16 && !ctx->knobs.legacy_search &&
         !ctx->knobs.bt_warp && !(ctx->knobs.bt_thread && small);
}

// greedy / backtrack(m), d <= 64: the lane-group kernel (or, for m > 2 on wide
// trees / PERSYN_BT_WARP, the warp-per-query kernel), then the deep-stack kernel for the
// queries whose frontier outgrew the pool.  a.qdelta set: approximate queries
// (see search_backtrack_group_kernel; uncertain queries go to a.amb_list and
// nothing overflows).  a.nq_dev set: a device-counted list of exact queries
// whose results go through a.out_map.
// Global scratch of the deep-stack kernel's frontiers (one region per warp of
// its num_sms x kSearchWarps grid), allocated once per context on first use.
constexpr int kDeepCap = 16384;
void ensure_deep_scratch(psg_ctx* ctx) {
  const size_t warps = (size_t)ctx->num_sms * kSearchWarps;
  if (!ctx->deep_key) {
    PSG_CUDA(cudaMalloc(&ctx->deep_key, sizeof(double) * warps * kDeepCap));
    PSG_CUDA(cudaMalloc(&ctx->deep_node, sizeof(int32_t) * warps * kDeepCap));
  }
}
static void deep_scratch(psg_ctx* ctx, SearchArgs& b) {
  ensure_deep_scratch(ctx);
  b.deep_key = ctx->deep_key;
  b.deep_node = ctx->deep_node;
  b.deep_cap = kDeepCap;
}

static void launch_backtrack(psg_ctx* ctx, const SearchArgs& a) {
  DBuf<int32_t> ovf;
  DBuf<int> ovf_n;
  SearchArgs b = a;
  // (the caller may provide the list buffers: levels allocate them once,
  // outside any captured iteration)
  if (!b.ovf_list || !b.ovf_count) {
    ovf.alloc((size_t)a.nq);
    ovf_n.alloc(1);
    b.ovf_list = ovf.p;
    b.ovf_count = ovf_n.p;
  }
  PSG_CUDA(cudaMemsetAsync(b.ovf_count, 0, sizeof(int), ctx->stream));
  const int mc = a.tree.max_children;
  const bool groups = b.proj_leaf_il && a.tree.centroid_il && mc <= 16 && !ctx->knobs.bt_warp;
  if (!groups && (a.qdelta || a.nq_dev || a.out_map))
    fail(PSG_E_LOGIC, "approximate / listed backtrack queries need the lane-group kernel");
  DBuf<int32_t> ovf2;
  DBuf<int> ovf2_n;
  if (groups) {
    // a group of 8 (16) lanes per query: 16 (8) queries per 4-warp CTA with a
    // pool of 96 (224) entries.  8-lane groups whose frontier outgrows the 96
    // (budgets past ~8 leaves, deep trees) are listed and re-run by a second
    // pass with the 224-entry pool in 2-warp CTAs (static shared memory stays
    // below 48 KB); what outgrows that goes to the deep-stack kernel.
    const dim3 blk(32 * kBgWarps), blk2(64);
#define PSG_BG_LAUNCH3(DPV, GV, CAPV, WV, GRID, BLK, ARGS)                                       \
  do {                                                                                           \
    if ((ARGS).qdelta)                                                                           \
      search_backtrack_group_kernel<DPV, GV, CAPV, true, WV>                                     \
          <<<(int)(GRID), BLK, 0, ctx->stream>>>(ARGS);                                          \
    else                                                                                         \
      search_backtrack_group_kernel<DPV, GV, CAPV, false, WV>                                    \
          <<<(int)(GRID), BLK, 0, ctx->stream>>>(ARGS);                                          \
  } while (0)
#define PSG_BG_LAUNCH(DPV)                                                          \
  do {                                                                              \
    if (mc > 8) {                                                                   \
      PSG_BG_LAUNCH3(DPV, 16, kBgCap16, kBgWarps, blocks, blk, b);                  \
    } else {                                                                        \
      PSG_BG_LAUNCH3(DPV, 8, kBgCap, kBgWarps, blocks, blk, b);                     \
      PSG_LAUNCHED(ctx);                                                            \
      PSG_BG_LAUNCH3(DPV, 8, kBgCap16, 2, blocks2, blk2, b2);                       \
    }                                                                               \
  } while (0)
    const int qpc = kBgWarps * (mc <= 8 ? 4 : 2);
    int64_t blocks = (a.nq + qpc - 1) / qpc;
    const int64_t cap = a.nq_dev ? (int64_t)ctx->num_sms : (int64_t)ctx->num_sms * 16;
    if (blocks > cap) blocks = cap;
    // second pass over the first pass's overflow list (device-counted)
    SearchArgs b2 = b;
    int64_t blocks2 = std::min<int64_t>((a.nq + 7) / 8, a.nq_dev ? ctx->num_sms : ctx->num_sms * 8);
    int32_t* l2 = a.ovf2_list;
    int* n2 = a.ovf2_count;
    if (mc <= 8) {
      if (!a.qdelta) {
        if (!l2 || !n2) {  // (levels provide these buffers)
          ovf2.alloc((size_t)a.nq);
          ovf2_n.alloc(1);
          l2 = ovf2.p;
          n2 = ovf2_n.p;
        }
        PSG_CUDA(cudaMemsetAsync(n2, 0, sizeof(int), ctx->stream));
      }
      b2.q_list = b.ovf_list;
      b2.nq_dev = b.ovf_count;
      // approximate queries: what outgrows the large pool too joins the
      // uncertain queries' list (exact re-run); exact ones go to the deep stack
      b2.ovf_list = a.qdelta ? nullptr : l2;
      b2.ovf_count = a.qdelta ? nullptr : n2;
    } else if (a.qdelta) {
      b.ovf_list = nullptr;  // 16-lane groups, approximate: overflows join the uncertain list
      b.ovf_count = nullptr;
    }
    // the blocks' width = the index's fp32 layout class (upload_tree)
    if (a.d <= 24) PSG_BG_LAUNCH(24);
    else if (a.d <= 32) PSG_BG_LAUNCH(32);
    else if (a.d <= 48) PSG_BG_LAUNCH(48);
    else PSG_BG_LAUNCH(64);
#undef PSG_BG_LAUNCH
#undef PSG_BG_LAUNCH3
    if (mc <= 8 && !a.qdelta) {  // the deep-stack kernel takes the second pass's list
      b.ovf_list = l2;
      b.ovf_count = n2;
    }
  } else {
    int64_t blocks = (a.nq + kBtWarps - 1) / kBtWarps;
    const int64_t cap = (int64_t)ctx->num_sms * 16;
    if (blocks > cap) blocks = cap;
    if (a.d <= 32)
      search_backtrack_kernel<32><<<(int)blocks, 32 * kBtWarps, 0, ctx->stream>>>(b);
    else
      search_backtrack_kernel<64><<<(int)blocks, 32 * kBtWarps, 0, ctx->stream>>>(b);
  }
  PSG_LAUNCHED(ctx);
  if (a.qdelta) return;  // uncertain / overflowing queries are on the caller's list
  b.nq_dev = nullptr;
  deep_scratch(ctx, b);
  search_kernel<<<ctx->num_sms, 32 * kSearchWarps, 0, ctx->stream>>>(b);
  PSG_LAUNCHED(ctx);
}

void launch_search(psg_ctx* ctx, const SearchArgs& a) {
  ProfScope _prof(ctx, a.nq_dev ? K_FALLBACK : K_SEARCH);
  if (a.nq <= 0) return;
  if (a.nq_dev) {
    // a device-counted list of unrelated queries (the exact fallback of the
    // tensor-core projection): one warp per query -- tiles of 32 unrelated
    // queries would traverse the union of their candidate sets
    if (a.mode != PSG_EXACT) {  // uncertain queries of an approximate greedy / backtrack search
      launch_backtrack(ctx, a);
      return;
    }
    if (a.mode != PSG_EXACT || !a.proj32_q4 || !a.tree.centroid32T)
      fail(PSG_E_LOGIC, "device-counted search needs the exact warp kernel");
    const int64_t blocks = 32;  // re-searches are rare: a few hundred warps
    if (a.d <= 32)
      search_exact_kernel<32><<<(int)blocks, 256, 0, ctx->stream>>>(a);
    else if (a.d <= 64)
      search_exact_kernel<64><<<(int)blocks, 256, 0, ctx->stream>>>(a);
    else
      search_exact_kernel<kMaxDP><<<(int)blocks, 256, 0, ctx->stream>>>(a);
    PSG_LAUNCHED(ctx);
    return;
  }
  if (a.d > kMaxD) fail(PSG_E_DOMAIN, "retained PCA dimension > 128 is not supported");
  const bool tile_ok = a.d <= 64 && a.tree.max_children <= kTileMaxB &&
                       1 + a.tree.max_depth * (a.tree.max_children - 1) <= kTileStack &&
                       (!a.qxs || a.qdelta || enough_tiles(ctx, a.nq));
  if (a.mode == PSG_EXACT && a.proj32_q4 && a.tree.centroid32 && tile_ok && !ctx->knobs.legacy_search) {
    if (!a.sched) fail(PSG_E_LOGIC, "tile search launched without its scheduler counters");
    const int64_t tiles = (a.nq + 31) / 32;
    const int wpb = a.d <= 32 ? 4 : 2;  // static smem <= 48 KB per CTA
    int64_t blocks = (tiles + wpb - 1) / wpb;
    // the instantiation's DP must equal the index's fp32 layout width (ix.dp:
    // the per-point half norms are split at DP / P2_SPLIT_DEN)
    const int64_t cap = a.d <= 24   ? tile_resident_ctas<24, 4>(ctx)
                        : a.d <= 32 ? tile_resident_ctas<32, 4>(ctx)
                        : a.d <= 48 ? tile_resident_ctas<48, 2>(ctx)
                                    : tile_resident_ctas<64, 2>(ctx);
    if (blocks > cap) blocks = cap;
    if (a.d <= 24)
      (a.qdelta ? search_tile_kernel<24, 4, true> : search_tile_kernel<24, 4, false>)
          <<<(int)blocks, 32 * 4, 0, ctx->stream>>>(a);
    else if (a.d <= 32)
      (a.qdelta ? search_tile_kernel<32, 4, true> : search_tile_kernel<32, 4, false>)
          <<<(int)blocks, 32 * 4, 0, ctx->stream>>>(a);
    else if (a.d <= 48)
      (a.qdelta ? search_tile_kernel<48, 2, true> : search_tile_kernel<48, 2, false>)
          <<<(int)blocks, 32 * 2, 0, ctx->stream>>>(a);
    else
      (a.qdelta ? search_tile_kernel<64, 2, true> : search_tile_kernel<64, 2, false>)
          <<<(int)blocks, 32 * 2, 0, ctx->stream>>>(a);
    PSG_LAUNCHED(ctx);
    return;
  }
  if (a.mode == PSG_EXACT && a.proj32_q4 && a.tree.centroid32T) {
    int64_t blocks = (a.nq + 7) / 8;
    const int64_t cap = (int64_t)ctx->num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (a.d <= 32)
      search_exact_kernel<32><<<(int)blocks, 256, 0, ctx->stream>>>(a);
    else if (a.d <= 64)
      search_exact_kernel<64><<<(int)blocks, 256, 0, ctx->stream>>>(a);
    else
      search_exact_kernel<kMaxDP><<<(int)blocks, 256, 0, ctx->stream>>>(a);
    PSG_LAUNCHED(ctx);
    return;
  }
  // thread-per-query kernel for greedy and short backtracks; longer frontiers
  // (m > 2) spill the per-thread heap and run faster warp-per-query (as does
  // d > 64: the per-thread query would not fit the register file)
  // greedy / backtrack(m) on the lane-group kernel whenever the tree fits it
  if (a.mode != PSG_EXACT && !ctx->knobs.legacy_search && a.d <= 64 && a.proj_leaf_il &&
      a.tree.centroid_il && a.tree.max_children <= 16 && !ctx->knobs.bt_warp &&
      !(ctx->knobs.bt_thread && (a.mode == PSG_GREEDY || a.max_leaves <= 2))) {
    launch_backtrack(ctx, a);
    return;
  }
  if (a.mode != PSG_EXACT && !ctx->knobs.legacy_search && a.d <= 64 &&
      (a.mode == PSG_GREEDY || a.max_leaves <= 2)) {
    int64_t blocks = (a.nq + 127) / 128;
    const int64_t cap = (int64_t)ctx->num_sms * 64;
    if (blocks > cap) blocks = cap;
    if (a.d <= 32)
      search_budget_kernel<32><<<(int)blocks, 128, 0, ctx->stream>>>(a);
    else
      search_budget_kernel<64><<<(int)blocks, 128, 0, ctx->stream>>>(a);
    PSG_LAUNCHED(ctx);
    return;
  }
  if (a.mode == PSG_BACKTRACK && a.d <= 64 && !ctx->knobs.legacy_search) {
    launch_backtrack(ctx, a);
    return;
  }
  int64_t blocks = (a.nq + kSearchWarps - 1) / kSearchWarps;
  const int64_t cap = (int64_t)ctx->num_sms * 16;
  if (blocks > cap) blocks = cap;
  SearchArgs c = a;  // all queries (not the overflow-list mode)
  c.ovf_list = nullptr;
  c.ovf_count = nullptr;
  if (c.mode == PSG_BACKTRACK) {  // frontiers may outgrow shared memory: one scratch region per warp
    if (blocks > ctx->num_sms) blocks = ctx->num_sms;
    deep_scratch(ctx, c);
  }
  search_kernel<<<(int)blocks, 32 * kSearchWarps, 0, ctx->stream>>>(c);
  PSG_LAUNCHED(ctx);
}

// ----------------------------------------------------------------------------
// Locality order for unstructured query sets (search-only workloads): each
// query's greedy-descent leaf (fp32 centroid distances) is a sort key, so the
// tile kernel's 32-query tiles share candidates.  Ordering only; results are
// scattered back and are independent of it.
__global__ void greedy_leaf_key_kernel(const double* __restrict__ q, int64_t nq, int d,
                                       DevTree tree, uint32_t* __restrict__ keys,
                                       int32_t* __restrict__ order) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* qi = q + i * d;
    int2 m = tree.meta[0];
    int node = 0;
    while (m.y < 0) {
      const int fc = m.x, nc = -m.y;
      float bd = __int_as_float(0x7f800000);
      int bc = 0;
      for (int c = 0; c < nc; ++c) {
        const float* cen = tree.centroid32 + (int64_t)(fc + c) * d;
        float s = 0.f;
        for (int j = 0; j < d; ++j) {
          const float t = (float)qi[j] - cen[j];
          s = fmaf(t, t, s);
        }
        if (s < bd) {
          bd = s;
          bc = c;
        }
      }
      node = fc + bc;
      m = tree.meta[node];
    }
    keys[i] = (uint32_t)node;
    order[i] = (int32_t)i;
  }
}

template <class T>
__global__ void gather_rows_kernel(const T* __restrict__ src, const int32_t* __restrict__ order,
                                   int64_t n, int width, T* __restrict__ dst) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n * width;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / width;
    const int j = (int)(f - i * width);
    dst[f] = src[(int64_t)order[i] * width + j];
  }
}

template <class T>
__global__ void scatter_kernel(const T* __restrict__ src, const int32_t* __restrict__ order,
                               int64_t n, T* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[order[i]] = src[i];
}

// Tile schedule for the next search of the same anchors: the previous search's
// per-tile work (its shared scan count, held by every lane of the tile) sorted
// into 64 quarter-octave buckets, costliest bucket first -- long tiles start
// first and the tail is short tiles.  One CTA: count, scan, scatter.  (The
// order within a bucket may vary run to run; every tile's result and counters
// are independent of when it runs.)
constexpr int kOrderBuckets = 64;

__device__ __forceinline__ int tile_cost_bucket(int64_t c) {
  const float l = log2f((float)max(c, (int64_t)0) + 1.f) * 4.f;
  return kOrderBuckets - 1 - max(0, min(kOrderBuckets - 1, (int)l));  // descending cost
}

__global__ void __launch_bounds__(1024) tile_order_kernel(const int64_t* __restrict__ scanned,
                                                          int qnx, int tnx, int64_t n_tiles,
                                                          int32_t* __restrict__ order) {
  __shared__ int cnt[kOrderBuckets], pos[kOrderBuckets];
  if (threadIdx.x < kOrderBuckets) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int tx = (int)(t % tnx), ty = (int)(t / tnx);
    atomicAdd(&cnt[tile_cost_bucket(scanned[(int64_t)ty * kTH * qnx + tx * kTW])], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = 0; b < kOrderBuckets; ++b) {
      pos[b] = acc;
      acc += cnt[b];
    }
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const int tx = (int)(t % tnx), ty = (int)(t / tnx);
    const int b = tile_cost_bucket(scanned[(int64_t)ty * kTH * qnx + tx * kTW]);
    order[atomicAdd(&pos[b], 1)] = (int32_t)t;
  }
}

int64_t image_tile_count(int64_t nq, int qnx) {
  const int qny = (int)(nq / qnx);
  return (int64_t)((qnx + kTW - 1) / kTW) * ((qny + kTH - 1) / kTH);
}

void launch_tile_order(psg_ctx* ctx, const int64_t* prev_scanned, int64_t nq, int qnx,
                       int32_t* order) {
  ProfScope _prof(ctx, K_SCHED);
  const int64_t nt = image_tile_count(nq, qnx);
  if (nt <= 0) return;
  tile_order_kernel<<<1, 1024, 0, ctx->stream>>>(prev_scanned, qnx, (qnx + kTW - 1) / kTW, nt, order);
  PSG_LAUNCHED(ctx);
}

size_t sort_pairs_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return bytes;
}

void sort_pairs_u32(psg_ctx* ctx, const uint32_t* kin, uint32_t* kout, const int32_t* vin,
                    int32_t* vout, int64_t n, void* temp, size_t temp_bytes) {
  PSG_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kin, kout, vin, vout, (int)n, 0, 32,
                                           ctx->stream));
  ctx->launches++;
}

void launch_greedy_keys(psg_ctx* ctx, const double* q, int64_t nq, int d, const DevTree& tree,
                        uint32_t* keys, int32_t* order) {
  ProfScope _prof(ctx, K_SEARCH);
  int64_t blocks = (nq + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  greedy_leaf_key_kernel<<<(int)blocks, 256, 0, ctx->stream>>>(q, nq, d, tree, keys, order);
  PSG_LAUNCHED(ctx);
}

void launch_interleave_blocks(psg_ctx* ctx, const double* rows, const int2* meta, int n_nodes,
                              int d, int dE, bool leaves, int64_t n_rows, double* out) {
  PSG_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)n_rows * dE, ctx->stream));
  int64_t blocks = ((int64_t)n_nodes * 32 + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  if (blocks < 1) blocks = 1;
  interleave_blocks_kernel<<<(int)blocks, 256, 0, ctx->stream>>>(rows, meta, n_nodes, d, dE,
                                                                 leaves ? 1 : 0, out);
  PSG_LAUNCHED(ctx);
}

void launch_gather_rows_f64(psg_ctx* ctx, const double* src, const int32_t* order, int64_t n,
                            int width, double* dst) {
  int64_t blocks = (n * width + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  gather_rows_kernel<double><<<(int)blocks, 256, 0, ctx->stream>>>(src, order, n, width, dst);
  PSG_LAUNCHED(ctx);
}

void launch_scatter_i32(psg_ctx* ctx, const int32_t* src, const int32_t* order, int64_t n,
                        int32_t* dst) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  scatter_kernel<int32_t><<<(int)blocks, 256, 0, ctx->stream>>>(src, order, n, dst);
  PSG_LAUNCHED(ctx);
}

void launch_scatter_f64(psg_ctx* ctx, const double* src, const int32_t* order, int64_t n,
                        double* dst) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  scatter_kernel<double><<<(int)blocks, 256, 0, ctx->stream>>>(src, order, n, dst);
  PSG_LAUNCHED(ctx);
}

void launch_scatter_i64(psg_ctx* ctx, const int64_t* src, const int32_t* order, int64_t n,
                        int64_t* dst) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  scatter_kernel<int64_t><<<(int)blocks, 256, 0, ctx->stream>>>(src, order, n, dst);
  PSG_LAUNCHED(ctx);
}

// fp32 filter copies in leaf order: q4[j/4][pos][j%4] = (float) soa[j][pos], |p| rounded up.
// pp: (|p~|^2, |p~_B|^2) of the fp32 point p~ (B = dims >= dp / P2_SPLIT_DEN), rounded
// to nearest from exact fp64 sums of the fp32 squares.
__global__ void make_fp32_copies_kernel(const double* __restrict__ soa, int64_t N, int d, int dp,
                                        float* __restrict__ q4, float* __restrict__ pn,
                                        float2* __restrict__ pp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    double n2 = 0.0, f2 = 0.0, h2 = 0.0;
    for (int j = 0; j < dp; ++j) {
      const double v = j < d ? soa[(int64_t)j * N + i] : 0.0;
      const float vf = (float)v;
      q4[((int64_t)(j / 4) * N + i) * 4 + (j % 4)] = vf;
      n2 += v * v;
      const double vv = (double)vf * (double)vf;
      f2 += vv;
      if (j >= p2_split(dp)) h2 += vv;
    }
    pn[i] = __double2float_ru(sqrt(n2) * (1.0 + 1e-12));
    if (pp) pp[i] = make_float2((float)f2, (float)h2);
  }
}

void launch_make_fp32_copies(psg_ctx* ctx, const double* soa, int64_t N, int d, int dp,
                             float* aos32, float* pn, float2* pp) {
  ProfScope _prof(ctx, K_BUILD);
  if (N <= 0) return;
  int64_t blocks = (N + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  make_fp32_copies_kernel<<<(int)blocks, 256, 0, ctx->stream>>>(soa, N, d, dp, aos32, pn, pp);
  PSG_LAUNCHED(ctx);
}

// ----------------------------------------------------------------------------
// Full-D rescoring (optimizer.cpp:117-124, :232-234): one thread per query,
// j ascending over the window (dy, dx, c) against the candidate's dense
// exemplar window — the candidate matrix is never materialised.
// Candidate rows from the 8-channel padded exemplar mirror (one 32-byte
// load per pixel), NC = C at compile time; same (dy, dx, c) order.
template <int NC>
__device__ __forceinline__ double window_dist2_pad(const float* __restrict__ mirror, int img_w,
                                                   int w, int ax, int ay,
                                                   const float* __restrict__ ex8, int ew, int ex,
                                                   int ey) {
  double acc = 0.0;
  for (int dy = 0; dy < w; ++dy) {
    const float* v = mirror + ((int64_t)(ay + dy) * img_w + ax) * NC;
    const float* z8 = ex8 + ((int64_t)(ey + dy) * ew + ex) * 8;
#pragma unroll 2
    for (int dx = 0; dx < w; ++dx) {
      float4 z0, z1;
      ldg256(z8 + 8 * dx, z0, z1);
      const float zc[8] = {z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w};
      float vc[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) vc[c] = __ldg(v + dx * NC + c);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double t = dsub((double)vc[c], (double)zc[c]);
        acc = dadd(acc, dmul(t, t));
      }
    }
  }
  return acc;
}

__device__ __forceinline__ double window_dist2_any(const float* __restrict__ mirror, int img_w,
                                                   int C, int w, int ax, int ay,
                                                   const float* __restrict__ ex_mirror,
                                                   const float* __restrict__ ex8, int ew, int ex,
                                                   int ey);

// Same chain, with a whole window row's loads (w = 8: 8 candidate pixels and
// 8 x NC state values) issued before the row's adds: one memory round trip per
// row instead of one per pixel pair, for the latency-bound few-anchor case.
template <int NC>
__device__ __forceinline__ double window_dist2_pad_rows8(const float* __restrict__ mirror, int img_w,
                                                         int ax, int ay, const float* __restrict__ ex8,
                                                         int ew, int ex, int ey) {
  double acc = 0.0;
  for (int dy = 0; dy < 8; ++dy) {
    const float* v = mirror + ((int64_t)(ay + dy) * img_w + ax) * NC;
    const float* z8 = ex8 + ((int64_t)(ey + dy) * ew + ex) * 8;
    float4 z0[8], z1[8];
    float vc[8 * NC];
    // volatile loads: issued in this order, all before the row's chain (the
    // compiler otherwise sinks each load next to its use, one round trip per
    // pixel)
#pragma unroll
    for (int dx = 0; dx < 8; ++dx)
      asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                   : "=f"(z0[dx].x), "=f"(z0[dx].y), "=f"(z0[dx].z), "=f"(z0[dx].w), "=f"(z1[dx].x),
                     "=f"(z1[dx].y), "=f"(z1[dx].z), "=f"(z1[dx].w)
                   : "l"(z8 + 8 * dx));
#pragma unroll
    for (int k = 0; k < 8 * NC; ++k) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(vc[k]) : "l"(v + k));
#pragma unroll
    for (int dx = 0; dx < 8; ++dx) {
      const float zc[8] = {z0[dx].x, z0[dx].y, z0[dx].z, z0[dx].w, z1[dx].x, z1[dx].y, z1[dx].z, z1[dx].w};
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double t = dsub((double)vc[dx * NC + c], (double)zc[c]);
        acc = dadd(acc, dmul(t, t));
      }
    }
  }
  return acc;
}

__device__ __forceinline__ double window_dist2(const float* __restrict__ mirror, int img_w, int C,
                                               int w, int ax, int ay,
                                               const float* __restrict__ ex_mirror, int ew,
                                               int ex, int ey) {
  const int row = w * C;
  double acc = 0.0;
  for (int dy = 0; dy < w; ++dy) {
    const float* v = mirror + ((int64_t)(ay + dy) * img_w + ax) * C;
    const float* z = ex_mirror + ((int64_t)(ey + dy) * ew + ex) * C;
    int jj = 0;
    for (; jj + 8 <= row; jj += 8) {  // loads batched ahead of the sequential adds
      float vv[8], zz[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        vv[u] = __ldg(v + jj + u);
        zz[u] = __ldg(z + jj + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double t = dsub((double)vv[u], (double)zz[u]);
        acc = dadd(acc, dmul(t, t));
      }
    }
    for (; jj < row; ++jj) {
      const double t = dsub((double)v[jj], (double)z[jj]);
      acc = dadd(acc, dmul(t, t));
    }
  }
  return acc;
}

__device__ __forceinline__ double window_dist2_any(const float* __restrict__ mirror, int img_w,
                                                   int C, int w, int ax, int ay,
                                                   const float* __restrict__ ex_mirror,
                                                   const float* __restrict__ ex8, int ew, int ex,
                                                   int ey) {
  if (ex8 && C == 5) return window_dist2_pad<5>(mirror, img_w, w, ax, ay, ex8, ew, ex, ey);
  if (ex8 && C == 4) return window_dist2_pad<4>(mirror, img_w, w, ax, ay, ex8, ew, ex, ey);
  return window_dist2(mirror, img_w, C, w, ax, ay, ex_mirror, ew, ex, ey);
}

__global__ void rescore_windows_kernel(const float* __restrict__ mirror, int img_w, int C, int w,
                                       const int32_t* __restrict__ xs,
                                       const int32_t* __restrict__ ys, int nx, int64_t n,
                                       const float* __restrict__ ex_mirror,
                                       const float* __restrict__ ex8, int ew, int nxe,
                                       const int32_t* __restrict__ idx,
                                       double* __restrict__ dist) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = idx[a];
    dist[a] = sqrt(window_dist2_any(mirror, img_w, C, w, xs[a % nx], ys[a / nx], ex_mirror, ex8,
                                    ew, id % nxe, id / nxe));
  }
}

// Rescoring after a search seeded with prev_idx on the SAME image: an anchor
// whose assignment did not change has the distance prev_dist already (the
// lsq-after diagnostic computed it: same window, same candidate, same chain),
// so only the changed anchors (~5% once EM settles) are recomputed: they are
// listed (warp-aggregated) and a thread per listed anchor runs the reference's
// chain (a warp per anchor with one lane adding the staged squares measured
// ~3x slower: the 320-step fp64 chain is the latency, not the loads).
constexpr int kRescoreBlock = 256;
__global__ void __launch_bounds__(kRescoreBlock) rescore_mark_kernel(
    int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ prev_idx,
    const double* __restrict__ prev_dist, double* __restrict__ dist, int32_t* __restrict__ list,
    int* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  for (int64_t a0 = blockIdx.x * (int64_t)blockDim.x; a0 < n; a0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = a0 + threadIdx.x;
    bool todo = false;
    if (a < n) {
      if (idx[a] == prev_idx[a])
        dist[a] = prev_dist[a];
      else
        todo = true;
    }
    const unsigned m = __ballot_sync(0xffffffffu, todo);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (todo) list[base + __popc(m & ((1u << lane) - 1u))] = (int32_t)a;
  }
}

// One thread per listed (changed) anchor: all lanes run a chain (the listed
// anchors are compacted globally, so warps are full even when few anchors
// changed).
__global__ void __maxnreg__(168) rescore_list_kernel(
    const float* __restrict__ mirror, int img_w, int C, int w, const int32_t* __restrict__ xs,
    const int32_t* __restrict__ ys, int nx, const float* __restrict__ ex_mirror,
    const float* __restrict__ ex8, int ew, int nxe, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ list, const int* __restrict__ count, double* __restrict__ dist) {
  const int n = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t b = list[i];
    const int32_t id = idx[b];
    const int ax = xs[b % nx], ay = ys[b / nx], ex = id % nxe, ey = id / nxe;
    double d2;
    if (ex8 && w == 8 && C == 5)
      d2 = window_dist2_pad_rows8<5>(mirror, img_w, ax, ay, ex8, ew, ex, ey);
    else if (ex8 && w == 8 && C == 4)
      d2 = window_dist2_pad_rows8<4>(mirror, img_w, ax, ay, ex8, ew, ex, ey);
    else
      d2 = window_dist2_any(mirror, img_w, C, w, ax, ay, ex_mirror, ex8, ew, ex, ey);
    dist[b] = sqrt(d2);
  }
}

void launch_rescore_windows(psg_ctx* ctx, const float* mirror, int img_w, int C, int w,
                            AnchorSet anchors, const Index& ix, const int32_t* idx,
                            double* dist, const int32_t* prev_idx, const double* prev_dist,
                            int32_t* list, int* count) {
  ProfScope _prof(ctx, K_RESCORE);
  if (anchors.count <= 0) return;
  const float* ex8 = ctx->knobs.no_ex8 ? nullptr : ix.ex_mirror8;
  if (prev_idx && prev_dist) {
    if (!list || !count) fail(PSG_E_LOGIC, "changed-only rescoring without its list buffers");
    PSG_CUDA(cudaMemsetAsync(count, 0, sizeof(int), ctx->stream));
    int64_t blocks = (anchors.count + kRescoreBlock - 1) / kRescoreBlock;
    if (blocks > (int64_t)ctx->num_sms * 8) blocks = (int64_t)ctx->num_sms * 8;
    rescore_mark_kernel<<<(unsigned)blocks, kRescoreBlock, 0, ctx->stream>>>(anchors.count, idx, prev_idx,
                                                                            prev_dist, dist, list, count);
    PSG_LAUNCHED(ctx);
    rescore_list_kernel<<<ctx->num_sms * 8, 128, 0, ctx->stream>>>(
        mirror, img_w, C, w, anchors.xs, anchors.ys, anchors.nx, ix.ex_mirror, ex8, ix.ew, ix.nxe, idx,
        list, count, dist);
    PSG_LAUNCHED(ctx);
    return;
  }
  const int threads = 128;
  int64_t blocks = (anchors.count + threads - 1) / threads;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  rescore_windows_kernel<<<(int)blocks, threads, 0, ctx->stream>>>(
      mirror, img_w, C, w, anchors.xs, anchors.ys, anchors.nx, anchors.count, ix.ex_mirror, ex8,
      ix.ew, ix.nxe, idx, dist);
  PSG_LAUNCHED(ctx);
}

// Explicit query vectors against a window index's candidates (batched
// PcaTreeIndex::nearest rescoring, optimizer.cpp:232-234): the candidate
// window is read from the exemplar mirror in (dy, dx, c) order.
__global__ void rescore_query_windows_kernel(const float* __restrict__ Q, int64_t nq, int C, int w,
                                             const float* __restrict__ ex_mirror, int ew, int nxe,
                                             const int32_t* __restrict__ idx,
                                             double* __restrict__ dist) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nq;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = idx[a];
    const int ex = id % nxe, ey = id / nxe;
    const int row = w * C;
    const float* v = Q + a * (int64_t)row * w;
    double acc = 0.0;
    for (int dy = 0; dy < w; ++dy) {
      const float* z = ex_mirror + ((int64_t)(ey + dy) * ew + ex) * C;
      for (int jj = 0; jj < row; ++jj) {
        const double t = dsub((double)v[dy * row + jj], (double)z[jj]);
        acc = dadd(acc, dmul(t, t));
      }
    }
    dist[a] = sqrt(acc);
  }
}

void launch_rescore_query_windows(psg_ctx* ctx, const float* Q, int64_t nq, const Index& ix,
                                  const int32_t* idx, double* dist) {
  ProfScope _prof(ctx, K_RESCORE);
  if (nq <= 0) return;
  const int threads = 128;
  int64_t blocks = (nq + threads - 1) / threads;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  rescore_query_windows_kernel<<<(int)blocks, threads, 0, ctx->stream>>>(
      Q, nq, ix.C, ix.w, ix.ex_mirror, ix.ew, ix.nxe, idx, dist);
  PSG_LAUNCHED(ctx);
}

__global__ void rescore_vectors_kernel(const float* __restrict__ Q, int64_t nq, int D,
                                       const float* __restrict__ X,
                                       const int32_t* __restrict__ idx,
                                       double* __restrict__ dist) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nq;
       a += (int64_t)gridDim.x * blockDim.x) {
    const float* v = Q + a * D;
    const float* z = X + (int64_t)idx[a] * D;
    double acc = 0.0;
    for (int j = 0; j < D; ++j) {
      const double t = dsub((double)v[j], (double)z[j]);
      acc = dadd(acc, dmul(t, t));
    }
    dist[a] = sqrt(acc);
  }
}

void launch_rescore_vectors(psg_ctx* ctx, const float* Q, int64_t nq, const Index& ix,
                            const int32_t* idx, double* dist) {
  ProfScope _prof(ctx, K_RESCORE);
  if (nq <= 0) return;
  const int threads = 128;
  int64_t blocks = (nq + threads - 1) / threads;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  rescore_vectors_kernel<<<(int)blocks, threads, 0, ctx->stream>>>(Q, nq, ix.D, ix.vectors, idx,
                                                                    dist);
  PSG_LAUNCHED(ctx);
}

// ----------------------------------------------------------------------------
// proj [N][d] (original order) -> soa [d][N] in leaf order.
__global__ void gather_soa_kernel(const double* __restrict__ proj, int64_t N, int d,
                                  const int32_t* __restrict__ perm, double* __restrict__ soa) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i / N);
    const int64_t pos = i - (int64_t)j * N;
    soa[i] = proj[(int64_t)perm[pos] * d + j];
  }
}

void launch_gather_soa(psg_ctx* ctx, const double* proj, int64_t N, int d, const int32_t* perm,
                       double* soa) {
  ProfScope _prof(ctx, K_BUILD);
  if (N <= 0 || d <= 0) return;
  int64_t blocks = (N * d + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  gather_soa_kernel<<<(int)blocks, 256, 0, ctx->stream>>>(proj, N, d, perm, soa);
  PSG_LAUNCHED(ctx);
}

}  // namespace psg
