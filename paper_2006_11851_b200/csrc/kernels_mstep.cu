// M-step kernels: IRLS weights, exact histograms + penalty, the gather-form
// overlapping-window average, and deterministic telemetry reductions.
//
// Reference semantics (paths under /root/reference/proj/core/src):
//   irls_weight          optimizer.cpp:112-115  pow(d*d + eps, (r-2)/2)
//   WeightMap::effective optimizer.hpp:32-34    irls / (1 + penalty)
//   build_histograms     optimizer.cpp:69-88    mass[b] += 1/P per pixel
//   histogram_penalty    optimizer.cpp:90-108   sum_p sum_s max(0, Hx-Hz) / w^2
//   update_step          optimizer.cpp:350-401  per pixel, ascending anchors
//   energy_from_distances optimizer.cpp:126-131
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "numerics.cuh"
#include "psg_internal.h"

namespace psg {

static int grid_for(psg_ctx* ctx, int64_t n, int threads, int per_sm = 32) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)ctx->num_sms * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// ---- IRLS weights ---------------------------------------------------------------
__global__ void weights_kernel(WeightArgs a) {
  const double e = (a.r - 2.0) / 2.0;  // same expression as optimizer.cpp:114
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.A;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = a.dist[i];
    if (d < 0.0) atomicOr(a.flags, FLAG_BAD_DISTANCE);
    const double w = pow_cr(dadd(dmul(d, d), a.eps), e);
    a.irls[i] = w;
    const double p = a.pen ? a.pen[i] : 0.0;
    const double we = w / dadd(1.0, p);
    a.eff[i] = we;
    if (!(we > 0.0) || !isfinite(we)) atomicOr(a.flags, FLAG_BAD_WEIGHT);
  }
}

void launch_weights(psg_ctx* ctx, const WeightArgs& a) {
  ProfScope _prof(ctx, K_WEIGHTS);
  if (a.A <= 0) return;
  weights_kernel<<<grid_for(ctx, a.A, 256), 256, 0, ctx->stream>>>(a);
  PSG_LAUNCHED(ctx);
}

__global__ void eff_kernel(const double* __restrict__ irls, const double* __restrict__ pen,
                           int64_t A, double* __restrict__ eff, int* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double we = irls[i] / dadd(1.0, pen[i]);
    eff[i] = we;
    if (!(we > 0.0) || !isfinite(we)) atomicOr(flags, FLAG_BAD_WEIGHT);
  }
}

void launch_eff_from(psg_ctx* ctx, const double* irls, const double* pen, int64_t A, double* eff,
                     int* flags) {
  ProfScope _prof(ctx, K_WEIGHTS);
  if (A <= 0) return;
  eff_kernel<<<grid_for(ctx, A, 256), 256, 0, ctx->stream>>>(irls, pen, A, eff, flags);
  PSG_LAUNCHED(ctx);
}

// ---- histograms -------------------------------------------------------------------
// Integer bin counts (exact, order-free), then the exact sequential-sum fold.
__global__ void hist_count_kernel(const double* __restrict__ planes, int64_t P, int64_t stride,
                                  int bins, int slots, unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned int sh[];
  for (int i = threadIdx.x; i < bins * slots; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < slots; ++s) {
      const int b = bin_of_f64(planes[s * stride + i], bins);
      atomicAdd(&sh[s * bins + b], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bins * slots; i += blockDim.x)
    if (sh[i]) atomicAdd(&counts[i], (unsigned long long)sh[i]);
}

void launch_hist_count(psg_ctx* ctx, const double* planes, int64_t P, int64_t stride, int bins,
                       int slots, unsigned long long* counts) {
  ProfScope _prof(ctx, K_HIST);
  PSG_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * bins * slots, ctx->stream));
  const size_t sm = sizeof(unsigned int) * bins * slots;
  hist_count_kernel<<<grid_for(ctx, P, 256, 4), 256, sm, ctx->stream>>>(planes, P, stride, bins,
                                                                         slots, counts);
  PSG_LAUNCHED(ctx);
}

__global__ void hist_fold_kernel(const unsigned long long* __restrict__ counts, int n, int64_t P,
                                 const double* __restrict__ ex_mass, double* __restrict__ mass,
                                 double* __restrict__ excess) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double inv = 1.0 / (double)P;  // optimizer.cpp:76
  const double m = hist_mass((int64_t)counts[i], inv);
  if (mass) mass[i] = m;
  if (excess) {
    const double diff = dsub(m, ex_mass[i]);  // optimizer.cpp:104
    excess[i] = diff > 0.0 ? diff : 0.0;
  }
}

void launch_hist_fold(psg_ctx* ctx, const unsigned long long* counts, int bins, int slots,
                      int64_t P, const double* ex_mass, double* mass, double* excess) {
  ProfScope _prof(ctx, K_HIST);
  const int n = bins * slots;
  hist_fold_kernel<<<(n + 63) / 64, 64, 0, ctx->stream>>>(counts, n, P, ex_mass, mass, excess);
  PSG_LAUNCHED(ctx);
}

// Penalty of each anchor's assigned candidate (optimizer.cpp:463-467): the
// candidate's values are the exemplar window at the candidate anchor; pixels
// in window order (dy, dx), slots inner, one sequential fp64 sum per anchor.
__global__ void penalty_kernel(const float* __restrict__ ex_mirror, int ew, int C, int w, int nxe,
                               const int32_t* __restrict__ idx, int64_t A,
                               const double* __restrict__ excess, int bins, int slots,
                               double* __restrict__ pen) {
  extern __shared__ double ex_s[];
  for (int i = threadIdx.x; i < bins * slots; i += blockDim.x) ex_s[i] = excess[i];
  __syncthreads();
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < A;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = idx[a];
    const int ex = id % nxe, ey = id / nxe;
    double total = 0.0;
    for (int dy = 0; dy < w; ++dy) {
      const float* z = ex_mirror + ((int64_t)(ey + dy) * ew + ex) * C;
      for (int dx = 0; dx < w; ++dx)
        for (int s = 0; s < slots; ++s) {
          const int b = bin_of_f32(z[dx * C + s], bins);
          total = dadd(total, ex_s[s * bins + b]);
        }
    }
    pen[a] = total / (double)(w * w);
  }
}

void launch_penalty(psg_ctx* ctx, const Index& ix, const int32_t* idx, int64_t A,
                    const double* excess, int bins, int slots, double* pen) {
  ProfScope _prof(ctx, K_PENALTY);
  if (A <= 0) return;
  const size_t sm = sizeof(double) * bins * slots;
  penalty_kernel<<<grid_for(ctx, A, 128), 128, sm, ctx->stream>>>(
      ix.ex_mirror, ix.ew, ix.C, ix.w, ix.nxe, idx, A, excess, bins, slots, pen);
  PSG_LAUNCHED(ctx);
}

// The penalty depends on the candidate only: one table entry per exemplar
// window (N ids) replaces the per-anchor sums (A ~ 4N at sp = 2), and
// consecutive threads read consecutive exemplar pixels (coalesced), where the
// per-anchor form gathers one random window per thread.  Same sequential sum
// per entry as penalty_kernel, so table[idx[a]] is bit-identical to pen[a].
template <int NS>  // NS > 0: compile-time histogram slot count
__global__ void penalty_table_kernel(const float* __restrict__ ex_mirror, int ew, int C, int w,
                                     int nxe, int64_t N, const double* __restrict__ excess,
                                     int bins, int slots_, double* __restrict__ table) {
  extern __shared__ double ex_s[];
  const int slots = NS > 0 ? NS : slots_;
  for (int i = threadIdx.x; i < bins * slots; i += blockDim.x) ex_s[i] = excess[i];
  __syncthreads();
  const double area = (double)(w * w);
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < N;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int ex = (int)(id % nxe), ey = (int)(id / nxe);
    double total = 0.0;
    for (int dy = 0; dy < w; ++dy) {
      const float* z = ex_mirror + ((int64_t)(ey + dy) * ew + ex) * C;
      int dx = 0;
      if constexpr (NS > 0) {
        // 4 pixels' loads and bins ahead of their sequential adds
        for (; dx + 4 <= w; dx += 4) {
          int b[4 * NS];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int s = 0; s < NS; ++s)
              b[u * NS + s] = s * bins + bin_of_f32(__ldg(z + (dx + u) * C + s), bins);
#pragma unroll
          for (int k = 0; k < 4 * NS; ++k) total = dadd(total, ex_s[b[k]]);
        }
      }
      for (; dx < w; ++dx)
        for (int s = 0; s < slots; ++s) {
          const int b = bin_of_f32(__ldg(z + dx * C + s), bins);
          total = dadd(total, ex_s[s * bins + b]);
        }
    }
    table[id] = total / area;
  }
}

void launch_penalty_table(psg_ctx* ctx, const Index& ix, const double* excess, int bins,
                          int slots, double* table) {
  ProfScope _prof(ctx, K_PENALTY);
  if (ix.N <= 0) return;
  const size_t sm = sizeof(double) * bins * slots;
  auto k = slots == 3 ? penalty_table_kernel<3> : penalty_table_kernel<0>;
  k<<<grid_for(ctx, ix.N, 128), 128, sm, ctx->stream>>>(ix.ex_mirror, ix.ew, ix.C, ix.w, ix.nxe,
                                                        ix.N, excess, bins, slots, table);
  PSG_LAUNCHED(ctx);
}

// pen[a] = table[idx[a]]; eff[a] = irls[a] / (1 + pen[a]) (optimizer.hpp:32-34).
__global__ void eff_gather_kernel(const double* __restrict__ irls,
                                  const double* __restrict__ table,
                                  const int32_t* __restrict__ idx, int64_t A,
                                  double* __restrict__ pen, double* __restrict__ eff, int* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double p = table[idx[i]];
    pen[i] = p;
    const double we = irls[i] / dadd(1.0, p);
    eff[i] = we;
    if (!(we > 0.0) || !isfinite(we)) atomicOr(flags, FLAG_BAD_WEIGHT);
  }
}

void launch_eff_gather(psg_ctx* ctx, const double* irls, const double* table, const int32_t* idx,
                       int64_t A, double* pen, double* eff, int* flags) {
  ProfScope _prof(ctx, K_WEIGHTS);
  if (A <= 0) return;
  eff_gather_kernel<<<grid_for(ctx, A, 256), 256, 0, ctx->stream>>>(irls, table, idx, A, pen, eff,
                                                                    flags);
  PSG_LAUNCHED(ctx);
}

// ---- M-step: gather form ----------------------------------------------------------
// The reference scatters anchors in ascending id into per-pixel accumulators;
// for a fixed pixel that is exactly the ascending (iy, ix) order of its
// covering anchors, which the gather walks.  No atomics, bit-identical sums.
//
// A CTA owns 32 x 8 output pixels (a warp = 32 consecutive pixels of a row):
// the (eff, exemplar offset) of every anchor covering the tile is formed once
// into shared memory -- the candidate id split into exemplar coordinates and
// the anchor position folded into one offset zb, so the candidate pixel of
// pixel (x, y) is zb + y * ew + x -- and each pixel then reads its covering
// anchors from there.  Interior pixels (w / spacing = 4: exactly 4 x 4 covering
// anchors) load all 16 entries and their candidate pixels eight at a time
// ahead of the sequential fp64 chain; edge pixels walk the general ranges.
// NC > 0: compile-time channel count; NC = 0: any C <= 8.
struct MstepEntry {
  double we;
  int32_t zb;
  int32_t pad;
};
constexpr int kMstepTX = 32, kMstepTY = 8;

__host__ __device__ inline int mstep_span(int tile, int w, int sp) { return (tile + w - 2) / sp + 2; }

template <int NC>
__global__ void __launch_bounds__(256) mstep_kernel(MstepArgs a) {
  constexpr int CMAX = NC > 0 ? NC : 8;
  const int C = NC > 0 ? NC : a.C;
  extern __shared__ __align__(16) unsigned char mstep_smem[];
  const int cap_r = mstep_span(kMstepTY, a.w, a.sp), cap_c = mstep_span(kMstepTX, a.w, a.sp);
  MstepEntry* ent = reinterpret_cast<MstepEntry*>(mstep_smem);
  // per warp: its 32 pixels' fp32 mirror values [32][C], stored as whole lines
  float* mir_s = reinterpret_cast<float*>(ent + cap_r * cap_c) + (threadIdx.x >> 5) * 32 * CMAX;
  unsigned int* hist_s = reinterpret_cast<unsigned int*>(ent + cap_r * cap_c) + 8 * 32 * CMAX;
  if (a.counts)
    for (int i = threadIdx.x; i < a.bins * a.slots; i += blockDim.x) hist_s[i] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t PS = (int64_t)a.W * a.plane_rows;  // plane stride (band: rows >= H)
  const int tnx = (a.W + kMstepTX - 1) / kMstepTX;
  const int n_tiles = tnx * ((a.H + kMstepTY - 1) / kMstepTY);
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int x0 = (t % tnx) * kMstepTX, y0 = (t / tnx) * kMstepTY;
    const int x1 = min(x0 + kMstepTX, a.W) - 1, y1 = min(y0 + kMstepTY, a.H) - 1;
    const int r0 = a.row_lo[y0], c0 = a.col_lo[x0];
    const int nr = a.row_hi[y1] - r0, ncl = a.col_hi[x1] - c0;
    __syncthreads();  // the previous tile's entries are consumed
    if (nr > cap_r || ncl > cap_c) {  // cannot happen: spans bounded by mstep_span
      if (threadIdx.x == 0) atomicOr(a.flags, FLAG_STACK_OVERFLOW);
      continue;
    }
    for (int e = threadIdx.x; e < nr * ncl; e += blockDim.x) {
      const int iy = r0 + e / ncl, ix = c0 + e % ncl;
      const int64_t ai = (int64_t)iy * a.nx + ix;
      const int32_t id = __ldg(a.idx + ai);
      const int ey = id / a.nxe, ex = id - ey * a.nxe;
      MstepEntry m;
      m.we = __ldg(a.eff + ai);
      m.zb = (ey - a.ys[iy]) * a.ew + ex - a.xs[ix];
      m.pad = 0;
      ent[e] = m;
    }
    __syncthreads();
    const int x = x0 + lane, y = y0 + warp;
    if (y >= a.H) continue;  // warp-uniform
    const int64_t pix = (int64_t)y * a.W + x;
    // the warp's mirror row segment [x0, x0 + nw) is stored cooperatively
    // after the pixel loop: C contiguous floats per pixel, lanes on
    // consecutive words (the per-pixel stride-C stores wasted ~4/5 of every
    // sector)
    const int nw = min(32, a.W - x0);
    if (x < a.W) {
    const int base = y * a.ew + x;
    double acc[CMAX];
#pragma unroll
    for (int c = 0; c < CMAX; ++c) acc[c] = 0.0;
    double wsum = 0.0;
    const int iy0 = a.row_lo[y] - r0, iy1 = a.row_hi[y] - r0;
    const int ix0 = a.col_lo[x] - c0, ix1 = a.col_hi[x] - c0;
    if (NC > 0 && a.ex8 && iy1 - iy0 == 4 && ix1 - ix0 == 4) {
      double we[16];
      int32_t zp[16];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const MstepEntry m = ent[(iy0 + r) * ncl + ix0 + c];
          we[r * 4 + c] = m.we;
          zp[r * 4 + c] = m.zb + base;
        }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 z0[8], z1[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float* zr = a.ex8 + (int64_t)zp[h * 8 + k] * 8;
          if (NC > 4) {
            ldg256(zr, z0[k], z1[k]);
          } else {
            z0[k] = __ldg(reinterpret_cast<const float4*>(zr));
            z1[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double w = we[h * 8 + k];
          const float zc[8] = {z0[k].x, z0[k].y, z0[k].z, z0[k].w,
                               z1[k].x, z1[k].y, z1[k].z, z1[k].w};
#pragma unroll
          for (int c = 0; c < CMAX; ++c) acc[c] = dadd(acc[c], dmul(w, (double)zc[c]));
          wsum = dadd(wsum, w);
        }
      }
    } else {
      for (int iy = iy0; iy < iy1; ++iy)
        for (int ix = ix0; ix < ix1; ++ix) {
          const MstepEntry m = ent[iy * ncl + ix];
          const int64_t zq = (int64_t)m.zb + base;
          float zv[CMAX];
          if (NC > 0 && a.ex8) {  // 32-byte padded pixel: two 16-byte loads
            float4 z0, z1;
            ldg256(a.ex8 + zq * 8, z0, z1);
            const float zc[8] = {z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w};
#pragma unroll
            for (int c = 0; c < CMAX; ++c) zv[c] = zc[c];
          } else {
            const float* z = a.ex_mirror + zq * C;
#pragma unroll
            for (int c = 0; c < CMAX; ++c) zv[c] = (NC > 0 || c < C) ? __ldg(z + c) : 0.f;
          }
#pragma unroll
          for (int c = 0; c < CMAX; ++c)
            if (NC > 0 || c < C) acc[c] = dadd(acc[c], dmul(m.we, (double)zv[c]));
          wsum = dadd(wsum, m.we);
        }
    }
    if (wsum <= 0.0) {
      atomicOr(a.flags, FLAG_UNCOVERED);
      wsum = 1.0;  // flagged: the call fails; keep the warp together for the stores
    }
    const double inv = 1.0 / wsum;  // optimizer.cpp:393
#pragma unroll
    for (int c = 0; c < CMAX; ++c) {
      if (NC == 0 && c >= C) break;
      double v = dmul(acc[c], inv);
      v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);  // std::clamp(.., 0, 1)
      a.planes[c * PS + pix] = v;
      mir_s[lane * C + c] = (float)v;
      if (a.counts && c < a.slots) {
        // lanes with the same bin add once (neighbouring pixels share bins:
        // unaggregated shared-memory atomics serialise)
        const int key = c * a.bins + bin_of_f64(v, a.bins);
        const unsigned peers = __match_any_sync(__activemask(), key);
        if (lane == __ffs(peers) - 1) atomicAdd(&hist_s[key], (unsigned)__popc(peers));
      }
    }
    }  // x < W
    __syncwarp();
    if (a.mirror) {
      float* dst = a.mirror + ((int64_t)y * a.W + x0) * C;
      for (int f = lane; f < nw * C; f += 32) dst[f] = mir_s[f];
    }
    __syncwarp();
  }
  if (a.counts) {  // same integer counts as hist_count_kernel over the written rows
    __syncthreads();
    for (int i = threadIdx.x; i < a.bins * a.slots; i += blockDim.x)
      if (hist_s[i]) atomicAdd(&a.counts[i], (unsigned long long)hist_s[i]);
  }
}

template <int NC>
static int mstep_blocks_per_sm(size_t sm) {
  int n = 0;
  PSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mstep_kernel<NC>, 256, sm));
  return n < 1 ? 1 : n;
}

void launch_mstep(psg_ctx* ctx, const MstepArgs& a) {
  ProfScope _prof(ctx, K_MSTEP);
  const int64_t P = (int64_t)a.W * a.H;
  if (P <= 0) return;
  if (a.C > 8) fail(PSG_E_DOMAIN, "more than 8 channels are not supported");
  if (a.sp < 1) fail(PSG_E_LOGIC, "M-step without the grid spacing");
  size_t sm = sizeof(MstepEntry) * mstep_span(kMstepTY, a.w, a.sp) * mstep_span(kMstepTX, a.w, a.sp) +
              sizeof(float) * 8 * 32 * (a.C == 4 ? 4 : a.C == 5 ? 5 : 8);
  if (a.counts) {
    if (a.slots > a.C) fail(PSG_E_DOMAIN, "histogram slots exceed the channel count");
    sm += sizeof(unsigned int) * a.bins * a.slots;
    PSG_CUDA(cudaMemsetAsync(a.counts, 0, sizeof(unsigned long long) * a.bins * a.slots,
                             ctx->stream));
  }
  if (sm > 48 * 1024) fail(PSG_E_DOMAIN, "M-step tile footprint exceeds 48 KB of shared memory");
  const int64_t tiles = (int64_t)((a.W + kMstepTX - 1) / kMstepTX) * ((a.H + kMstepTY - 1) / kMstepTY);
  // persistent CTAs striding over the tiles: the histogram flush (one per
  // CTA) and the barrier tail are paid per resident CTA, not per tile
  auto blocks = [&](int per_sm) { return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)per_sm * ctx->num_sms)); };
  switch (a.C) {
    case 4: mstep_kernel<4><<<blocks(mstep_blocks_per_sm<4>(sm)), 256, sm, ctx->stream>>>(a); break;
    case 5: mstep_kernel<5><<<blocks(mstep_blocks_per_sm<5>(sm)), 256, sm, ctx->stream>>>(a); break;
    default: mstep_kernel<0><<<blocks(mstep_blocks_per_sm<0>(sm)), 256, sm, ctx->stream>>>(a); break;
  }
  PSG_LAUNCHED(ctx);
}

// ---- deterministic telemetry reductions ---------------------------------------------
// Two passes with a fixed partition and fixed trees (run-to-run identical):
// kStatsBlocks CTAs reduce contiguous anchor ranges, one CTA folds the partials.
constexpr int kStatsThreads = 256;
constexpr int kStatsBlocks = 296;

__global__ void __launch_bounds__(kStatsThreads) stats_partial_kernel(StatsArgs a,
                                                                      double* __restrict__ part) {
  __shared__ double sd[3][kStatsThreads];
  __shared__ long long si[3][kStatsThreads];
  const int64_t chunk = (a.A + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk;
  const int64_t hi = min(a.A, lo + chunk);
  double lb = 0.0, la = 0.0, en = 0.0;
  long long ch = 0, sp = 0, su = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    if (a.eff && a.cur_dist) {
      const double d = a.cur_dist[i];
      lb = dadd(lb, dmul(dmul(a.eff[i], d), d));  // optimizer.cpp:473
    }
    if (a.eff && a.after_dist) {
      const double d = a.after_dist[i];
      la = dadd(la, dmul(dmul(a.eff[i], d), d));  // optimizer.cpp:482
    }
    // energy sum d^r (optimizer.cpp:129): a telemetry value with a 1e-4
    // tolerance (the summation order differs anyway), so CUDA's pow (< 2 ulp)
    // instead of the correctly rounded one the IRLS weights need
    if (a.next_dist) en = dadd(en, pow(a.next_dist[i], a.r));
    if (a.cur_idx && a.next_idx) ch += a.cur_idx[i] != a.next_idx[i];
    if (a.scanned) {
      su += a.scanned[i];
      sp += (long long)a.scanned[i] * (a.mult ? a.mult[i] : 1);
    }
  }
  const int t = threadIdx.x;
  sd[0][t] = lb;
  sd[1][t] = la;
  sd[2][t] = en;
  si[0][t] = ch;
  si[1][t] = sp;
  si[2][t] = su;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) {
      for (int k = 0; k < 3; ++k) sd[k][t] = dadd(sd[k][t], sd[k][t + s]);
      for (int k = 0; k < 3; ++k) si[k][t] += si[k][t + s];
    }
    __syncthreads();
  }
  if (t == 0) {
    double* o = part + blockIdx.x * 6;
    o[0] = sd[0][0];
    o[1] = sd[1][0];
    o[2] = sd[2][0];
    o[3] = (double)si[0][0];
    o[4] = (double)si[1][0];
    o[5] = (double)si[2][0];
  }
  // the last CTA to finish folds the partials in a fixed order (
  // run-to-run identical); the ticket re-arms itself for the next launch
  __shared__ bool last;
  if (t == 0) {
    __threadfence();
    const unsigned long long prev = atomicAdd(a.ticket, 1ull);
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nb = gridDim.x;
  // fixed two-level fold: thread t sums blocks t, t + 256, ... then the tree
  double f0 = 0.0, f1 = 0.0, f2 = 0.0;
  long long g0 = 0, g1 = 0, g2 = 0;
  for (int b = t; b < nb; b += blockDim.x) {
    const double* o = part + b * 6;
    f0 = dadd(f0, __ldcg(o + 0));
    f1 = dadd(f1, __ldcg(o + 1));
    f2 = dadd(f2, __ldcg(o + 2));
    g0 += (long long)__ldcg(o + 3);
    g1 += (long long)__ldcg(o + 4);
    g2 += (long long)__ldcg(o + 5);
  }
  sd[0][t] = f0;
  sd[1][t] = f1;
  sd[2][t] = f2;
  si[0][t] = g0;
  si[1][t] = g1;
  si[2][t] = g2;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) {
      for (int k = 0; k < 3; ++k) sd[k][t] = dadd(sd[k][t], sd[k][t + s]);
      for (int k = 0; k < 3; ++k) si[k][t] += si[k][t + s];
    }
    __syncthreads();
  }
  if (t < 3) a.out[t] = sd[t][0];
  if (t >= 3 && t < 6) a.out[t] = (double)si[t - 3][0];
  if (t == 0) *a.ticket = 0ull;
}

void launch_stats(psg_ctx* ctx, const StatsArgs& a) {
  ProfScope _prof(ctx, K_STATS);
  const int nb = (int)std::min<int64_t>(kStatsBlocks, std::max<int64_t>(1, (a.A + 255) / 256));
  StatsArgs b = a;
  if (!b.ticket) b.ticket = reinterpret_cast<unsigned long long*>(ctx->d_sched + 2);
  stats_partial_kernel<<<nb, kStatsThreads, 0, ctx->stream>>>(b, a.out + 8);
  PSG_LAUNCHED(ctx);
}

}  // namespace psg
