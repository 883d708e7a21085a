// Exact tree search with the (query x point) filter on the 5th-generation
// tensor cores (tcgen05 / TMEM), sm_100a.
//
// A CTA owns 128 queries (a 16 x 8 anchor tile; one query per thread) that
// share one depth-first traversal of the k-means tree, like
// search_tile_kernel.  Leaf points are staged 128 at a time in shared memory
// and ONE elected thread issues UMMAs
//     D[128 x 128] (fp32, TMEM) = Qhi.Phi^T + Qhi.Plo^T + Qlo.Phi^T
// where x = hi + lo is a two-term bf16 split of the fp32 PCA coordinates
// (K = 32 or 64).  Each thread then reads its query's row of D with
// tcgen05.ld and forms s = |q|^2 + |p|^2 - 2 q.p.  A rigorous bound on
// |s - exact dist^2| (split residual, fp32 accumulation, epilogue rounding:
// DESIGN.md §4) keeps every point that can still beat the thread's best; only
// those are re-evaluated with the reference's exact fp64 j-sequential chain
// (km_tree.cpp:15-22), so the result is the exact lexicographic minimum of
// (fp64 dist^2, id) — bit-identical to KmTree exact / brute force.
//
// Operands use the no-swizzle K-major canonical layout: 8-row x 16-byte core
// matrices; LBO = 128 B between the two K-halves of one UMMA step (K = 16),
// SBO = 128 * K/8 B between 8-row groups.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "numerics.cuh"
#include "psg_internal.h"
#include "umma.cuh"

namespace psg {


constexpr int kMmaM = 128;      // queries per CTA
constexpr int kMmaN = 128;      // staged points per UMMA batch
constexpr int kMmaStack = 48;
constexpr int kMmaMaxB = 16;

__device__ __forceinline__ double dist2_seq_mma(const double* __restrict__ q,
                                                const double* __restrict__ p, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = dsub(q[j], p[j]);
    acc = dadd(acc, dmul(t, t));
  }
  return acc;
}

struct MmaSmem {
  // offsets (bytes) into the dynamic shared memory block
  uint32_t a_hi, a_lo, b_hi, b_lo, pn2, pnorm, pid, cst, caux, cmeta, cbox, st_meta, st_lb, tlb,
      tkey, wkey, misc, total;
};

template <int DP>
__host__ __device__ constexpr MmaSmem mma_smem_layout() {
  MmaSmem s{};
  uint32_t o = 0;
  const uint32_t op = kMmaM * DP * 2;  // one bf16 operand tile
  s.a_hi = o; o += op;
  s.a_lo = o; o += op;
  s.b_hi = o; o += kMmaN * DP * 2;
  s.b_lo = o; o += kMmaN * DP * 2;
  s.pn2 = o; o += kMmaN * 4;
  s.pnorm = o; o += kMmaN * 4;
  s.pid = o; o += kMmaN * 4;
  s.cst = o; o += kMmaMaxB * (DP + 4) * 4;
  s.caux = o; o += 2 * kMmaMaxB * 4;
  s.cmeta = o; o += kMmaMaxB * 8;
  s.cbox = o; o += kMmaMaxB * 2 * kBoxDims * 4;
  s.st_meta = o; o += kMmaStack * 8;
  s.st_lb = o; o += kMmaStack * kMmaM * 4;
  s.tlb = o; o += kMmaMaxB * kMmaM * 4;
  s.tkey = o; o += kMmaMaxB * 4;
  s.wkey = o; o += 4 * kMmaMaxB * 4;
  s.misc = o; o += 64;  // mbarrier (8 B) + tmem base (4 B)
  s.total = o;
  return s;
}

template <int DP>
__global__ void __launch_bounds__(kMmaM, 1) search_mma_kernel(SearchArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr MmaSmem L = mma_smem_layout<DP>();
  constexpr int RS = DP + 4;
  uint8_t* a_hi = smem + L.a_hi;
  uint8_t* a_lo = smem + L.a_lo;
  uint8_t* b_hi = smem + L.b_hi;
  uint8_t* b_lo = smem + L.b_lo;
  float* pn2_s = reinterpret_cast<float*>(smem + L.pn2);
  float* pnorm_s = reinterpret_cast<float*>(smem + L.pnorm);
  int32_t* pid_s = reinterpret_cast<int32_t*>(smem + L.pid);
  float* cst = reinterpret_cast<float*>(smem + L.cst);
  float* caux = reinterpret_cast<float*>(smem + L.caux);
  int2* cmeta = reinterpret_cast<int2*>(smem + L.cmeta);
  float* cbox = reinterpret_cast<float*>(smem + L.cbox);
  int2* st_meta = reinterpret_cast<int2*>(smem + L.st_meta);
  float* st_lb = reinterpret_cast<float*>(smem + L.st_lb);  // [S][128]
  float* tlb = reinterpret_cast<float*>(smem + L.tlb);      // [16][128]
  uint32_t* tkey = reinterpret_cast<uint32_t*>(smem + L.tkey);
  uint32_t* wkey = reinterpret_cast<uint32_t*>(smem + L.wkey);  // [4][16]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.misc);
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(smem + L.misc + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int d = a.d;
  const int N = (int)a.N;
  const int nn = a.tree.n_nodes;
  const int KB = d < kBoxDims ? d : kBoxDims;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const float kInfF = __int_as_float(0x7f800000);
  constexpr uint32_t kIdesc = mma::make_idesc(kMmaM, kMmaN);
  constexpr uint32_t kSbo = 128 * (DP / 8);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     mma::smem_u32(tmem_base_s)),
                 "r"(kMmaN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mma::mbar_init(mbar, 1);
    mma::fence_async_smem();
  }
  mma::fence_before();
  __syncthreads();
  mma::fence_after();
  const uint32_t tmem = *tmem_base_s;
  uint32_t phase = 0;

  const int qny = a.qxs ? (int)(a.nq / a.qnx) : 0;
  const int tnx = a.qxs ? (a.qnx + 15) / 16 : 0;
  const int64_t n_tiles = a.qxs ? (int64_t)tnx * ((qny + 7) / 8) : (a.nq + kMmaM - 1) / kMmaM;

  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    int64_t q;
    bool valid;
    if (a.qxs) {
      const int tx = (int)(t % tnx), ty = (int)(t / tnx);
      const int ix = tx * 16 + (tid & 15), iy = ty * 8 + (tid >> 4);
      valid = ix < a.qnx && iy < qny;
      q = valid ? (int64_t)iy * a.qnx + ix : 0;
    } else {
      q = t * kMmaM + tid;
      valid = q < a.nq;
    }
    const double* qrow = a.q + (valid ? q : 0) * d;
    float q32[DP];
    float qn2f = 0.f;
    double qn2 = 0.0;
#pragma unroll
    for (int j = 0; j < DP; ++j) {
      const double v = (valid && j < d) ? qrow[j] : 0.0;
      q32[j] = (float)v;
      qn2 += v * v;
      qn2f = fmaf(q32[j], q32[j], qn2f);
    }
    const float qn = __double2float_ru(sqrt(qn2) * (1.0 + 1e-12));
    // A operand rows: bf16 split of this thread's query
#pragma unroll
    for (int j = 0; j < DP; j += 2) {
      const __nv_bfloat16 h0 = __float2bfloat16_rn(q32[j]), h1 = __float2bfloat16_rn(q32[j + 1]);
      const __nv_bfloat16 l0 = __float2bfloat16_rn(q32[j] - __bfloat162float(h0));
      const __nv_bfloat16 l1 = __float2bfloat16_rn(q32[j + 1] - __bfloat162float(h1));
      const uint32_t off = mma::op_off(tid, j, DP);
      *reinterpret_cast<__nv_bfloat162*>(a_hi + off) = __halves2bfloat162(h0, h1);
      *reinterpret_cast<__nv_bfloat162*>(a_lo + off) = __halves2bfloat162(l0, l1);
    }

    double best = valid ? kInf : -1.0;
    int32_t best_id = 0x7fffffff;
    int64_t scanned = 0, exact_evals = 0;
    int32_t visited = 0;
    if (a.seed_idx && valid) {
      const int qix = a.qxs ? (int)(q % a.qnx) : 0, qiy = a.qxs ? (int)(q / a.qnx) : 0;
#pragma unroll 1
      for (int k = 0; k < 5; ++k) {
        int32_t cand = -1;
        if (k == 0) {
          cand = a.seed_idx[q];
        } else if (a.qxs) {
          const int nix = qix + (k == 1 ? -1 : k == 2 ? 1 : 0);
          const int niy = qiy + (k == 3 ? -1 : k == 4 ? 1 : 0);
          if (nix >= 0 && nix < a.qnx && niy >= 0 && niy < qny) {
            const int32_t e = a.seed_idx[(int64_t)niy * a.qnx + nix];
            const int ex = e % a.nxe + (a.qxs[qix] - a.qxs[nix]);
            const int ey = e / a.nxe + (a.qys[qiy] - a.qys[niy]);
            if (ex >= 0 && ex < a.nxe && ey >= 0 && ey < a.nye) cand = ey * a.nxe + ex;
          }
        }
        if (cand < 0) continue;
        const double d2 = dist2_seq_mma(qrow, a.proj + (int64_t)cand * d, d);
        ++scanned;
        ++exact_evals;
        if (d2 < best || (d2 == best && cand < best_id)) {
          best = d2;
          best_id = cand;
        }
      }
    }
    float best_up = __double2float_ru(best);

    if (tid == 0) st_meta[0] = a.tree.meta[0];
    st_lb[tid] = 0.f;
    int top = 1;
    __syncthreads();
    while (top > 0) {
      // ---- pop: drop entries no query still wants; batch consecutive leaves -----
      int bstart[8], bcnt[8];
      int nb = 0, tot = 0;
      int2 node = make_int2(0, 0);
      while (top > 0) {
        const int2 md = st_meta[top - 1];
        const bool want = (double)st_lb[(top - 1) * kMmaM + tid] <= best;
        if (!__syncthreads_or(want)) {
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
        if (nb > 0 && (tot + md.y > kMmaN || nb == 8)) break;
        --top;
        bstart[nb] = md.x;
        bcnt[nb] = md.y;
        ++nb;
        tot += md.y;
        if (tot >= kMmaN) break;
      }
      if (nb > 0) {
        visited += nb;
        scanned += tot;
        for (int c0 = 0; c0 < tot; c0 += kMmaN) {
          const int cn = min(kMmaN, tot - c0);
          // ---- stage <= 128 points as bf16 hi/lo B rows (row = thread) --------
          {
            float p[DP];
            float pn2f = 0.f;
            int32_t pid = -1;
            float pnrm = 0.f;
            if (tid < cn) {
              int i = c0 + tid, b = 0;
#pragma unroll
              for (int k = 0; k < 7; ++k)
                if (b < nb - 1 && i >= bcnt[b]) i -= bcnt[b++];
              const int pos = bstart[b] + i;
              const float4* col = reinterpret_cast<const float4*>(a.proj32_q4) + pos;
#pragma unroll
              for (int k = 0; k < DP / 4; ++k) {
                const float4 v = (4 * k < d) ? __ldg(col + (int64_t)k * N)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                p[4 * k] = v.x;
                p[4 * k + 1] = v.y;
                p[4 * k + 2] = v.z;
                p[4 * k + 3] = v.w;
              }
              pid = a.perm[pos];
              pnrm = a.pnorm32[pos];
            } else {
#pragma unroll
              for (int k = 0; k < DP; ++k) p[k] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < DP; ++j) pn2f = fmaf(p[j], p[j], pn2f);
#pragma unroll
            for (int j = 0; j < DP; j += 2) {
              const __nv_bfloat16 h0 = __float2bfloat16_rn(p[j]), h1 = __float2bfloat16_rn(p[j + 1]);
              const __nv_bfloat16 l0 = __float2bfloat16_rn(p[j] - __bfloat162float(h0));
              const __nv_bfloat16 l1 = __float2bfloat16_rn(p[j + 1] - __bfloat162float(h1));
              const uint32_t off = mma::op_off(tid, j, DP);
              *reinterpret_cast<__nv_bfloat162*>(b_hi + off) = __halves2bfloat162(h0, h1);
              *reinterpret_cast<__nv_bfloat162*>(b_lo + off) = __halves2bfloat162(l0, l1);
            }
            pn2_s[tid] = pn2f;
            pnorm_s[tid] = pnrm;
            pid_s[tid] = pid;
          }
          mma::fence_async_smem();
          mma::fence_before();
          __syncthreads();
          mma::fence_after();
          if (tid == 0) {
            const uint32_t ah = mma::smem_u32(a_hi), al = mma::smem_u32(a_lo);
            const uint32_t bh = mma::smem_u32(b_hi), bl = mma::smem_u32(b_lo);
#pragma unroll
            for (int s = 0; s < DP / 16; ++s) {
              const uint32_t ko = s * 256;  // two 8-element K chunks per UMMA step
              const uint64_t dah = mma::make_desc(ah + ko, 128, kSbo);
              const uint64_t dal = mma::make_desc(al + ko, 128, kSbo);
              const uint64_t dbh = mma::make_desc(bh + ko, 128, kSbo);
              const uint64_t dbl = mma::make_desc(bl + ko, 128, kSbo);
              mma::mma_bf16(tmem, dah, dbh, kIdesc, s > 0 ? 1u : 0u);
              mma::mma_bf16(tmem, dah, dbl, kIdesc, 1u);
              mma::mma_bf16(tmem, dal, dbh, kIdesc, 1u);
            }
            mma::commit(mbar);
          }
          mma::mbar_wait(mbar, phase);
          phase ^= 1u;
          mma::fence_after();
          // ---- epilogue: this thread's query row of D ----------------------------
          float thr = best_up * (1.f + 1e-4f) +
                      1.01f * (1.6e-4f * qn * a.pnorm_max +
                               1e-5f * (qn * qn + a.pnorm_max * a.pnorm_max)) + 1e-30f;
          for (int j0 = 0; j0 < cn; j0 += 32) {
            float dot[32];
            mma::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j0, dot);
#pragma unroll 4
            for (int jj = 0; jj < 32; ++jj) {
              const int j = j0 + jj;
              if (j >= cn) break;
              const float s = fmaf(-2.f, dot[jj], qn2f + pn2_s[j]);
              if (s <= thr) {
                const float pnr = pnorm_s[j];
                const float eps = 1.6e-4f * qn * pnr + 1e-5f * (qn * qn + pnr * pnr) + 1e-30f;
                if (s - eps <= best_up) {
                  const int32_t id = pid_s[j];
                  const double d2 = dist2_seq_mma(qrow, a.proj + (int64_t)id * d, d);
                  ++exact_evals;
                  if (d2 < best || (d2 == best && id < best_id)) {
                    best = d2;
                    best_id = id;
                    best_up = __double2float_ru(best);
                    thr = best_up * (1.f + 1e-4f) +
                          1.01f * (1.6e-4f * qn * a.pnorm_max +
                                   1e-5f * (qn * qn + a.pnorm_max * a.pnorm_max)) + 1e-30f;
                  }
                }
              }
            }
          }
          mma::fence_before();
          __syncthreads();  // D and the B tiles are free again
        }
        continue;
      }
      if (node.y >= 0) break;
      // ---- expand an internal node: children bounds (fp32 SIMT, conservative) -----
      ++visited;
      const int nc = -node.y;
      const int fc = node.x;
      for (int f = tid; f < nc * DP; f += kMmaM) {
        const int c = f / DP, j = f - c * DP;
        cst[c * RS + j] = j < d ? __ldg(a.tree.centroid32 + (int64_t)(fc + c) * d + j) : 0.f;
      }
      if (tid < nc) {
        caux[tid] = a.tree.radius32[fc + tid];
        caux[kMmaMaxB + tid] = a.tree.cnorm32[fc + tid];
        cmeta[tid] = a.tree.meta[fc + tid];
      }
      for (int f = tid; f < nc * KB; f += kMmaM) {
        const int c = f % nc, j = f / nc;
        cbox[(c * kBoxDims + j) * 2] = __ldg(a.tree.boxlo + (int64_t)j * nn + fc + c);
        cbox[(c * kBoxDims + j) * 2 + 1] = __ldg(a.tree.boxhi + (int64_t)j * nn + fc + c);
      }
      __syncthreads();
#pragma unroll 1
      for (int c = 0; c < nc; ++c) {
        const float* cr = cst + c * RS;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int k = 0; k < DP / 4; ++k) {
          const float4 pv = *reinterpret_cast<const float4*>(cr + 4 * k);
          float u = q32[4 * k] - pv.x;
          s0 = fmaf(u, u, s0);
          u = q32[4 * k + 1] - pv.y;
          s1 = fmaf(u, u, s1);
          u = q32[4 * k + 2] - pv.z;
          s2 = fmaf(u, u, s2);
          u = q32[4 * k + 3] - pv.w;
          s3 = fmaf(u, u, s3);
        }
        const float s = (s0 + s1) + (s2 + s3);
        float bx = 0.f;
#pragma unroll
        for (int j = 0; j < kBoxDims; ++j) {
          if (j < KB) {
            const float lo = cbox[(c * kBoxDims + j) * 2], hi = cbox[(c * kBoxDims + j) * 2 + 1];
            const float qj = q32[j];
            float gap = fmaxf(lo - qj, qj - hi) - 2.4e-7f * (fabsf(qj) + fabsf(lo) + fabsf(hi));
            gap = fmaxf(gap, 0.f);
            bx = fmaf(gap, gap, bx);
          }
        }
        const float dc = sqrtf(s);
        const float rad = caux[c];
        const float slack = 2e-5f * (1.f + dc + rad + qn + caux[kMmaMaxB + c]);
        const float lb = dc - rad - slack;
        float lb2 = lb > 0.f ? lb * lb * (1.f - 1e-6f) : 0.f;
        lb2 = fmaxf(lb2, bx * (1.f - 1e-5f));
        tlb[c * kMmaM + tid] = lb2;
        const bool want = (double)lb2 <= best;
        const unsigned key =
            __reduce_min_sync(0xffffffffu, want ? __float_as_uint(lb2) : 0xffffffffu);
        if (lane == 0) wkey[warp * kMmaMaxB + c] = key;
      }
      __syncthreads();
      if (tid < nc) {
        unsigned k = wkey[tid];
#pragma unroll
        for (int w = 1; w < 4; ++w) k = min(k, wkey[w * kMmaMaxB + tid]);
        tkey[tid] = k;
      }
      __syncthreads();
      unsigned keepmask = 0;
      for (int c = 0; c < nc; ++c)
        if (tkey[c] != 0xffffffffu) keepmask |= 1u << c;
      const int nkeep = __popc(keepmask);
      if (top + nkeep > kMmaStack) {
        if (tid == 0) atomicOr(a.flags, FLAG_STACK_OVERFLOW);
        break;
      }
      for (int c = 0; c < nc; ++c) {
        if (!((keepmask >> c) & 1u)) continue;
        const unsigned kc = tkey[c];
        int rank = 0;
        for (int o = 0; o < nc; ++o) {
          const unsigned ko = tkey[o];
          if (ko != 0xffffffffu && (ko < kc || (ko == kc && o < c))) ++rank;
        }
        const int slot = top + nkeep - 1 - rank;  // nearest child popped first
        st_lb[slot * kMmaM + tid] = tlb[c * kMmaM + tid];
        if (tid == 0) st_meta[slot] = cmeta[c];
      }
      top += nkeep;
      __syncthreads();
    }
    if (valid) {
      a.out_idx[q] = best_id;
      a.out_d2[q] = best;
      if (a.out_scanned) a.out_scanned[q] = scanned;
      if (a.out_exact) a.out_exact[q] = exact_evals;
      if (a.out_visited) a.out_visited[q] = visited;
    }
    __syncthreads();
  }
  mma::fence_before();
  __syncthreads();
  if (warp == 0) {
    mma::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kMmaN));
  }
}

bool launch_search_mma(psg_ctx* ctx, const SearchArgs& a) {
  ProfScope _prof(ctx, K_SEARCH);
  if (a.nq <= 0) return true;
  if (a.tree.max_children > kMmaMaxB || 1 + a.tree.max_depth * (a.tree.max_children - 1) > kMmaStack)
    return false;
  const int64_t tiles = a.qxs ? (int64_t)((a.qnx + 15) / 16) * (((a.nq / a.qnx) + 7) / 8)
                              : (a.nq + kMmaM - 1) / kMmaM;
  if (a.d <= 32) {
    constexpr MmaSmem L = mma_smem_layout<32>();
    auto k = search_mma_kernel<32>;
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    int64_t blocks = tiles < (int64_t)ctx->num_sms * 3 ? tiles : (int64_t)ctx->num_sms * 3;
    k<<<(int)blocks, kMmaM, L.total, ctx->stream>>>(a);
  } else if (a.d <= 64) {
    constexpr MmaSmem L = mma_smem_layout<64>();
    auto k = search_mma_kernel<64>;
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    int64_t blocks = tiles < (int64_t)ctx->num_sms * 2 ? tiles : (int64_t)ctx->num_sms * 2;
    k<<<(int)blocks, kMmaM, L.total, ctx->stream>>>(a);
  } else {
    return false;
  }
  PSG_LAUNCHED(ctx);
  return true;
}

}  // namespace psg
