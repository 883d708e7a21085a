// Exact tile search with the leaf filter on the tensor cores (warp-level
// mma.sync, bf16 m16n8k16), sm_100a, d <= 32.
//
// Same traversal as search_tile_kernel (one warp = 32 queries of an 8 x 4
// anchor tile sharing one depth-first walk of the k-means tree, lanes =
// queries, SIMT fp32 child bounds), but each batch of <= 32 leaf points is
// filtered as a 32 x 32 x 32 GEMM:
//     D = Qhi.Phi^T + Qhi.Plo^T + Qlo.Phi^T     (x = hi + lo, bf16 split)
// with fp32 accumulation, s = |q|^2 + |p|^2 - 2 D, and the rigorous bound
// |s - dist^2| <= 1.6e-4 |q||p| + 1e-5 (|q|^2 + |p|^2) (split residual,
// accumulation, epilogue) — the bound of the tcgen05 variant.
// Survivors (s - eps <= the query's best) are re-evaluated by the query's
// lane with the reference's exact fp64 chain (km_tree.cpp:15-22), so the
// result is the lexicographic (dist^2, id) minimum, bit-identical to the
// reference.  Measured on B200: mma.sync bf16 ~555 TFLOP/s vs 71 TFLOP/s FFMA
// (scripts/micro/mma_sync_bench.cu), and 48 HMMA replace ~1000 FFMA2/FADD2
// per 32-point batch — but the leaf filter is only ~20% of the SIMT kernel's
// instructions (child bounds and traversal dominate) and the SIMT filter
// exits early after 8/16 leading dims, so this variant is ~15% slower on the
// bench stage (4.26 vs 3.71 ms).  Kept as PERSYN_SEARCH=hmma, parity-tested.
//
// Fragment layouts (PTX ISA, mma.m16n8k16): g = lane / 4, t = lane % 4;
// A (queries x dims, row-major) a0 = (g, 2t..2t+1), a1 = (g+8, ..), a2 = (g,
// 2t+8..), a3 = (g+8, 2t+8..); B (dims x points) b0 = (2t..2t+1, g), b1 =
// (2t+8.., g); C c0,c1 = (g, 2t..2t+1), c2,c3 = (g+8, ..).  Staged rows hold
// 40 bf16 (32 dims + pad): 32-bit fragment loads are bank-conflict free.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>

#include "numerics.cuh"
#include "psg_internal.h"

namespace psg {

namespace {

constexpr int kHStack = 48;
constexpr int kHMaxB = 16;
constexpr int kHW = 3;     // warps per CTA
constexpr int kRowB = 40;  // bf16 per staged row
constexpr int kRS = 36;    // floats per fp32 child staging row

__device__ __forceinline__ bool lexl(double a, int32_t ia, double b, int32_t ib) {
  return a < b || (a == b && ia < ib);
}

__device__ __noinline__ double d2seq(const double* __restrict__ q, const double* __restrict__ p,
                                     int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = dsub(q[j], p[j]);
    acc = dadd(acc, dmul(t, t));
  }
  return acc;
}

__device__ __forceinline__ void hmma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                     uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t bf2(float x0, float x1, uint32_t& lo) {
  const __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1 = __float2bfloat16_rn(x1);
  const __nv_bfloat16 l0 = __float2bfloat16_rn(x0 - __bfloat162float(h0));
  const __nv_bfloat16 l1 = __float2bfloat16_rn(x1 - __bfloat162float(h1));
  const __nv_bfloat162 l = __halves2bfloat162(l0, l1), h = __halves2bfloat162(h0, h1);
  lo = *reinterpret_cast<const uint32_t*>(&l);
  return *reinterpret_cast<const uint32_t*>(&h);
}

struct __align__(16) HWarp {
  // leaf batch: B rows hi [32][40] + lo [32][40] bf16 | child staging fp32
  // [16][36] | query rows at tile start
  uint32_t buf[2 * 32 * kRowB / 2];
  float st_lb[kHStack][32];
  float tlb[kHMaxB][32];
  float box[kHMaxB][2 * kBoxDims];
  int2 st_meta[kHStack];
  int2 cmeta[kHMaxB];
  float aux0[32], aux1[32];  // leaves: |p| rounded up, |p|^2 (fp32); children: radius, |c|
  int32_t pid[32];
  float thrL[32], thrP[32];  // per query: loose / precise filter threshold
  float qn2s[32], qns[32];
  unsigned smask[32];
  unsigned tkey[kHMaxB];
};

__global__ void __launch_bounds__(32 * kHW) search_tile_hmma_kernel(SearchArgs a) {
  __shared__ HWarp sm_all[kHW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  HWarp& S = sm_all[warp];
  const int g = lane >> 2, tq = lane & 3;
  const int d = a.d;
  const int N = (int)a.N;
  const int nn = a.tree.n_nodes;
  const int KB = d < kBoxDims ? d : kBoxDims;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const float pnm = a.pnorm_max;
  const int qny = a.qxs ? (int)(a.nq / a.qnx) : 0;
  const int tnx = a.qxs ? (a.qnx + 7) / 8 : 0;
  const int64_t n_tiles = a.qxs ? (int64_t)tnx * ((qny + 3) / 4) : (a.nq + 31) / 32;
  __nv_bfloat16* Bh = reinterpret_cast<__nv_bfloat16*>(S.buf);
  __nv_bfloat16* Bl = Bh + 32 * kRowB;
  float* stage = reinterpret_cast<float*>(S.buf);

  for (int64_t t = (int64_t)blockIdx.x * kHW + warp; t < n_tiles;
       t += (int64_t)gridDim.x * kHW) {
    int64_t q;
    bool valid;
    if (a.qxs) {
      const int tx = (int)(t % tnx), ty = (int)(t / tnx);
      const int ix = tx * 8 + (lane & 7), iy = ty * 4 + (lane >> 3);
      valid = ix < a.qnx && iy < qny;
      q = valid ? (int64_t)iy * a.qnx + ix : 0;
    } else {
      q = t * 32 + lane;
      valid = q < a.nq;
    }
    const double* qrow = a.q + (valid ? q : 0) * d;
    float2 q2[16];
    double qn2 = 0.0;
    float qn2f = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const double v0 = (valid && 2 * j < d) ? qrow[2 * j] : 0.0;
      const double v1 = (valid && 2 * j + 1 < d) ? qrow[2 * j + 1] : 0.0;
      q2[j] = make_float2((float)v0, (float)v1);
      qn2 += v0 * v0 + v1 * v1;
      qn2f = fmaf(q2[j].x, q2[j].x, qn2f);
      qn2f = fmaf(q2[j].y, q2[j].y, qn2f);
    }
    const float qn = __double2float_ru(sqrt(qn2) * (1.0 + 1e-12));
    const float qdelta = 1.2e-7f * qn;  // >= |float(q_j) - q_j| for every j
    // query rows (bf16 split) -> A fragments in registers
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      uint32_t lo;
      const uint32_t hi = bf2(q2[j].x, q2[j].y, lo);
      reinterpret_cast<uint32_t*>(Bh)[lane * (kRowB / 2) + j] = hi;
      reinterpret_cast<uint32_t*>(Bl)[lane * (kRowB / 2) + j] = lo;
    }
    S.qn2s[lane] = qn2f;
    S.qns[lane] = qn;
    __syncwarp();
    uint32_t Ah[2][2][4], Al[2][2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int r0 = mt * 16 + g, c0 = ks * 8 + tq;  // 32-bit column index
        const uint32_t* H = reinterpret_cast<const uint32_t*>(Bh);
        const uint32_t* Lw = reinterpret_cast<const uint32_t*>(Bl);
        Ah[mt][ks][0] = H[r0 * (kRowB / 2) + c0];
        Ah[mt][ks][1] = H[(r0 + 8) * (kRowB / 2) + c0];
        Ah[mt][ks][2] = H[r0 * (kRowB / 2) + c0 + 4];
        Ah[mt][ks][3] = H[(r0 + 8) * (kRowB / 2) + c0 + 4];
        Al[mt][ks][0] = Lw[r0 * (kRowB / 2) + c0];
        Al[mt][ks][1] = Lw[(r0 + 8) * (kRowB / 2) + c0];
        Al[mt][ks][2] = Lw[r0 * (kRowB / 2) + c0 + 4];
        Al[mt][ks][3] = Lw[(r0 + 8) * (kRowB / 2) + c0 + 4];
      }
    // this lane's four epilogue rows: g, g + 8, 16 + g, 24 + g
    float qn2r[4], qnr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (i >> 1) * 16 + g + (i & 1) * 8;
      qn2r[i] = S.qn2s[r];
      qnr[i] = S.qns[r];
    }
    double best = valid ? kInf : -1.0;
    int32_t best_id = 0x7fffffff;
    int64_t scanned = 0, exact_evals = 0;
    int32_t visited = 0;

    // ---- coherence seeds (exact fp64), per lane ----------------------------------
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
        const double d2 = d2seq(qrow, a.proj + (int64_t)cand * d, d);
        ++scanned;
        ++exact_evals;
        if (lexl(d2, cand, best, best_id)) {
          best = d2;
          best_id = cand;
        }
      }
    }
    // filter thresholds: a float compare can only keep more points
    float best_up = __double2float_ru(best);
    auto publish = [&]() {
      S.thrP[lane] = best_up;
      S.thrL[lane] = best_up * (1.f + 1e-4f) +
                     1.01f * (1.6e-4f * qn * pnm + 1e-5f * (qn * qn + pnm * pnm)) + 1e-30f;
    };
    publish();
    S.smask[lane] = 0u;

    if (lane == 0) S.st_meta[0] = a.tree.meta[0];
    S.st_lb[0][lane] = 0.f;
    int top = 1;
    __syncwarp();
    while (top > 0) {
      // ---- pop: drop entries no lane still wants; batch consecutive leaves ------
      int bstart[4], bcnt[4];
      int nb = 0, tot = 0;
      int2 node = make_int2(0, 0);
      while (top > 0) {
        const int2 md = S.st_meta[top - 1];
        const bool want = (double)S.st_lb[top - 1][lane] <= best;
        if (!__any_sync(0xffffffffu, want)) {
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
          // ---- stage <= 32 points as bf16 hi/lo rows (lane i: point c0 + i) ----------
          __syncwarp();
          {
            float p[32];
            int32_t pidv = -1;
            float pnr = 0.f;
            if (lane < cn) {
              int i = c0 + lane, b = 0;
#pragma unroll
              for (int k = 0; k < 3; ++k)
                if (b < nb - 1 && i >= bcnt[b]) i -= bcnt[b++];
              const int pos = bstart[b] + i;
              const float4* col = reinterpret_cast<const float4*>(a.proj32_q4) + pos;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float4 v = (4 * k < d) ? __ldg(col + (int64_t)k * N)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                p[4 * k] = v.x;
                p[4 * k + 1] = v.y;
                p[4 * k + 2] = v.z;
                p[4 * k + 3] = v.w;
              }
              pidv = a.perm[pos];
              pnr = a.pnorm32[pos];
            } else {
#pragma unroll
              for (int k = 0; k < 32; ++k) p[k] = 0.f;
            }
            float pn2f = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) pn2f = fmaf(p[j], p[j], pn2f);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              uint32_t lo;
              const uint32_t hi = bf2(p[2 * j], p[2 * j + 1], lo);
              reinterpret_cast<uint32_t*>(Bh)[lane * (kRowB / 2) + j] = hi;
              reinterpret_cast<uint32_t*>(Bl)[lane * (kRowB / 2) + j] = lo;
            }
            S.aux0[lane] = pnr;
            S.aux1[lane] = pn2f;
            S.pid[lane] = pidv;
          }
          __syncwarp();
          float tl[4], tp[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = (i >> 1) * 16 + g + (i & 1) * 8;
            tl[i] = S.thrL[r];
            tp[i] = S.thrP[r];
          }
          bool any = false;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            if (nt * 8 < cn) {
              float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {
                const int w0 = (nt * 8 + g) * (kRowB / 2) + ks * 8 + tq;
                const uint32_t bh0 = reinterpret_cast<const uint32_t*>(Bh)[w0];
                const uint32_t bh1 = reinterpret_cast<const uint32_t*>(Bh)[w0 + 4];
                const uint32_t bl0 = reinterpret_cast<const uint32_t*>(Bl)[w0];
                const uint32_t bl1 = reinterpret_cast<const uint32_t*>(Bl)[w0 + 4];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                  hmma(acc[mt], Ah[mt][ks], bh0, bh1);
                  hmma(acc[mt], Ah[mt][ks], bl0, bl1);
                  hmma(acc[mt], Al[mt][ks], bh0, bh1);
                }
              }
#pragma unroll
              for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int ri = mt * 2 + (e >> 1);
                  const int col = nt * 8 + 2 * tq + (e & 1);
                  const float s = fmaf(-2.f, acc[mt][e], qn2r[ri] + S.aux1[col]);
                  if (col < cn && s <= tl[ri]) {
                    const float pr = S.aux0[col];
                    const float eps = 1.6e-4f * qnr[ri] * pr +
                                      1e-5f * (qnr[ri] * qnr[ri] + pr * pr) + 1e-30f;
                    if (s - eps <= tp[ri]) {
                      const int row = mt * 16 + g + (e >> 1) * 8;
                      atomicOr(&S.smask[row], 1u << col);
                      any = true;
                    }
                  }
                }
            }
          }
          if (__any_sync(0xffffffffu, any)) {
            __syncwarp();
            unsigned m = S.smask[lane];
            S.smask[lane] = 0u;
            while (m) {
              const int c = __ffs(m) - 1;
              m &= m - 1;
              const int32_t id = S.pid[c];
              const double d2 = d2seq(qrow, a.proj + (int64_t)id * d, d);
              ++exact_evals;
              if (lexl(d2, id, best, best_id)) {
                best = d2;
                best_id = id;
                best_up = __double2float_ru(best);
              }
            }
            publish();
            __syncwarp();
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
      for (int f = lane; f < nc * 32; f += 32) {
        const int c = f >> 5, j = f & 31;
        stage[c * kRS + j] = j < d ? -__ldg(a.tree.centroid32 + (int64_t)(fc + c) * d + j) : 0.f;
      }
      if (lane < nc) {
        S.aux0[lane] = a.tree.radius32[fc + lane];
        S.aux1[lane] = a.tree.cnorm32[fc + lane];
        S.cmeta[lane] = a.tree.meta[fc + lane];
      }
      for (int f = lane; f < nc * KB; f += 32) {
        const int c = f % nc, j = f / nc;
        S.box[c][2 * j] = __ldg(a.tree.boxlo + (int64_t)j * nn + fc + c);
        S.box[c][2 * j + 1] = __ldg(a.tree.boxhi + (int64_t)j * nn + fc + c);
      }
      __syncwarp();
#pragma unroll 1
      for (int c = 0; c < nc; ++c) {
        // box bound first (kernels_search.cu, search_tile_kernel: same bounds)
        float bx = 0.f;
#pragma unroll
        for (int j = 0; j < kBoxDims; ++j) {
          if (j < KB) {
            const float lo = S.box[c][2 * j], hi = S.box[c][2 * j + 1];
            const float qj = (j & 1) ? q2[j >> 1].y : q2[j >> 1].x;
            const float gap = fmaxf(fmaxf(lo - qj, qj - hi) - qdelta, 0.f);
            bx = fmaf(gap, gap, bx);
          }
        }
        bx *= 1.f - 1e-5f;
        float lb2 = bx;
        if (__any_sync(0xffffffffu, (double)bx <= best)) {
          const float4* cr = reinterpret_cast<const float4*>(stage + c * kRS);
          float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 pv = cr[k];
            const float2 u0 = __fadd2_rn(q2[2 * k], make_float2(pv.x, pv.y));
            const float2 u1 = __fadd2_rn(q2[2 * k + 1], make_float2(pv.z, pv.w));
            sa = __ffma2_rn(u0, u0, sa);
            sb = __ffma2_rn(u1, u1, sb);
          }
          const float s = (sa.x + sa.y) + (sb.x + sb.y);
          const float dc = sqrtf(s);
          const float rad = S.aux0[c];
          const float slack = 2e-5f * (1.f + dc + rad + qn + S.aux1[c]);
          const float lb = dc - rad - slack;
          lb2 = fmaxf(lb > 0.f ? lb * lb * (1.f - 1e-6f) : 0.f, bx);
        }
        S.tlb[c][lane] = lb2;
        const bool want = (double)lb2 <= best;
        const unsigned key =
            __reduce_min_sync(0xffffffffu, want ? __float_as_uint(lb2) : 0xffffffffu);
        if (lane == 0) S.tkey[c] = key;
      }
      __syncwarp();
      const unsigned mykey = lane < nc ? S.tkey[lane] : 0xffffffffu;
      const bool kept = mykey != 0xffffffffu;
      const unsigned keepmask = __ballot_sync(0xffffffffu, kept);
      const int nkeep = __popc(keepmask);
      if (top + nkeep > kHStack) {
        if (lane == 0) atomicOr(a.flags, FLAG_STACK_OVERFLOW);
        break;
      }
      int myslot = -1;
      if (kept) {
        int rank = 0;
        for (int o = 0; o < nc; ++o) {
          const unsigned ko = S.tkey[o];
          if (ko != 0xffffffffu && (ko < mykey || (ko == mykey && o < lane))) ++rank;
        }
        myslot = top + nkeep - 1 - rank;
        S.st_meta[myslot] = S.cmeta[lane];
      }
#pragma unroll 1
      for (int c = 0; c < nc; ++c) {
        const int slot = __shfl_sync(0xffffffffu, myslot, c);
        if (slot >= 0) S.st_lb[slot][lane] = S.tlb[c][lane];
      }
      top += nkeep;
      __syncwarp();
    }
    if (valid) {
      a.out_idx[q] = best_id;
      a.out_d2[q] = best;
      if (a.out_scanned) a.out_scanned[q] = scanned;
      if (a.out_exact) a.out_exact[q] = exact_evals;
      if (a.out_visited) a.out_visited[q] = visited;
    }
    __syncwarp();
  }
}

}  // namespace

bool launch_search_hmma(psg_ctx* ctx, const SearchArgs& a) {
  if (a.d > 32 || a.tree.max_children > kHMaxB ||
      1 + a.tree.max_depth * (a.tree.max_children - 1) > kHStack)
    return false;
  const int64_t tiles = (a.nq + 31) / 32;
  int64_t blocks = (tiles + kHW - 1) / kHW;
  const int64_t cap = (int64_t)ctx->num_sms * 24;
  if (blocks > cap) blocks = cap;
  search_tile_hmma_kernel<<<(int)blocks, 32 * kHW, 0, ctx->stream>>>(a);
  PSG_LAUNCHED(ctx);
  return true;
}

}  // namespace psg
