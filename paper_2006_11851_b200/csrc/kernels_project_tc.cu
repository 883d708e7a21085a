// PCA projection of the E-step's query windows on the 5th-gen tensor cores.
//
// The reference projects every window in fp64, j-sequential, mul then add
// (pca.cpp:27-41, called per query from optimizer.cpp:228-230).  That chain is
// what the nearest-neighbour comparison ultimately uses, but almost every
// query's winner is separated from its runner-up by far more than the chain's
// rounding.  So the E-step first computes an approximation q^ with a RIGOROUS
// error bound on the tensor cores, and the search keeps every candidate within
// that bound of the best (kernels_search.cu, approximate-query mode); only the
// queries whose winner is not separated (near-ties) are re-projected with the
// exact chain and searched again (launch_project_list + an exact warp search),
// so NN indices stay bit-identical to the reference's.
//
// The approximation is computed EXACTLY in integers:
//   v^  = V 2^-29,  V = rint(v 2^29) in [0, 2^29]   (|v - v^| <= 2^-30)
//   B^  = Bq 2^-30, Bq = rint(B 2^30)               (|B - B^| <= 2^-31)
//   q^_k = sum_{s,t} 256^(s+t) (sum_j a_s,j b_t,kj) 2^-59 - (B mu)_k
// with V in four unsigned base-256 digits a_s (u8) and Bq in four balanced
// signed digits b_t (s8).  Each digit product runs as tcgen05.mma kind::i8
// with int32 accumulation (exact); the four B digit slices are stacked along
// UMMA N, so one instruction per A slice computes all its products.  The 3 of
// 16 products with s + t <= 1 contribute < 2^-59 32640 513 D and are dropped
// (bounded below).  Per k:
//   |q^_k - q_k| <= 2^-30 |B_k|_1 + 2^-31 D + 2^-59 32640 513 D
//                   + (2D + 2) 2^-53 |B_k|_1 + 2^-52 (|B mu_k| + |B_k|_1)
//                   + 20 D 2^-53 (the final fp64 conversion, generous) + 1e-12
// (|v - mu| <= 1 bounds |q_k| by |B_k|_1; the reference's own chain is within
// (2D + 2) 2^-53 |B_k|_1 of the exact value), and delta = the 2-norm over k:
// about 1e-6 at w = 8, d = 32, so only true near-ties reach the fallback.
//
// Operands: windows of the digit mirror q8 [4][H][W][8] (8-byte pixels: a
// window row is w x 8 contiguous bytes and, at spacing 2, consecutive anchors'
// 16-byte K groups are consecutive 16-byte blocks: one 1-D bulk copy per slice
// and group), staged in the UMMA K-major no-swizzle layout (K group g of the
// 128 anchors = one contiguous 2 KB block).  Persistent, warp-specialised:
// warp 0 stages, warp 1 issues the UMMAs, warps 2-9 drain TMEM.  Basis rows
// go in blocks of 32 (TMEM holds 416 accumulator columns per block).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "numerics.cuh"
#include "psg_internal.h"
#include "umma.cuh"

namespace psg {
namespace {

constexpr int kTM = 128;                        // anchors per tile (UMMA M)
constexpr int kGC = 4;                          // 16-byte K groups per stage (2 UMMA K-steps)
constexpr int kSA = 4, kSB = 4;                 // digit slices of V and Bq
constexpr int kNB = 32;                         // basis rows per block
constexpr int kNP = kSB * kNB;                  // stacked B rows: t * 32 + n
constexpr uint32_t kAGroup = kTM * 16;          // 2 KB per K group (one slice)
constexpr uint32_t kASlice = kGC * kAGroup;     // 8 KB per slice per stage
constexpr uint32_t kBStage = kGC * kNP * 16;    // 8 KB per stage
constexpr uint32_t kStageBytes = kSA * kASlice + kBStage;  // 40 KB
constexpr int kStages = 5;
constexpr int kTcThreads = 320;  // producer, MMA issuer, 8 epilogue warps
constexpr uint32_t kBarOff = kStages * kStageBytes;
constexpr uint32_t kSmemBytes = kBarOff + (2 * kStages + 3) * 8 + 16;
// strip mode (spacing 2, w % 4 == 0, one basis block, w <= 8): the basis digits
// stay resident (<= 64 KB) and a stage is ONE window row of the tile: per digit
// slice the contiguous strip of 2 (nt - 1) + w pixels.  K group g' of that row
// is the strip at byte offset 16 g' (row m at 16 m): the UMMA descriptor points
// into the strip with a 16-byte leading-dimension offset, so each row is
// copied once instead of once per K group (w / 2 times).
constexpr uint32_t kBresBytes = 64 * 1024;
constexpr uint32_t kStripSlot = 2304;                // >= 16 * 127 + 8 * 8
constexpr int kStripStages = 8;
constexpr uint32_t kStripStage = kSA * kStripSlot;
constexpr uint32_t kStripBarOff = kBresBytes + kStripStages * kStripStage;
constexpr uint32_t kStripSmemBytes = kStripBarOff + (2 * kStripStages + 3) * 8 + 16;
// kept products per A slice s: t in [tmin(s), 4); TMEM columns [col0(s), +32 (4 - tmin))
__host__ __device__ constexpr int tmin_of(int s) { return s == 0 ? 2 : (s == 1 ? 1 : 0); }
__host__ __device__ constexpr int col0_of(int s) { return s == 0 ? 0 : (s == 1 ? 64 : 160 + (s - 2) * 128); }
constexpr uint32_t kTmemCols = 512;  // 416 used

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// kind::i8 instruction descriptor: D s32, A u8, B s8, both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (int32_t)r[i];
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- digit mirror ----------------------------------------------------------------
__global__ void make_digits_kernel(const float* __restrict__ mirror, int C, int64_t P,
                                   uint8_t* __restrict__ q8, int64_t slice_bytes,
                                   int* __restrict__ bad) {
  bool oob = false;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t lo[kSA] = {0, 0, 0, 0}, hi[kSA] = {0, 0, 0, 0};
    for (int c = 0; c < C; ++c) {
      const float v = __ldg(mirror + p * C + c);
      if (!(v >= 0.f && v <= 1.f)) oob = true;
      const float vc = fminf(fmaxf(v, 0.f), 1.f);
      const uint32_t V = (uint32_t)__float2int_rn(vc * 536870912.f);  // v 2^29: exact, rn
      const uint32_t sh = (uint32_t)(c & 3) * 8;
#pragma unroll
      for (int s = 0; s < kSA; ++s) {
        const uint32_t dg = (V >> (8 * s)) & 255u;
        if (c < 4) lo[s] |= dg << sh;
        else hi[s] |= dg << sh;
      }
    }
#pragma unroll
    for (int s = 0; s < kSA; ++s)
      *reinterpret_cast<uint2*>(q8 + s * slice_bytes + p * 8) = make_uint2(lo[s], hi[s]);
  }
  if (__syncthreads_or(oob) && threadIdx.x == 0) atomicOr(bad, 1);
}

// ---- the projection ----------------------------------------------------------------
struct TcArgs {
  const uint8_t* q8;
  int64_t slice_bytes;
  int img_w, w;
  const int* bad;
  const int32_t* xs;
  const int32_t* ys;
  int nx, ny;
  const int8_t* bop;    // [kblocks][kb/16][128][16]: row t * 32 + n = digit t of basis row 32 kblk + n
  const double* bmu;    // [d]
  float delta;          // the error band (2-norm), identical for every query
  int d, kb;
  double* out;          // [nx * ny][d]
  float* delta_out;     // [nx * ny]
  int tma_sp = 0;       // > 0: anchor spacing of the tensor map (strided tiles by TMA)
  int kb_first = 0;     // first basis block of this launch
  int nkb_run = 0;      // basis blocks of this launch (0: all)
};

// A work item = (tile of <= 128 consecutive anchors of one anchor row, basis block).
// 5-D TMA of one K group of 128 anchors at a uniform anchor spacing sp:
// dims (16 bytes, sp / 2 pixel pairs, anchor column, row, digit slice)
__device__ __forceinline__ void tma_group(void* dst, const CUtensorMap* map, int c1, int c2, int c3,
                                          int c4, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5, %6}], [%7];" ::"r"(mma::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(mma::smem_u32(mbar))
      : "memory");
}

template <bool kStrip>
__global__ void __launch_bounds__(kTcThreads, 1) project_tc_kernel(TcArgs a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int S = kStrip ? kStripStages : kStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (kStrip ? kStripBarOff : kBarOff));
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 1;
  uint64_t* bfull = tempty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     mma::smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < S; ++s) {
      mma::mbar_init(&full[s], 1);
      mma::mbar_init(&empty[s], 1);
    }
    mma::mbar_init(tfull, 1);
    mma::mbar_init(tempty, 8);
    mma::mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  mma::fence_before();
  __syncthreads();
  mma::fence_after();
  const uint32_t tmem = *tmem_slot;

  const int tpr = (a.nx + kTM - 1) / kTM;  // tiles per anchor row
  const int nkb = a.nkb_run > 0 ? a.nkb_run : (a.d + kNB - 1) / kNB;  // basis blocks (this launch)
  const int64_t n_items = (int64_t)tpr * a.ny * nkb;
  const int gpr = a.w >> 1;                // 16-byte groups per window row
  const int n_groups = a.kb >> 4;          // per slice
  const int n_chunks = (n_groups + kGC - 1) / kGC;

  if (kStrip && warp == 0) {
    // ---- producer (strip mode): the basis once, then one window row per stage --------
    if (lane == 0) {
      mma::mbar_expect_tx(bfull, (uint32_t)(n_groups * kNP * 16));
      mma::bulk_g2s(smem, a.bop + (int64_t)a.kb_first * n_groups * kNP * 16, n_groups * kNP * 16, bfull);
      int stage = 0;
      uint32_t ph = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int iy = (int)(it / tpr), ix0 = (int)(it - (int64_t)iy * tpr) * kTM;
        const int nt = min(kTM, a.nx - ix0);
        const int ay = a.ys[iy], x0 = a.xs[ix0];
        const uint32_t len = (uint32_t)(16 * (nt - 1) + 8 * a.w);
        for (int dy = 0; dy < a.w; ++dy) {
          mma::mbar_wait(&empty[stage], ph ^ 1u);
          uint8_t* A = smem + kBresBytes + stage * kStripStage;
          mma::mbar_expect_tx(&full[stage], kSA * len);
          const int64_t off = ((int64_t)(ay + dy) * a.img_w + x0) * 8;
          for (int s = 0; s < kSA; ++s)
            mma::bulk_g2s(A + s * kStripSlot, a.q8 + s * a.slice_bytes + off, len, &full[stage]);
          if (++stage == S) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (kStrip && warp == 1) {
    // ---- MMA issuer (strip mode) -------------------------------------------------------
    if (lane == 0) {
      mma::mbar_wait(bfull, 0);
      int stage = 0;
      uint32_t ph = 0, tph = 0;
      const int ksr = gpr >> 1;  // K steps per window row
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        mma::mbar_wait(tempty, tph ^ 1u);
        mma::fence_after();
        for (int dy = 0; dy < a.w; ++dy) {
          mma::mbar_wait(&full[stage], ph);
          mma::fence_after();
          const uint8_t* A = smem + kBresBytes + stage * kStripStage;
          for (int ks = 0; ks < ksr; ++ks) {
            const int g = dy * gpr + 2 * ks;
#pragma unroll
            for (int s = 0; s < kSA; ++s) {
              const int t0 = tmin_of(s), n = (kSB - t0) * kNB;
              const uint64_t ad =
                  mma::make_desc(mma::smem_u32(A + s * kStripSlot) + 32 * ks, 16, 128);
              const uint64_t bd = mma::make_desc(
                  mma::smem_u32(smem) + (g * kNP + t0 * kNB) * 16, kNP * 16, 128);
              mma_i8(tmem + (uint32_t)col0_of(s), ad, bd, idesc_i8(kTM, n),
                     (dy | ks) ? 1u : 0u);
            }
          }
          mma::commit(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            ph ^= 1u;
          }
        }
        mma::commit(tfull);
        tph ^= 1u;
      }
    }
  } else if (warp == 0) {
    // ---- producer ---------------------------------------------------------------------
    int stage = 0;
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t t = it / nkb;
      const int kblk = a.kb_first + (int)(it - t * nkb);
      const int iy = (int)(t / tpr), ix0 = (int)(t - (int64_t)iy * tpr) * kTM;
      const int nt = min(kTM, a.nx - ix0);
      const int ay = a.ys[iy];
      const int x0 = a.xs[ix0];
      // window rows of consecutive anchors are consecutive 16-byte blocks when
      // the anchors step by 2 pixels (16-byte aligned: even pixel index)
      const bool contig = a.xs[ix0 + nt - 1] - x0 == 2 * (nt - 1) && (x0 & 1) == 0 &&
                          (a.img_w & 1) == 0;
      // uniform spacing sp > 2: one 5-D TMA per (slice, K group) gathers the
      // 128 anchors' 16-byte chunks (anchor column stride sp pixels)
      const bool tma = !contig && a.tma_sp > 0 && (x0 & 1) == 0 &&
                       a.xs[ix0 + nt - 1] - x0 == a.tma_sp * (nt - 1);
      const int8_t* bsrc = a.bop + (int64_t)kblk * n_groups * kNP * 16;
      for (int c = 0; c < n_chunks; ++c) {
        mma::mbar_wait(&empty[stage], ph ^ 1u);
        uint8_t* A = smem + stage * kStageBytes;
        uint8_t* B = A + kSA * kASlice;
        const int g0 = c * kGC, ng = min(kGC, n_groups - g0);
        if (tma) {
          if (lane == 0) {
            mma::mbar_expect_tx(&full[stage], (uint32_t)(ng * (kSA * kAGroup + kNP * 16)));
            mma::bulk_g2s(B, bsrc + (int64_t)g0 * kNP * 16, ng * kNP * 16, &full[stage]);
            for (int g = 0; g < ng; ++g) {
              const int gg = g0 + g, dy = gg / gpr, dx = (gg - dy * gpr) * 2;
              const int X = x0 + dx, c2 = X / a.tma_sp, c1 = (X - c2 * a.tma_sp) >> 1;
              for (int s = 0; s < kSA; ++s)
                tma_group(A + s * kASlice + g * kAGroup, &tmap, c1, c2, ay + dy, s, &full[stage]);
            }
          }
        } else if (contig) {
          if (lane == 0) {
            mma::mbar_expect_tx(&full[stage], (uint32_t)(ng * (kSA * nt * 16 + kNP * 16)));
            mma::bulk_g2s(B, bsrc + (int64_t)g0 * kNP * 16, ng * kNP * 16, &full[stage]);
            for (int g = 0; g < ng; ++g) {
              const int gg = g0 + g, dy = gg / gpr, dx = (gg - dy * gpr) * 2;
              const int64_t off = ((int64_t)(ay + dy) * a.img_w + x0 + dx) * 8;
              for (int s = 0; s < kSA; ++s)
                mma::bulk_g2s(A + s * kASlice + g * kAGroup, a.q8 + s * a.slice_bytes + off,
                              nt * 16, &full[stage]);
            }
          }
        } else {
          // strided rows (spacing > 2, or a clamped last anchor): lane copies
          const uint4* src = reinterpret_cast<const uint4*>(bsrc + (int64_t)g0 * kNP * 16);
          for (int i = lane; i < ng * kNP; i += 32) reinterpret_cast<uint4*>(B)[i] = __ldg(src + i);
          for (int i = lane; i < ng * nt; i += 32) {
            const int g = i / nt, m = i - g * nt;
            const int gg = g0 + g, dy = gg / gpr, dx = (gg - dy * gpr) * 2;
            const int64_t off = ((int64_t)(ay + dy) * a.img_w + a.xs[ix0 + m] + dx) * 8;
#pragma unroll
            for (int s = 0; s < kSA; ++s) {
              const uint2* p = reinterpret_cast<const uint2*>(a.q8 + s * a.slice_bytes + off);
              const uint2 u0 = __ldg(p), u1 = __ldg(p + 1);
              *reinterpret_cast<uint4*>(A + s * kASlice + g * kAGroup + m * 16) =
                  make_uint4(u0.x, u0.y, u1.x, u1.y);
            }
          }
          mma::fence_async_smem();
          __syncwarp();
          if (lane == 0) mma::mbar_arrive(&full[stage]);
        }
        if (++stage == kStages) {
          stage = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: per K step one UMMA per A slice, N = the kept B digits ------------
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, tph = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        mma::mbar_wait(tempty, tph ^ 1u);
        mma::fence_after();
        for (int c = 0; c < n_chunks; ++c) {
          mma::mbar_wait(&full[stage], ph);
          mma::fence_after();
          const uint8_t* A = smem + stage * kStageBytes;
          const uint8_t* B = A + kSA * kASlice;
          const int ng = min(kGC, n_groups - c * kGC);
          for (int ks = 0; ks < (ng + 1) >> 1; ++ks) {
#pragma unroll
            for (int s = 0; s < kSA; ++s) {
              const int t0 = tmin_of(s), n = (kSB - t0) * kNB;
              const uint64_t ad = mma::make_desc(mma::smem_u32(A + s * kASlice) + ks * 2 * kAGroup,
                                                 kAGroup, 128);
              const uint64_t bd = mma::make_desc(
                  mma::smem_u32(B) + ks * 2 * kNP * 16 + t0 * kNB * 16, kNP * 16, 128);
              mma_i8(tmem + (uint32_t)col0_of(s), ad, bd, idesc_i8(kTM, n),
                     (c | ks) ? 1u : 0u);
            }
          }
          mma::commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            ph ^= 1u;
          }
        }
        mma::commit(tfull);
        tph ^= 1u;
      }
    }
  } else {
    // ---- epilogue: warp w (2..9) owns TMEM lanes 32 (w & 3) .. + 31 and basis
    // columns [16 h, 16 h + 16), h = (w - 2) / 4.  The digit products are
    // combined EXACTLY in two int64 halves, q^ 2^59 = P_hi 2^32 + P_lo
    // (|P_lo| < 2^54, |P_hi| < 2^44), so TMEM is released right after the loads
    // and the next tile's MMAs overlap the conversion and the stores.
    const int lg = warp & 3, h = (warp - 2) >> 2;
    const bool bad = *a.bad != 0;
    uint32_t tph = 0;
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int64_t t = it / nkb;
      const int kblk = a.kb_first + (int)(it - t * nkb);
      mma::mbar_wait(tfull, tph);
      tph ^= 1u;
      mma::fence_after();
      const int iy = (int)(t / tpr), ix0 = (int)(t - (int64_t)iy * tpr) * kTM;
      const int m = lg * 32 + lane;
      const bool valid = ix0 + m < a.nx;
      const int64_t q = (int64_t)iy * a.nx + ix0 + m;
      const uint32_t base = tmem + ((uint32_t)(lg * 32) << 16);
      long long plo[16], phi[16];
#pragma unroll
      for (int n = 0; n < 16; ++n) plo[n] = phi[n] = 0;
#pragma unroll
      for (int s = 0; s < kSA; ++s) {
#pragma unroll
        for (int tt = tmin_of(s); tt < kSB; ++tt) {
          int32_t r[16];
          tmem_ld16(base + (uint32_t)(col0_of(s) + (tt - tmin_of(s)) * kNB + 16 * h), r);
          tmem_wait_ld();
          const int u = s + tt;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (u <= 3) plo[i] += (long long)r[i] << (8 * u);
            else phi[i] += (long long)r[i] << (8 * (u - 4));
          }
        }
      }
      mma::fence_before();
      __syncwarp();
      if (lane == 0) mma::mbar_arrive(tempty);
      if (valid) {
        const int k0 = kblk * kNB + 16 * h;
        double* orow = a.out + q * a.d + k0;
#pragma unroll
        for (int n = 0; n < 16; ++n)
          if (k0 + n < a.d) {
            const double qh = dadd((double)phi[n] * 0x1p-27, (double)plo[n] * 0x1p-59);
            orow[n] = dsub(qh, a.bmu[k0 + n]);
          }
        if (kblk == 0 && h == 0) a.delta_out[q] = bad ? __int_as_float(0x7f800000) : a.delta;
      }
    }
  }
  mma::fence_before();
  __syncthreads();
  if (warp == 0) {
    mma::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

// ---- exact fallback for the ambiguous queries ------------------------------------------
// One warp per listed query.  Lane k accumulates the reference's projection
// chain acc = acc + ((double)v_j - mean_j) * basis[k][j], j ascending, no FMA
// (the centred window values are staged per 128-element chunk in shared
// memory, basis loads run 8 ahead).  Then, when the band held exactly two
// points, lanes 0 and 1 evaluate the reference's dist2 chain (km_tree.cpp:
// 15-22) for each and the lexicographic (dist^2, id) minimum is the answer.
constexpr int kListWarps = 8, kListChunk = 128;
__device__ __forceinline__ double dist2_chain(const double* q, const double* p, int d) {
  double acc = 0.0;
  for (int j = 0; j < d; ++j) {
    const double t = dsub(q[j], p[j]);
    acc = dadd(acc, dmul(t, t));
  }
  return acc;
}

// One warp per listed query: the reference's projection chain for every
// component (lane k: acc_k += c_j * B[k][j], j ascending), in chunks of 32
// window features; the next chunk's basis rows and features are loaded into
// registers while the current chunk's chain runs from shared memory.
constexpr int kResolveWarps = 2, kRC = 32;
__global__ void __launch_bounds__(32 * kResolveWarps) resolve_kernel(
    ResolveArgs r, const double* __restrict__ mean, const double* __restrict__ basisT, int KP,
    int D, int d, const double* __restrict__ proj) {
  __shared__ double bs_all[kResolveWarps][kRC][64];
  __shared__ double cs_all[kResolveWarps][kRC];
  __shared__ double qs_all[kResolveWarps][64];
  __shared__ double ps_all[kResolveWarps][2][64];  // the two band candidates' rows
  const int n = *r.count;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double(*bs)[64] = bs_all[warp];
  double* cs = cs_all[warp];
  double* qs = qs_all[warp];
  const int wc = r.w * r.C;
  const int nch = (D + kRC - 1) / kRC;
  for (int i = blockIdx.x * kResolveWarps + warp; i < n; i += gridDim.x * kResolveWarps) {
    const int32_t a = r.list[i];
    const int64_t base =
        ((int64_t)r.anchors.ys[a / r.anchors.nx] * r.img_w + r.anchors.xs[a % r.anchors.nx]) * r.C;
    double nb0[kRC], nb1[kRC], ncs = 0.0;
    auto load = [&](int ch) {
      const int j0 = ch * kRC;
      const double* bt = basisT + (int64_t)j0 * KP + lane;
#pragma unroll
      for (int u = 0; u < kRC; ++u) {
        const bool ok = j0 + u < D;
        nb0[u] = ok ? __ldg(bt + (int64_t)u * KP) : 0.0;
        nb1[u] = (KP > 32 && ok) ? __ldg(bt + (int64_t)u * KP + 32) : 0.0;
      }
      const int j = j0 + lane;
      if (j < D) {
        const int dy = j / wc, off = j - dy * wc;
        const float v = __ldg(r.mirror + base + (int64_t)dy * r.img_w * r.C + off);
        ncs = dsub((double)v, __ldg(mean + j));
      }
    };
    load(0);
    double acc0 = 0.0, acc1 = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
      __syncwarp();
#pragma unroll
      for (int u = 0; u < kRC; ++u) {
        bs[u][lane] = nb0[u];
        if (KP > 32) bs[u][lane + 32] = nb1[u];
      }
      cs[lane] = ncs;
      __syncwarp();
      const int jn = min(kRC, D - ch * kRC);
      if (ch + 1 < nch) load(ch + 1);
#pragma unroll 8
      for (int t = 0; t < jn; ++t) {
        const double cj = cs[t];
        acc0 = dadd(acc0, dmul(cj, bs[t][lane]));
        if (KP > 32) acc1 = dadd(acc1, dmul(cj, bs[t][lane + 32]));
      }
    }
    if (lane < d) qs[lane] = acc0;
    if (lane + 32 < d) qs[lane + 32] = acc1;
    __syncwarp();
    const int32_t c0 = r.c0[i], c1 = r.c1[i];
    if (c1 >= 0) {
      double(*ps)[64] = ps_all[warp];
      for (int j = lane; j < d; j += 32) {  // coalesced rows, then the chains from SMEM
        ps[0][j] = __ldg(proj + (int64_t)c0 * d + j);
        ps[1][j] = __ldg(proj + (int64_t)c1 * d + j);
      }
      __syncwarp();
      double dd = 0.0;
      if (lane < 2) dd = dist2_chain(qs, ps[lane], d);
      const double d1 = __shfl_sync(0xffffffffu, dd, 1);
      if (lane == 0) {
        const bool take1 = d1 < dd || (d1 == dd && c1 < c0);
        r.idx[a] = take1 ? c1 : c0;
        if (r.scanned) r.scanned[a] += 2;
        if (r.exact) r.exact[a] += 2;
      }
    } else {
      int slot = 0;
      if (lane == 0) slot = atomicAdd(r.full_count, 1);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (lane < d) r.full_q[(int64_t)slot * d + lane] = acc0;
      if (lane + 32 < d) r.full_q[(int64_t)slot * d + 32 + lane] = acc1;
      if (lane == 0) {
        r.full_anchor[slot] = a;
        r.full_seed[slot] = c0;
      }
    }
  }
}

__global__ void list_gather_kernel(const int32_t* __restrict__ src,
                                   const int32_t* __restrict__ list, const int* __restrict__ count,
                                   int32_t* __restrict__ out) {
  const int n = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = src[list[i]];
}

__global__ void list_scatter_kernel(const int32_t* __restrict__ list, const int* __restrict__ count,
                                    const int32_t* __restrict__ idx_c,
                                    const int64_t* __restrict__ sc_c,
                                    const int64_t* __restrict__ ex_c, int32_t* __restrict__ idx,
                                    int64_t* __restrict__ scanned, int64_t* __restrict__ exact) {
  const int n = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t a = list[i];
    idx[a] = idx_c[i];
    if (scanned) scanned[a] += sc_c[i];
    if (exact) exact[a] += ex_c[i];
  }
}

}  // namespace

void launch_make_digits(psg_ctx* ctx, const float* mirror, int C, int W, int H, uint8_t* q8,
                        int64_t slice_bytes, int* bad) {
  ProfScope _prof(ctx, K_MIRROR);
  const int64_t P = (int64_t)W * H;
  if (P <= 0) return;
  if (C > 8) fail(PSG_E_DOMAIN, "more than 8 channels are not supported");
  int64_t blocks = (P + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 16) blocks = (int64_t)ctx->num_sms * 16;
  make_digits_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(mirror, C, P, q8, slice_bytes,
                                                                bad);
  PSG_LAUNCHED(ctx);
}

bool tc_prepare(psg_ctx* ctx, Index& ix) {
  ix.tc = false;
  const int d = ix.d, D = ix.D, C = ix.C, w = ix.w;
  if (ix.from_vectors || d < 1 || d > 64 || C > 8 || (w & 1)) return false;
  for (double b : ix.h_basis)
    if (!(std::fabs(b) <= 1.0)) return false;
  const int kb = w * w * 8, ng = kb / 16, nkb = (d + kNB - 1) / kNB;
  std::vector<int8_t> op((size_t)nkb * ng * kNP * 16, 0);
  std::vector<double> bmu(d);
  double delta2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const double* row = ix.h_basis.data() + (size_t)k * D;
    const int blk = k / kNB, n = k - blk * kNB;
    long double mu = 0.0L;
    double l1 = 0.0;
    for (int j = 0; j < D; ++j) {
      const int pix = j / C, c = j - pix * C, kk = pix * 8 + c;  // window element -> K byte
      int64_t r = std::llrint(std::ldexp(row[j], 30));            // |r| <= 2^30
      for (int t = 0; t < kSB; ++t) {
        const int64_t dg = t < kSB - 1 ? ((r + 128) & 255) - 128 : r;  // last: |r| <= 64
        r = (r - dg) >> 8;
        const int nn = t * kNB + n;
        op[(((size_t)blk * ng + (kk >> 4)) * kNP + nn) * 16 + (kk & 15)] = (int8_t)dg;
      }
      mu += (long double)row[j] * (long double)ix.h_mean[j];
      l1 += std::fabs(row[j]);
    }
    bmu[k] = (double)mu;
    l1 *= 1.0 + 1e-12;
    const double e = std::ldexp(l1, -30) + std::ldexp((double)D, -31) +
                     std::ldexp(32640.0 * 513.0 * D, -59) + (2.0 * D + 2.0) * std::ldexp(l1, -53) +
                     std::ldexp(std::fabs(bmu[k]) + l1, -52) +
                     std::ldexp(20.0 * D, -53) /* the epilogue's fp64 digit combination */ + 1e-12;
    delta2 += e * e;
  }
  ix.tc_kb = kb;
  ix.tc_delta = (float)(std::sqrt(delta2) * (1.0 + 1e-6));
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.tc_b), op.size(), ctx->stream));
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.tc_bmu), sizeof(double) * d, ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(ix.tc_b, op.data(), op.size(), cudaMemcpyHostToDevice, ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(ix.tc_bmu, bmu.data(), sizeof(double) * d, cudaMemcpyHostToDevice,
                           ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  ix.tc = true;
  return true;
}

void launch_project_windows_tc(psg_ctx* ctx, const uint8_t* q8, int64_t slice_bytes, int img_w,
                               const int* bad, AnchorSet anchors, bool stride2, const Index& ix,
                               double* out, float* delta, int sp) {
  ProfScope _prof(ctx, K_PROJECT);
  if (anchors.count <= 0) return;
  if (!ix.tc) fail(PSG_E_LOGIC, "tensor-core projection without a prepared basis");
  TcArgs a{};
  a.q8 = q8;
  a.slice_bytes = slice_bytes;
  a.img_w = img_w;
  a.w = ix.w;
  a.bad = bad;
  a.xs = anchors.xs;
  a.ys = anchors.ys;
  a.nx = anchors.nx;
  a.ny = (int)(anchors.count / anchors.nx);
  a.bop = ix.tc_b;
  a.bmu = ix.tc_bmu;
  a.delta = ix.tc_delta;
  a.d = ix.d;
  a.kb = ix.tc_kb;
  a.out = out;
  a.delta_out = delta;
  static bool attr = false;
  if (!attr) {
    PSG_CUDA(cudaFuncSetAttribute(project_tc_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
    PSG_CUDA(cudaFuncSetAttribute(project_tc_kernel<true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kStripSmemBytes));
    attr = true;
  }
  const int nkb = (a.d + kNB - 1) / kNB;
  const int64_t items = (int64_t)((a.nx + kTM - 1) / kTM) * a.ny * nkb;
  const int blocks = (int)std::min<int64_t>(items, ctx->num_sms);
  // strip mode keeps one basis block resident: d > 32 runs one strip launch
  // per block (the window rows are streamed once per block)
  const bool strip = stride2 && a.w % 4 == 0 && a.w <= 8 && (img_w & 1) == 0 &&
                     (uint32_t)(a.kb / 16) * kNP * 16 <= kBresBytes;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  if (!strip && sp > 2 && (sp & 1) == 0 && (img_w & 1) == 0 && img_w >= sp) {
    // digit mirror slice s, row y, anchor column c, pixel pair p, byte e at
    // s * slice_bytes + y * img_w * 8 + c * sp * 8 + p * 16 + e
    // (a driver without the tensor-map entry point keeps the register-copy
    // staging of strided tiles: same results, slower)
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool probed = false;
    if (!probed) {
      probed = true;
      cudaDriverEntryPointQueryResult qr;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
          qr == cudaDriverEntryPointSuccess && fn)
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
      else
        (void)cudaGetLastError();
    }
    const int64_t rows = slice_bytes / ((int64_t)img_w * 8);
    const cuuint64_t dims[5] = {16, (cuuint64_t)(sp / 2), (cuuint64_t)(img_w / sp), (cuuint64_t)rows,
                                (cuuint64_t)kSA};
    const cuuint64_t strides[4] = {16, (cuuint64_t)sp * 8, (cuuint64_t)img_w * 8, (cuuint64_t)slice_bytes};
    const cuuint32_t box[5] = {16, 1, (cuuint32_t)kTM, 1, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUresult r = !encode ? CUDA_ERROR_NOT_SUPPORTED : encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<uint8_t*>(q8), dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) a.tma_sp = sp;
  }
  if (strip) {
    const int blocks1 = (int)std::min<int64_t>(items / nkb, ctx->num_sms);
    for (int b = 0; b < nkb; ++b) {
      TcArgs ab = a;
      ab.kb_first = b;
      ab.nkb_run = 1;
      project_tc_kernel<true><<<blocks1, kTcThreads, kStripSmemBytes, ctx->stream>>>(ab, tmap);
      if (b + 1 < nkb) PSG_LAUNCHED(ctx);
    }
  } else
    project_tc_kernel<false><<<blocks, kTcThreads, kSmemBytes, ctx->stream>>>(a, tmap);
  PSG_LAUNCHED(ctx);
}

void launch_resolve(psg_ctx* ctx, const ResolveArgs& r, const Index& ix) {
  ProfScope _prof(ctx, K_FALLBACK);
  const int KP = ix.d <= 32 ? 32 : 64;
  resolve_kernel<<<2 * ctx->num_sms, 32 * kResolveWarps, 0, ctx->stream>>>(r, ix.mean, ix.basis, KP,
                                                                        ix.D, ix.d, ix.proj);
  PSG_LAUNCHED(ctx);
}

void launch_list_gather_i32(psg_ctx* ctx, const int32_t* src, const int32_t* list,
                            const int* count, int32_t* out) {
  ProfScope _prof(ctx, K_FALLBACK);
  list_gather_kernel<<<ctx->num_sms, 256, 0, ctx->stream>>>(src, list, count, out);
  PSG_LAUNCHED(ctx);
}

void launch_list_scatter(psg_ctx* ctx, const int32_t* list, const int* count,
                         const int32_t* idx_c, const int64_t* sc_c, const int64_t* ex_c,
                         int32_t* idx, int64_t* scanned, int64_t* exact) {
  ProfScope _prof(ctx, K_FALLBACK);
  list_scatter_kernel<<<ctx->num_sms, 256, 0, ctx->stream>>>(list, count, idx_c, sc_c, ex_c, idx,
                                                             scanned, exact);
  PSG_LAUNCHED(ctx);
}

}  // namespace psg
