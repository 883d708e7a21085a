// PCA projection of the E-step's query windows on the 5th-gen tensor cores.
//
// The reference projects every window in fp64, j-sequential, mul then add
// (pca.cpp:27-41, called per query from optimizer.cpp:228-230).  That chain is
// what the nearest-neighbour comparison ultimately uses, but almost every
// query's winner is separated from its runner-up by far more than the chain's
// rounding.  So the E-step first computes an approximation q^ with a RIGOROUS
// error bound on the tensor cores, and the search keeps every candidate within
// that bound of the best (kernels_search.cu, approximate-query mode); only the
// queries whose winner is not separated (near-ties, ~0.1%) are re-projected
// with the exact chain and searched again (launch_project_list + the exact
// tile search), so NN indices stay bit-identical to the reference's.
//
// The approximation is computed EXACTLY in integers:
//   v^  = V 2^-21,  V = rint(v 2^21) in [0, 2^21]   (|v - v^| <= 2^-22)
//   B^  = Bq 2^-22, Bq = rint(B 2^22)               (|B - B^| <= 2^-23)
//   q^_k = (sum_j Bq_kj V_j) 2^-43 - (B mu)_k
// V is split into three unsigned base-256 digits (u8), Bq into three balanced
// signed digits (s8); the nine digit products run as tcgen05.mma kind::i8
// (int32 accumulation: exact) into five TMEM accumulators, one per digit
// scale 256^(s+t), combined in int64 in the epilogue.  An extra basis row of
// ones returns sum_j V_j, which bounds the basis rounding per query:
//   |q^_k - q_k| <= 2^-22 |B_k|_1 + 2^-23 sum_j v^_j + (2D+2) 2^-53 |B_k|_1
//                   + 2^-52 (|B mu_k| + |q^_k|) + 1e-12.
//
// Operands: windows of the digit mirror q8 [3][H][W][8] (8-byte pixels, so a
// window row is w x 8 contiguous bytes and, at spacing 2, consecutive anchors'
// 16-byte groups are consecutive 16-byte blocks: coalesced loads), staged in
// shared memory in the UMMA K-major no-swizzle layout (K group g of the 128
// anchors = one contiguous 2 KB block); the basis digits stream in per chunk.
// One CTA = 128 anchors (UMMA M), 4 warps: all threads stage, one thread
// issues the MMAs, all threads drain TMEM (lane = anchor).
#include <cstdint>
#include <cmath>
#include <vector>

#include "numerics.cuh"
#include "psg_internal.h"
#include "umma.cuh"

namespace psg {
namespace {

constexpr int kTM = 128;          // anchors per CTA (UMMA M)
constexpr int kGC = 4;            // 16-byte K groups per chunk (2 UMMA K-steps of 32 bytes)
constexpr int kAccs = 5;          // digit scales 256^0 .. 256^4
constexpr int kSlices = 3;
constexpr uint32_t kAGroup = kTM * 16;               // 2 KB per K group (one slice)
constexpr uint32_t kASlice = kGC * kAGroup;          // 8 KB per slice per chunk

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
    uint32_t lo[kSlices] = {0, 0, 0}, hi[kSlices] = {0, 0, 0};
    for (int c = 0; c < C; ++c) {
      const float v = __ldg(mirror + p * C + c);
      if (!(v >= 0.f && v <= 1.f)) oob = true;
      const float vc = fminf(fmaxf(v, 0.f), 1.f);
      const uint32_t V = (uint32_t)__float2int_rn(vc * 2097152.f);  // exact scaling, rn
      const uint32_t sh = (uint32_t)(c & 3) * 8;
      const uint32_t d0 = V & 255u, d1 = (V >> 8) & 255u, d2 = V >> 16;
      if (c < 4) {
        lo[0] |= d0 << sh;
        lo[1] |= d1 << sh;
        lo[2] |= d2 << sh;
      } else {
        hi[0] |= d0 << sh;
        hi[1] |= d1 << sh;
        hi[2] |= d2 << sh;
      }
    }
#pragma unroll
    for (int s = 0; s < kSlices; ++s)
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
  int nx;
  int64_t n;
  const int8_t* bop;    // [3][kb/16][np][16]
  const double* bmu;    // [d]
  const double* err;    // [d]
  int d, kb;
  double* out;          // [n][d]
  float* delta;         // [n]
};

template <int NP>
__global__ void __launch_bounds__(kTM) project_tc_kernel(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t kBSlice = kGC * NP * 16;                  // per slice per chunk
  constexpr uint32_t kStage = kSlices * (kASlice + kBSlice);
  constexpr uint32_t kCols = kAccs * NP <= 128 ? 128 : (kAccs * NP <= 256 ? 256 : 512);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * kStage);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     mma::smem_u32(tmem_slot)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    mma::mbar_init(&bar[0], 1);
    mma::mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  mma::fence_before();
  __syncthreads();
  mma::fence_after();
  const uint32_t tmem = *tmem_slot;

  // this thread's anchor (row tid of the tile)
  const int64_t q = (int64_t)blockIdx.x * kTM + tid;
  const bool valid = q < a.n;
  int64_t pix0 = 0;  // first pixel of the window
  if (valid) pix0 = (int64_t)a.ys[q / a.nx] * a.img_w + a.xs[q % a.nx];
  const int gpr = a.w >> 1;               // 16-byte groups per window row
  const int n_groups = a.kb >> 4;         // per slice
  const int n_chunks = (n_groups + kGC - 1) / kGC;
  constexpr uint32_t kIdesc = idesc_i8(kTM, NP);

  for (int c = 0; c < n_chunks; ++c) {
    const int st = c & 1;
    uint8_t* A = smem + st * kStage;
    uint8_t* B = A + kSlices * kASlice;
    if (c >= 2) mma::mbar_wait(&bar[st], (uint32_t)((c - 2) >> 1) & 1u);  // stage free
    const int g0 = c * kGC;
    const int ng = min(kGC, n_groups - g0);
    // basis digits of this chunk: per slice a contiguous ng * NP * 16 bytes
    for (int s = 0; s < kSlices; ++s) {
      const uint4* src = reinterpret_cast<const uint4*>(a.bop + ((int64_t)s * n_groups + g0) * NP * 16);
      uint4* dst = reinterpret_cast<uint4*>(B + s * kBSlice);
      for (int i = tid; i < ng * NP; i += kTM) dst[i] = __ldg(src + i);
    }
    // window digits: 16 bytes (two 8-byte pixels) per (slice, group), all
    // loads of the chunk issued before the stores
    uint2 v[kSlices][kGC][2];
#pragma unroll
    for (int g = 0; g < kGC; ++g) {
      const int gg = g0 + g;
      const int dy = gg / gpr, dx = (gg - dy * gpr) * 2;
      const int64_t off = (pix0 + (int64_t)dy * a.img_w + dx) * 8;
#pragma unroll
      for (int s = 0; s < kSlices; ++s) {
        if (valid && g < ng) {
          const uint2* p = reinterpret_cast<const uint2*>(a.q8 + s * a.slice_bytes + off);
          v[s][g][0] = __ldg(p);
          v[s][g][1] = __ldg(p + 1);
        } else {
          v[s][g][0] = v[s][g][1] = make_uint2(0u, 0u);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < kSlices; ++s)
#pragma unroll
      for (int g = 0; g < kGC; ++g)
        *reinterpret_cast<uint4*>(A + s * kASlice + g * kAGroup + tid * 16) =
            make_uint4(v[s][g][0].x, v[s][g][0].y, v[s][g][1].x, v[s][g][1].y);
    mma::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      mma::fence_after();
      const int ksteps = (ng + 1) >> 1;  // 32 bytes = 2 groups per UMMA
      for (int ks = 0; ks < ksteps; ++ks) {
        // K-step ks covers groups 2ks, 2ks+1: LBO = group stride, SBO = 8-row stride
#pragma unroll
        for (int s = 0; s < kSlices; ++s) {
          const uint64_t ad = mma::make_desc(mma::smem_u32(A + s * kASlice) + ks * 2 * kAGroup,
                                             kAGroup, 128);
#pragma unroll
          for (int t = 0; t < kSlices; ++t) {
            const uint64_t bd = mma::make_desc(mma::smem_u32(B + t * kBSlice) + ks * 2 * NP * 16,
                                               NP * 16, 128);
            const int u = s + t;
            // the first product into each accumulator overwrites it
            const bool first = c == 0 && ks == 0 && (u < 3 ? s == 0 : t == 2);
            mma_i8(tmem + (uint32_t)(u * NP), ad, bd, kIdesc, first ? 0u : 1u);
          }
        }
      }
      mma::commit(&bar[st]);
    }
  }
  const int cl = n_chunks - 1;
  mma::mbar_wait(&bar[cl & 1], (uint32_t)(cl >> 1) & 1u);
  mma::fence_after();

  // ---- epilogue: warp w drains TMEM lanes 32w..32w+31 (lane = anchor) ----------------
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const bool bad = *a.bad != 0;
  double* orow = a.out + (valid ? q : 0) * a.d;
  double err2 = 0.0, sumv = 0.0;
  double eq[NP];  // q^ (first d columns)
#pragma unroll
  for (int nb = 0; nb < NP; nb += 16) {
    int32_t r[kAccs][16];
#pragma unroll
    for (int u = 0; u < kAccs; ++u) tmem_ld16(tmem + lane_base + (uint32_t)(u * NP + nb), r[u]);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int64_t P = 0;
#pragma unroll
      for (int u = kAccs - 1; u >= 0; --u) P = P * 256 + (int64_t)r[u][i];
      const int n = nb + i;
      if (n < a.d) eq[n] = (double)P * 0x1p-43;  // exact: |P| < 2^53
      else if (n == a.d) sumv = (double)P * 0x1p-21;  // sum_j v^_j (exact)
    }
  }
  if (valid) {
#pragma unroll
    for (int n = 0; n < NP; ++n) {
      if (n >= a.d) break;
      const double qk = eq[n] - a.bmu[n];
      orow[n] = qk;
      const double e = a.err[n] + 0x1p-23 * sumv + 0x1p-52 * fabs(qk);
      err2 += e * e;
    }
    a.delta[q] = bad ? __int_as_float(0x7f800000) : __double2float_ru(sqrt(err2) * (1.0 + 1e-9));
  }
  mma::fence_before();
  __syncthreads();
  if (warp == 0) {
    mma::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
  }
}

template <int NP>
void launch_tc(psg_ctx* ctx, const TcArgs& a) {
  constexpr uint32_t kBSlice = kGC * NP * 16;
  constexpr uint32_t kStage = kSlices * (kASlice + kBSlice);
  const size_t sm = 2 * kStage + 64;
  auto k = project_tc_kernel<NP>;
  static bool attr = false;
  if (!attr) {
    PSG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  const int64_t blocks = (a.n + kTM - 1) / kTM;
  k<<<(unsigned)blocks, kTM, sm, ctx->stream>>>(a);
  PSG_LAUNCHED(ctx);
}

// ---- exact fallback for listed anchors -------------------------------------------
// One warp per listed anchor; lane k accumulates the reference's chain
// acc = acc + ((double)v_j - mean_j) * basis[k][j], j ascending, no FMA.
__global__ void project_list_kernel(const float* __restrict__ mirror, int img_w, int C, int w,
                                    const int32_t* __restrict__ xs, const int32_t* __restrict__ ys,
                                    int nx, const int32_t* __restrict__ list,
                                    const int* __restrict__ count, const double* __restrict__ mean,
                                    const double* __restrict__ basisT, int KP, int D, int d,
                                    double* __restrict__ out) {
  const int n = *count;
  const int lane = threadIdx.x & 31;
  const int wc = w * C;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (gridDim.x * blockDim.x) >> 5) {
    const int32_t a = list[i];
    const int64_t base = ((int64_t)ys[a / nx] * img_w + xs[a % nx]) * C;
    double acc0 = 0.0, acc1 = 0.0;
    int dy = 0, off = 0;
    for (int j = 0; j < D; ++j) {
      const float v = __ldg(mirror + base + (int64_t)dy * img_w * C + off);
      if (++off == wc) {
        off = 0;
        ++dy;
      }
      const double cj = dsub((double)v, __ldg(mean + j));
      acc0 = dadd(acc0, dmul(cj, __ldg(basisT + (int64_t)j * KP + lane)));
      if (KP > 32) acc1 = dadd(acc1, dmul(cj, __ldg(basisT + (int64_t)j * KP + 32 + lane)));
    }
    if (lane < d) out[(int64_t)i * d + lane] = acc0;
    if (lane + 32 < d) out[(int64_t)i * d + 32 + lane] = acc1;
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
  const int np = ((d + 1 + 15) / 16) * 16;
  const int kb = w * w * 8;
  for (double b : ix.h_basis)
    if (!(std::fabs(b) <= 1.0)) return false;
  const int ng = kb / 16;
  std::vector<int8_t> op((size_t)kSlices * kb * np, 0);
  auto put = [&](int n, int kk, int64_t bq) {
    int64_t r = bq;
    for (int t = 0; t < kSlices; ++t) {
      int64_t dg = ((r + 128) & 255) - 128;
      if (t == kSlices - 1) dg = r;  // |r| <= 64 after two balanced digits
      r = (r - dg) >> 8;
      const size_t o = ((size_t)t * ng + (kk >> 4)) * np * 16 + (size_t)(n >> 3) * 128 +
                       (size_t)(n & 7) * 16 + (kk & 15);
      op[o] = (int8_t)dg;
    }
  };
  std::vector<double> bmu(d), err(d);
  for (int k = 0; k < d; ++k) {
    const double* row = ix.h_basis.data() + (size_t)k * D;
    long double mu = 0.0L;
    double l1 = 0.0;
    for (int j = 0; j < D; ++j) {
      const int pix = j / C, c = j - pix * C;  // window element (pixel, channel)
      put(k, pix * 8 + c, std::llrint(std::ldexp(row[j], 22)));
      mu += (long double)row[j] * (long double)ix.h_mean[j];
      l1 += std::fabs(row[j]);
    }
    bmu[k] = (double)mu;
    l1 *= 1.0 + 1e-12;
    err[k] = std::ldexp(l1, -22) + (2.0 * D + 2.0) * std::ldexp(l1, -53) +
             std::ldexp(std::fabs(bmu[k]), -52) + 1e-12;
  }
  for (int j = 0; j < D; ++j) {  // the ones row: sum_j V_j
    const int pix = j / C, c = j - pix * C;
    put(d, pix * 8 + c, 1);
  }
  ix.tc_np = np;
  ix.tc_kb = kb;
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.tc_b), op.size(), ctx->stream));
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.tc_bmu), sizeof(double) * d, ctx->stream));
  PSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ix.tc_err), sizeof(double) * d, ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(ix.tc_b, op.data(), op.size(), cudaMemcpyHostToDevice, ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(ix.tc_bmu, bmu.data(), sizeof(double) * d, cudaMemcpyHostToDevice,
                           ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(ix.tc_err, err.data(), sizeof(double) * d, cudaMemcpyHostToDevice,
                           ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  ix.tc = true;
  return true;
}

void launch_project_windows_tc(psg_ctx* ctx, const uint8_t* q8, int64_t slice_bytes, int img_w,
                               const int* bad, AnchorSet anchors, const Index& ix, double* out,
                               float* delta) {
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
  a.n = anchors.count;
  a.bop = ix.tc_b;
  a.bmu = ix.tc_bmu;
  a.err = ix.tc_err;
  a.d = ix.d;
  a.kb = ix.tc_kb;
  a.out = out;
  a.delta = delta;
  switch (ix.tc_np) {
    case 16: launch_tc<16>(ctx, a); break;
    case 32: launch_tc<32>(ctx, a); break;
    case 48: launch_tc<48>(ctx, a); break;
    case 64: launch_tc<64>(ctx, a); break;
    case 80: launch_tc<80>(ctx, a); break;
    default: fail(PSG_E_LOGIC, "unsupported tensor-core projection width");
  }
}

void launch_project_list(psg_ctx* ctx, const float* mirror, int img_w, int C, int w,
                         AnchorSet anchors, const int32_t* list, const int* count,
                         const Index& ix, double* out) {
  ProfScope _prof(ctx, K_PROJECT);
  const int KP = ix.d <= 32 ? 32 : 64;
  project_list_kernel<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(
      mirror, img_w, C, w, anchors.xs, anchors.ys, anchors.nx, list, count, ix.mean, ix.basis, KP,
      ix.D, ix.d, out);
  PSG_LAUNCHED(ctx);
}

void launch_list_gather_i32(psg_ctx* ctx, const int32_t* src, const int32_t* list,
                            const int* count, int32_t* out) {
  ProfScope _prof(ctx, K_SEARCH);
  list_gather_kernel<<<ctx->num_sms, 256, 0, ctx->stream>>>(src, list, count, out);
  PSG_LAUNCHED(ctx);
}

void launch_list_scatter(psg_ctx* ctx, const int32_t* list, const int* count,
                         const int32_t* idx_c, const int64_t* sc_c, const int64_t* ex_c,
                         int32_t* idx, int64_t* scanned, int64_t* exact) {
  ProfScope _prof(ctx, K_SEARCH);
  list_scatter_kernel<<<ctx->num_sms, 256, 0, ctx->stream>>>(list, count, idx_c, sc_c, ex_c, idx,
                                                             scanned, exact);
  PSG_LAUNCHED(ctx);
}

}  // namespace psg
