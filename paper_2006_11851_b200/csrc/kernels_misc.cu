// Per-stage build kernels (PCA inputs) and pyramid resampling.
//
//   fit_pca inputs   pca.cpp:57-65      mean + centred fp64 design matrix
//   downsample       image.cpp:38-62    block mean, acc * (1/f^2)
//   upsample_bilinear image.cpp:64-109  half-pixel centres, clamp to edge
//   fit_to           pipeline.cpp:39-52 crop / edge-replicate
#include <cuda_runtime.h>

#include "numerics.cuh"
#include "psg_internal.h"

namespace psg {

static int grid_cap(psg_ctx* ctx, int64_t n, int threads, int per_sm = 32) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)ctx->num_sms * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// Column means of the dense window matrix without materialising it: one CTA
// per feature j, fixed-order strided partial sums + fixed tree (deterministic).
__global__ void window_mean_kernel(const float* __restrict__ mirror, int img_w, int C, int w,
                                   int nxe, int64_t N, double* __restrict__ mean) {
  __shared__ double red[256];
  const int j = blockIdx.x;
  const int row = w * C;
  const int dy = j / row, rem = j - dy * row;
  const int dx = rem / C, c = rem - dx * C;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
    const int ax = (int)(i % nxe), ay = (int)(i / nxe);
    acc += (double)mirror[((int64_t)(ay + dy) * img_w + ax + dx) * C + c];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) mean[j] = red[0] / (double)N;
}

void launch_window_mean(psg_ctx* ctx, const float* mirror, int img_w, int C, int w, int nxe,
                        int64_t N, double* mean) {
  ProfScope _prof(ctx, K_BUILD);
  const int D = w * w * C;
  window_mean_kernel<<<D, 256, 0, ctx->stream>>>(mirror, img_w, C, w, nxe, N, mean);
  PSG_LAUNCHED(ctx);
}

__global__ void center_windows_kernel(const float* __restrict__ mirror, int img_w, int C, int w,
                                      int nxe, int64_t N, const double* __restrict__ mean,
                                      double* __restrict__ Xc) {
  const int D = w * w * C;
  const int row = w * C;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < N * D;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / D;
    const int j = (int)(f - i * D);
    const int ax = (int)(i % nxe), ay = (int)(i / nxe);
    const int dy = j / row, jj = j - dy * row;
    const float v = mirror[((int64_t)(ay + dy) * img_w + ax) * C + jj];
    Xc[f] = (double)v - mean[j];
  }
}

void launch_center_windows(psg_ctx* ctx, const float* mirror, int img_w, int C, int w, int nxe,
                           int64_t N, const double* mean, double* Xc) {
  ProfScope _prof(ctx, K_BUILD);
  const int64_t n = N * (int64_t)w * w * C;
  center_windows_kernel<<<grid_cap(ctx, n, 256), 256, 0, ctx->stream>>>(mirror, img_w, C, w, nxe,
                                                                         N, mean, Xc);
  PSG_LAUNCHED(ctx);
}

__global__ void vector_mean_kernel(const float* __restrict__ X, int64_t N, int D,
                                   double* __restrict__ mean) {
  __shared__ double red[256];
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) acc += (double)X[i * D + j];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) mean[j] = red[0] / (double)N;
}

void launch_vector_mean(psg_ctx* ctx, const float* X, int64_t N, int D, double* mean) {
  ProfScope _prof(ctx, K_BUILD);
  vector_mean_kernel<<<D, 256, 0, ctx->stream>>>(X, N, D, mean);
  PSG_LAUNCHED(ctx);
}

__global__ void center_vectors_kernel(const float* __restrict__ X, int64_t N, int D,
                                      const double* __restrict__ mean, double* __restrict__ Xc) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < N * D;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(f % D);
    Xc[f] = (double)X[f] - mean[j];
  }
}

void launch_center_vectors(psg_ctx* ctx, const float* X, int64_t N, int D, const double* mean,
                           double* Xc) {
  ProfScope _prof(ctx, K_BUILD);
  center_vectors_kernel<<<grid_cap(ctx, N * D, 256), 256, 0, ctx->stream>>>(X, N, D, mean, Xc);
  PSG_LAUNCHED(ctx);
}

// ---- pyramid ----------------------------------------------------------------------
__global__ void downsample_kernel(const double* __restrict__ in, int W, int H, int f,
                                  double* __restrict__ out, int ow, int oh) {
  const double inv = 1.0 / ((double)f * f);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)ow * oh;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / ow), x = (int)(i - (int64_t)y * ow);
    double acc = 0.0;
    for (int dy = 0; dy < f; ++dy)
      for (int dx = 0; dx < f; ++dx)
        acc = dadd(acc, in[(int64_t)(y * f + dy) * W + x * f + dx]);
    out[i] = dmul(acc, inv);
  }
}

// Guidance ramps (BASELINE cfg: "row index / (H-1) as fp32", widened to
// fp64): even planes vary with the row, odd planes with the column.  IEEE
// fp32 division, identical to the host rule.
__global__ void ramp_planes_kernel(int G, int W, int H, double* __restrict__ out) {
  const int64_t P = (int64_t)W * H;
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < P * G;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(f / P);
    const int64_t i = f - (int64_t)g * P;
    const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
    double v;
    if (g % 2 == 0)
      v = H > 1 ? (double)__fdiv_rn((float)y, (float)(H - 1)) : 0.5;
    else
      v = W > 1 ? (double)__fdiv_rn((float)x, (float)(W - 1)) : 0.5;
    out[f] = v;
  }
}

void launch_ramp_planes(psg_ctx* ctx, int G, int W, int H, double* out) {
  ProfScope _prof(ctx, K_PYRAMID);
  const int64_t n = (int64_t)W * H * G;
  if (n <= 0) return;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  ramp_planes_kernel<<<(int)blocks, 256, 0, ctx->stream>>>(G, W, H, out);
  PSG_LAUNCHED(ctx);
}

// Seed for a stage's first search from the previous stage's assignment
// (synthesize driver): each new anchor takes the previous anchor whose window
// centre is nearest (in the previous stage's pixel grid, scale = 1 for the
// next window size of a level, 2^k across levels) and shifts that anchor's
// exemplar window by the same offset.  Only the search bound uses it.
__device__ __forceinline__ int nearest_centre(const int32_t* __restrict__ pos, int n, double half,
                                              double c) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((double)pos[mid] + half <= c) lo = mid;
    else hi = mid - 1;
  }
  if (lo + 1 < n && fabs((double)pos[lo + 1] + half - c) < fabs((double)pos[lo] + half - c)) ++lo;
  return lo;
}

__global__ void carry_seed_kernel(CarryArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < a.nq; q += stride) {
    const int bx = (int)(q % a.nx), by = (int)(q / a.nx);
    const double inv = 1.0 / a.scale, ph = 0.5 * a.pw;
    const double cx = ((double)a.xs[bx] + 0.5 * a.w) * inv;
    const double cy = ((double)a.ys[by] + 0.5 * a.w) * inv;
    const int j = nearest_centre(a.pxs, a.pnx, ph, cx);
    const int k = nearest_centre(a.pys, a.pny, ph, cy);
    const int32_t e = a.pidx[(int64_t)k * a.pnx + j];
    const double ecx = (double)(e % a.pnxe) + ph + (cx - ((double)a.pxs[j] + ph));
    const double ecy = (double)(e / a.pnxe) + ph + (cy - ((double)a.pys[k] + ph));
    const int tx = min(max((int)lrint(ecx * a.scale - 0.5 * a.w), 0), a.nxe - 1);
    const int ty = min(max((int)lrint(ecy * a.scale - 0.5 * a.w), 0), a.nye - 1);
    a.out[q] = ty * a.nxe + tx;
  }
}

void launch_carry_seed(psg_ctx* ctx, const CarryArgs& a) {
  ProfScope _prof(ctx, K_PYRAMID);
  if (a.nq <= 0) return;
  carry_seed_kernel<<<grid_cap(ctx, a.nq, 256), 256, 0, ctx->stream>>>(a);
  PSG_LAUNCHED(ctx);
}

void launch_downsample(psg_ctx* ctx, const double* in, int W, int H, int f, double* out) {
  ProfScope _prof(ctx, K_PYRAMID);
  const int ow = W / f, oh = H / f;
  downsample_kernel<<<grid_cap(ctx, (int64_t)ow * oh, 256), 256, 0, ctx->stream>>>(in, W, H, f,
                                                                                    out, ow, oh);
  PSG_LAUNCHED(ctx);
}

__device__ __forceinline__ void src_coord(int dst, int limit, double inv, int& lo, int& hi,
                                          double& frac) {
  const double s = dsub(dmul(dadd((double)dst, 0.5), inv), 0.5);
  const double fl = floor(s);
  lo = (int)fl;
  frac = dsub(s, fl);
  hi = min(lo + 1, limit - 1);
  lo = max(lo, 0);
  if (hi < lo) hi = lo;
}

__global__ void upsample_kernel(const double* __restrict__ in, int W, int H, int f,
                                double* __restrict__ out) {
  const int ow = W * f, oh = H * f;
  const double inv = 1.0 / f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)ow * oh;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / ow), x = (int)(i - (int64_t)y * ow);
    int y0, y1, x0, x1;
    double fy, fx;
    src_coord(y, H, inv, y0, y1, fy);
    src_coord(x, W, inv, x0, x1, fx);
    const double v00 = in[(int64_t)y0 * W + x0], v10 = in[(int64_t)y0 * W + x1];
    const double v01 = in[(int64_t)y1 * W + x0], v11 = in[(int64_t)y1 * W + x1];
    const double gx = dsub(1.0, fx), gy = dsub(1.0, fy);
    const double a = dadd(dmul(gx, v00), dmul(fx, v10));
    const double b = dadd(dmul(gx, v01), dmul(fx, v11));
    out[i] = dadd(dmul(gy, a), dmul(fy, b));
  }
}

void launch_upsample_bilinear(psg_ctx* ctx, const double* in, int W, int H, int f, double* out) {
  ProfScope _prof(ctx, K_PYRAMID);
  upsample_kernel<<<grid_cap(ctx, (int64_t)W * f * H * f, 256), 256, 0, ctx->stream>>>(in, W, H,
                                                                                       f, out);
  PSG_LAUNCHED(ctx);
}

__global__ void fit_to_kernel(const double* __restrict__ in, int W, int H, int ow, int oh,
                              double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)ow * oh;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / ow), x = (int)(i - (int64_t)y * ow);
    const int sy = min(y, H - 1), sx = min(x, W - 1);
    out[i] = in[(int64_t)sy * W + sx];
  }
}

void launch_fit_to(psg_ctx* ctx, const double* in, int W, int H, int ow, int oh, double* out) {
  ProfScope _prof(ctx, K_PYRAMID);
  fit_to_kernel<<<grid_cap(ctx, (int64_t)ow * oh, 256), 256, 0, ctx->stream>>>(in, W, H, ow, oh,
                                                                               out);
  PSG_LAUNCHED(ctx);
}

}  // namespace psg
