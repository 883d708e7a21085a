// Covariance of the dense window database without materialising it
// (fit_pca's cov = Xc^T Xc / (n-1), pca.cpp:57-65, for X = extract_all of the
// exemplar, neighborhood.cpp:103-118).
//
// Entry (i, j) with i = (dy1, dx1, c1), j = (dy2, dx2, c2) is a sum over all
// anchors a of Y_c1(a + (dy1, dx1)) * Y_c2(a + (dy2, dx2)): a box sum, over the
// anchor rectangle shifted by (dy1, dx1), of the product image
// Y_c1(p) * Y_c2(p + delta) with delta = (dy2 - dy1, dx2 - dx1).  One CTA per
// (c1, c2, delta) computes the box sums for every (dy1, dx1) with sliding row
// and column sums: O(C^2 (2w-1)^2 ew eh) work instead of the O(N D^2) of a
// DSYRK over the N x D window matrix (N = 50,625, D = 5,120 at cfg3 w = 32:
// 1.3 TFLOP -> 6.5 GFLOP).  Y = x - s_c (a per-channel shift close to the
// mean) keeps the raw product sums small; cov = (S - N m_i m_j) / (N - 1) with
// the window means m.  Symmetric halves are computed once and mirrored.
// fit_pca's bit-level parity is unpinned (Eigen3 is absent); the
// entries agree with the DSYRK formulation to ~1e-14 relative.
#include <cuda_runtime.h>

#include "psg_internal.h"

namespace psg {

namespace {

__global__ void shifted_planes_kernel(const float* __restrict__ mirror, int C, int64_t P,
                                      const double* __restrict__ shift, double* __restrict__ Y) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < P * C;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(f / P);
    const int64_t p = f - (int64_t)c * P;
    Y[f] = (double)mirror[p * C + c] - shift[c];
  }
}

// grid: x = delta index over (2w-1)^2, y = c1 * C + c2
__global__ void __launch_bounds__(256) window_cov_kernel(const double* __restrict__ Y, int ew,
                                                         int eh, int C, int w,
                                                         const double* __restrict__ wmean,
                                                         const double* __restrict__ shift,
                                                         double* __restrict__ cov) {
  extern __shared__ double Rs[];  // [nrows][nx1]
  const int W2 = 2 * w - 1;
  const int ddy = (int)(blockIdx.x / W2) - (w - 1), ddx = (int)(blockIdx.x % W2) - (w - 1);
  const int c1 = blockIdx.y / C, c2 = blockIdx.y % C;
  // symmetric half: (c1, c2, delta) mirrors (c2, c1, -delta)
  if (c1 > c2 || (c1 == c2 && (ddy < 0 || (ddy == 0 && ddx < 0)))) return;
  const int nxe = ew - w + 1, nye = eh - w + 1;
  const int64_t N = (int64_t)nxe * nye;
  const int D = w * w * C;
  const int ny1 = w - abs(ddy), nx1 = w - abs(ddx);
  const int y0 = max(0, -ddy), x0 = max(0, -ddx);
  const int nrows = ny1 - 1 + nye;
  const double* Y1 = Y + (int64_t)c1 * ew * eh;
  const double* Y2 = Y + (int64_t)c2 * ew * eh;
  // row sums R(y, dx1) = sum_{x = dx1}^{dx1 + nxe - 1} Y1(y, x) Y2(y + ddy, x + ddx)
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
    const int y = y0 + r;
    const double* a = Y1 + (int64_t)y * ew;
    const double* b = Y2 + (int64_t)(y + ddy) * ew + ddx;
    double acc = 0.0;
    for (int x = x0; x < x0 + nxe; ++x) acc += a[x] * b[x];
    Rs[r * nx1] = acc;
    for (int t = 1; t < nx1; ++t) {
      const int xo = x0 + t - 1, xi = x0 + t - 1 + nxe;
      acc += a[xi] * b[xi] - a[xo] * b[xo];
      Rs[r * nx1 + t] = acc;
    }
  }
  __syncthreads();
  // column sums over the nye rows of each box, sliding over dy1
  const double inv = 1.0 / (double)(N - 1);
  for (int t = threadIdx.x; t < nx1; t += blockDim.x) {
    double B = 0.0;
    for (int r = 0; r < nye; ++r) B += Rs[r * nx1 + t];
    for (int u = 0; u < ny1; ++u) {
      if (u > 0) B += Rs[(u - 1 + nye) * nx1 + t] - Rs[(u - 1) * nx1 + t];
      const int dy1 = y0 + u, dx1 = x0 + t;
      const int i = (dy1 * w + dx1) * C + c1;
      const int j = ((dy1 + ddy) * w + dx1 + ddx) * C + c2;
      const double mi = wmean[i] - shift[c1], mj = wmean[j] - shift[c2];
      const double v = (B - (double)N * mi * mj) * inv;
      cov[(int64_t)i * D + j] = v;
      cov[(int64_t)j * D + i] = v;
    }
  }
}

}  // namespace

void launch_window_cov(psg_ctx* ctx, const float* ex_mirror, int ew, int eh, int C, int w,
                       const double* wmean, double* cov) {
  ProfScope _prof(ctx, K_BUILD);
  const int64_t P = (int64_t)ew * eh;
  double* Y = nullptr;
  double* shift = nullptr;
  PSG_CUDA(cudaMallocAsync(&Y, sizeof(double) * P * C, ctx->stream));
  PSG_CUDA(cudaMallocAsync(&shift, sizeof(double) * C, ctx->stream));
  // shift = the mean of window coordinate (0, 0, c): within rounding of the channel mean
  PSG_CUDA(cudaMemcpyAsync(shift, wmean, sizeof(double) * C, cudaMemcpyDeviceToDevice,
                           ctx->stream));
  int64_t blocks = (P * C + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 32) blocks = (int64_t)ctx->num_sms * 32;
  shifted_planes_kernel<<<(int)blocks, 256, 0, ctx->stream>>>(ex_mirror, C, P, shift, Y);
  PSG_LAUNCHED(ctx);
  const int W2 = 2 * w - 1;
  const int nrows_max = eh;  // ny1 - 1 + nye <= eh
  const size_t smem = sizeof(double) * (size_t)nrows_max * w;
  PSG_CUDA(cudaFuncSetAttribute(window_cov_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  window_cov_kernel<<<dim3((unsigned)(W2 * W2), (unsigned)(C * C)), 256, smem, ctx->stream>>>(
      Y, ew, eh, C, w, wmean, shift, cov);
  PSG_LAUNCHED(ctx);
  PSG_CUDA(cudaFreeAsync(Y, ctx->stream));
  PSG_CUDA(cudaFreeAsync(shift, ctx->stream));
}

}  // namespace psg
