// Per-stage PCA fit on device (fit_pca, pca.cpp:49-101).
//
// mean (deterministic per-feature reduction) -> centred fp64 design matrix
// -> covariance X^T X / (n-1) with cuBLAS DSYRK -> cuSOLVER eigensolver -> on
// the host: variances descending and clamped >= 0 (pca.cpp:72-77), smallest
// prefix reaching the variance target (pca.cpp:79-87) optionally capped or
// fixed (the BASELINE configs' d), sign fix "largest-|.| entry positive",
// first index on ties (pca.cpp:92-95, Eigen maxCoeff).
//
// When the retained dimension is bounded (d fixed or capped, always <= 64) only
// the top eigenpairs are computed (DSYEVDX, range I): the total variance is the
// trace of the covariance, the reference's sum of clamped eigenvalues up to
// rounding of the (tiny) negative ones; the unreported tail of `variances` is
// zero.  Unbounded variance targets use the full DSYEVD spectrum.
//
// Eigen3 is not available to pin the reference's fit bit-for-bit (SURVEY
// §8c: "parity unpinned"); the fit is property-tested and the resulting basis
// is injected into the oracle for every parity check.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "psg_internal.h"

namespace psg {

namespace {
void cublas_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS)
    fail(PSG_E_CUDA, std::string(what) + ": cuBLAS status " + std::to_string((int)s));
}
void cusolver_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS)
    fail(PSG_E_CUDA, std::string(what) + ": cuSOLVER status " + std::to_string((int)s));
}

thread_local cudaStream_t g_pca_stream = nullptr;  // stream of the fit in flight
struct DevMem {
  void* p = nullptr;
  cudaStream_t s = g_pca_stream;
  explicit DevMem(size_t bytes) { PSG_CUDA(cudaMallocAsync(&p, bytes ? bytes : 1, s)); }
  ~DevMem() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* as() { return static_cast<T*>(p); }
};
}  // namespace

// ||W_i - theta_i V_i||_2 for the columns i of D x k matrices (one block per column).
__global__ void ritz_residual_kernel(const double* __restrict__ W, const double* __restrict__ V,
                                     const double* __restrict__ theta, int D, int c0,
                                     double* __restrict__ res) {
  __shared__ double red[256];
  const int col = c0 + blockIdx.x;
  const double th = theta[col];
  double acc = 0.0;
  for (int r = threadIdx.x; r < D; r += blockDim.x) {
    const double e = W[(int64_t)col * D + r] - th * V[(int64_t)col * D + r];
    acc += e * e;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) res[blockIdx.x] = sqrt(red[0]);
}

// Top-m eigenpairs of the symmetric D x D matrix `cov` by subspace iteration
// with Rayleigh-Ritz (k = block size > m): Q <- orth(C Q) (Householder QR),
// every few steps H = Q^T C Q, H = U diag(theta) U^T, Ritz vectors V = Q U and
// residuals ||C v - theta v||; converged when every top-m residual is
// <= 1e-11 * theta_max.  The error of the top-m subspace shrinks by
// lambda_{k+1} / lambda_m per step (cfg3 w = 32 windows: 0.03 at k = 96).
// On success writes the eigenvalues ascending into evals[0, m) and the
// eigenvectors into the first m columns of cov (ascending) and returns m;
// returns 0 (cov untouched) if it does not converge.
int subspace_top_eigen(psg_ctx* ctx, cublasHandle_t cb, cusolverDnHandle_t cs, double* cov, int D,
                       int m, double* evals, bool verbose) {
  const int k = std::min(D, std::max(3 * m, m + 48));
  if (3 * k > D || D < 1024) return 0;  // small problems: the direct solver is faster
  cudaStream_t st = ctx->stream;
  const double one = 1.0, zero = 0.0;
  DevMem Q(sizeof(double) * (size_t)D * k), Z(sizeof(double) * (size_t)D * k);
  DevMem V(sizeof(double) * (size_t)D * k), Wm(sizeof(double) * (size_t)D * k);
  DevMem H(sizeof(double) * (size_t)k * k), theta(sizeof(double) * k), tau(sizeof(double) * k);
  DevMem res(sizeof(double) * k), info(sizeof(int));
  int lw_qr = 0, lw_or = 0, lw_ev = 0;
  cusolver_check(cusolverDnDgeqrf_bufferSize(cs, D, k, Z.as<double>(), D, &lw_qr), "geqrf_bs");
  cusolver_check(cusolverDnDorgqr_bufferSize(cs, D, k, k, Z.as<double>(), D, tau.as<double>(), &lw_or),
                 "orgqr_bs");
  cusolver_check(cusolverDnDsyevd_bufferSize(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k,
                                             H.as<double>(), k, theta.as<double>(), &lw_ev),
                 "syevd_bs");
  DevMem work(sizeof(double) * (size_t)std::max(lw_qr, std::max(lw_or, lw_ev)));
  const int lwork = std::max(lw_qr, std::max(lw_or, lw_ev));
  // A <- orthonormal basis of span(A) by CholeskyQR2 (two passes of G = A^T A,
  // G = R^T R, A <- A R^-1: GEMM-shaped, no host round trip).  cond(C Q) is
  // bounded by lambda_1 / lambda_k, far inside CholeskyQR2's range; a failed
  // factorisation (info != 0, checked at the Rayleigh-Ritz points) makes the
  // caller fall back to the direct solver.
  DevMem G(sizeof(double) * (size_t)k * k), pinfo(sizeof(int));
  PSG_CUDA(cudaMemsetAsync(pinfo.p, 0, sizeof(int), st));
  int lw_po = 0;
  cusolver_check(cusolverDnDpotrf_bufferSize(cs, CUBLAS_FILL_MODE_UPPER, k, G.as<double>(), k,
                                             &lw_po), "potrf_bs");
  DevMem pwork(sizeof(double) * (size_t)std::max(lw_po, 1));
  auto orth = [&](double* A) {
    for (int pass = 0; pass < 2; ++pass) {
      cublas_check(cublasDsyrk(cb, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, k, D, &one, A, D, &zero,
                               G.as<double>(), k), "dsyrk G");
      cusolver_check(cusolverDnDpotrf(cs, CUBLAS_FILL_MODE_UPPER, k, G.as<double>(), k,
                                      pwork.as<double>(), lw_po, pinfo.as<int>()), "potrf");
      cublas_check(cublasDtrsm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                               CUBLAS_DIAG_NON_UNIT, D, k, &one, G.as<double>(), k, A, D), "dtrsm");
    }
  };
  auto householder = [&](double* A) {  // start block only
    cusolver_check(cusolverDnDgeqrf(cs, D, k, A, D, tau.as<double>(), work.as<double>(), lwork,
                                    info.as<int>()), "geqrf");
    cusolver_check(cusolverDnDorgqr(cs, D, k, k, A, D, tau.as<double>(), work.as<double>(), lwork,
                                    info.as<int>()), "orgqr");
  };
  {  // deterministic start block
    std::vector<double> h((size_t)D * k);
    uint64_t s = 0x5DEECE66Dull;
    for (auto& v : h) {
      s += 0x9E3779B97F4A7C15ull;
      uint64_t z = s;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      v = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
    PSG_CUDA(cudaMemcpyAsync(Q.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st));
  }
  householder(Q.as<double>());
  const int max_it = 200;
  double prev_worst = 0.0;
  int prev_it = 0;
  std::vector<double> hth(k), hres(m);
  for (int it = 1; it <= max_it; ++it) {
    cublas_check(cublasDsymm(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, D, k, &one, cov, D,
                             Q.as<double>(), D, &zero, Z.as<double>(), D), "dsymm");
    ctx->launches++;
    if ((it >= 6 && it % 3 == 0) || it == max_it) {
      // Rayleigh-Ritz on span(Q): H = Q^T (C Q)
      cublas_check(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, D, &one, Q.as<double>(), D,
                               Z.as<double>(), D, &zero, H.as<double>(), k), "dgemm H");
      cusolver_check(cusolverDnDsyevd(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, k,
                                      H.as<double>(), k, theta.as<double>(), work.as<double>(),
                                      lwork, info.as<int>()), "syevd H");
      cublas_check(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, D, k, k, &one, Q.as<double>(), D,
                               H.as<double>(), k, &zero, V.as<double>(), D), "dgemm V");
      cublas_check(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, D, k, k, &one, Z.as<double>(), D,
                               H.as<double>(), k, &zero, Wm.as<double>(), D), "dgemm W");
      ritz_residual_kernel<<<m, 256, 0, st>>>(Wm.as<double>(), V.as<double>(), theta.as<double>(),
                                              D, k - m, res.as<double>());
      PSG_LAUNCHED(ctx);
      PSG_CUDA(cudaMemcpyAsync(hth.data(), theta.p, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
      PSG_CUDA(cudaMemcpyAsync(hres.data(), res.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
      int hpinfo = 0;
      PSG_CUDA(cudaMemcpyAsync(&hpinfo, pinfo.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      PSG_CUDA(cudaStreamSynchronize(st));
      if (hpinfo != 0) return 0;  // CholeskyQR broke down: direct solver
      double worst = 0.0;
      for (double r : hres) worst = std::max(worst, r);
      const double scale = std::max(std::fabs(hth[k - 1]), 1e-300);
      if (verbose)
        fprintf(stderr, "[persyn]     subspace it %d (k=%d): max residual %.3e x theta_max\n", it,
                k, worst / scale);
      // too slow a contraction (flat spectrum around the m-th eigenvalue):
      // hand over to the direct solver instead of iterating to the cap
      if (prev_worst > 0.0 && worst > 1e-11 * scale) {
        const double rate = std::pow(worst / prev_worst, 1.0 / (it - prev_it));
        const double need = rate < 1.0 ? std::log(1e-11 * scale / worst) / std::log(rate) : 1e30;
        if (it + need > max_it) {
          if (verbose)
            fprintf(stderr, "[persyn]     subspace: %.3f per step, %.0f more steps: direct solver\n",
                    rate, need);
          return 0;
        }
      }
      prev_worst = worst;
      prev_it = it;
      if (worst <= 1e-11 * scale) {
        PSG_CUDA(cudaMemcpyAsync(evals, theta.as<double>() + (k - m), sizeof(double) * m,
                                 cudaMemcpyDeviceToDevice, st));
        PSG_CUDA(cudaMemcpyAsync(cov, V.as<double>() + (size_t)(k - m) * D,
                                 sizeof(double) * (size_t)m * D, cudaMemcpyDeviceToDevice, st));
        PSG_CUDA(cudaStreamSynchronize(st));
        return m;
      }
      PSG_CUDA(cudaMemcpyAsync(Z.p, Wm.p, sizeof(double) * (size_t)D * k, cudaMemcpyDeviceToDevice,
                               st));  // C V: continue from the Ritz basis
    }
    orth(Z.as<double>());
    std::swap(Q.p, Z.p);
  }
  return 0;
}

void create_solver_handles(psg_ctx* ctx) {
  if (!ctx->cublas) {
    cublasHandle_t h;
    cublas_check(cublasCreate(&h), "cublasCreate");
    ctx->cublas = h;
  }
  if (!ctx->cusolver) {
    cusolverDnHandle_t h;
    cusolver_check(cusolverDnCreate(&h), "cusolverDnCreate");
    ctx->cusolver = h;
  }
}

void fit_pca_device(psg_ctx* ctx, Index& ix, const psg_index_cfg& cfg) {
  const int64_t n = ix.N;
  const int D = ix.D;
  if (n < 2) fail(PSG_E_DOMAIN, "PCA needs at least 2 points");
  if (cfg.d_fixed <= 0 && !(cfg.variance_target > 0.0 && cfg.variance_target <= 1.0))
    fail(PSG_E_DOMAIN, "variance target must be in (0, 1]");

  create_solver_handles(ctx);
  g_pca_stream = ctx->stream;
  auto cb = static_cast<cublasHandle_t>(ctx->cublas);
  auto cs = static_cast<cusolverDnHandle_t>(ctx->cusolver);
  cublas_check(cublasSetStream(cb, ctx->stream), "cublasSetStream");
  cusolver_check(cusolverDnSetStream(cs, ctx->stream), "cusolverDnSetStream");

  const bool verbose = ctx->knobs.verbose;
  auto tick = [&](const char* what) {
    if (!verbose) return;
    static thread_local std::chrono::steady_clock::time_point t0;
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    const auto t1 = std::chrono::steady_clock::now();
    if (what) fprintf(stderr, "[persyn]   pca %s %.2f ms\n", what,
                      std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  tick(nullptr);
  DevMem mean(sizeof(double) * D);
  DevMem cov(sizeof(double) * (size_t)D * D);
  const bool structured = !ix.from_vectors && (size_t)ix.eh * ix.w * sizeof(double) <= 200 * 1024;
  if (structured) {
    // window database: box sums of product images (kernels_pca.cu), no N x D matrix
    launch_window_mean(ctx, ix.ex_mirror, ix.ew, ix.C, ix.w, ix.nxe, n, mean.as<double>());
    launch_window_cov(ctx, ix.ex_mirror, ix.ew, ix.eh, ix.C, ix.w, mean.as<double>(),
                      cov.as<double>());
  } else {
    DevMem Xc(sizeof(double) * (size_t)n * D);
    if (ix.from_vectors) {
      launch_vector_mean(ctx, ix.vectors, n, D, mean.as<double>());
      launch_center_vectors(ctx, ix.vectors, n, D, mean.as<double>(), Xc.as<double>());
    } else {
      launch_window_mean(ctx, ix.ex_mirror, ix.ew, ix.C, ix.w, ix.nxe, n, mean.as<double>());
      launch_center_windows(ctx, ix.ex_mirror, ix.ew, ix.C, ix.w, ix.nxe, n, mean.as<double>(),
                            Xc.as<double>());
    }
    // Row-major Xc[n][D] is column-major D x n: cov = Xc^T Xc = A A^T.
    const double alpha = 1.0 / (double)(n - 1), beta = 0.0;
    cublas_check(cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, D, (int)n, &alpha,
                             Xc.as<double>(), D, &beta, cov.as<double>(), D),
                 "cublasDsyrk");
    ctx->launches++;
  }
  tick(structured ? "window covariance (box sums)" : "mean + centre + dsyrk");

  // number of top eigenpairs needed (0 = full spectrum)
  int m_top = 0;
  if (cfg.d_fixed > 0) m_top = std::min(cfg.d_fixed, D);
  else if (cfg.d_cap > 0) m_top = std::min(cfg.d_cap, D);
  const bool subset = m_top > 0 && m_top < D;
  std::vector<double> diag;
  if (subset) {  // trace before the solver overwrites the matrix
    std::vector<double> h((size_t)D);
    PSG_CUDA(cudaMemcpy2DAsync(h.data(), sizeof(double), cov.as<double>(),
                               sizeof(double) * (D + 1), sizeof(double), D,
                               cudaMemcpyDeviceToHost, ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    diag = std::move(h);
  }
  DevMem evals(sizeof(double) * D);
  DevMem info(sizeof(int));
  PSG_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), ctx->stream));
  int lwork = 0, meig = D;
  bool iterative = false;
  if (subset && !ctx->knobs.eig_direct) {
    meig = subspace_top_eigen(ctx, cb, cs, cov.as<double>(), D, m_top, evals.as<double>(), verbose);
    iterative = meig > 0;
  }
  if (iterative) {
    // top m_top eigenpairs already in evals / cov (ascending)
  } else if (subset) {
    const int il = D - m_top + 1, iu = D;
    cusolver_check(cusolverDnDsyevdx_bufferSize(cs, CUSOLVER_EIG_MODE_VECTOR,
                                                CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, D,
                                                cov.as<double>(), D, 0.0, 0.0, il, iu, &meig,
                                                evals.as<double>(), &lwork),
                   "syevdx_bufferSize");
    DevMem work(sizeof(double) * (size_t)lwork);
    cusolver_check(cusolverDnDsyevdx(cs, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                     CUBLAS_FILL_MODE_LOWER, D, cov.as<double>(), D, 0.0, 0.0, il,
                                     iu, &meig, evals.as<double>(), work.as<double>(), lwork,
                                     info.as<int>()),
                   "cusolverDnDsyevdx");
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  } else {
    cusolver_check(cusolverDnDsyevd_bufferSize(cs, CUSOLVER_EIG_MODE_VECTOR,
                                               CUBLAS_FILL_MODE_LOWER, D, cov.as<double>(), D,
                                               evals.as<double>(), &lwork),
                   "syevd_bufferSize");
    DevMem work(sizeof(double) * (size_t)lwork);
    cusolver_check(cusolverDnDsyevd(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D,
                                    cov.as<double>(), D, evals.as<double>(), work.as<double>(),
                                    lwork, info.as<int>()),
                   "cusolverDnDsyevd");
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ctx->launches++;

  tick(iterative ? "subspace iteration" : subset ? "syevdx" : "syevd");
  const int ne = subset ? meig : D;  // eigenpairs computed, ascending in cov's first columns
  std::vector<double> h_eval(ne), h_mean(D);
  int h_info = 0;
  PSG_CUDA(cudaMemcpyAsync(h_eval.data(), evals.p, sizeof(double) * ne, cudaMemcpyDeviceToHost,
                           ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(h_mean.data(), mean.p, sizeof(double) * D, cudaMemcpyDeviceToHost,
                           ctx->stream));
  PSG_CUDA(cudaMemcpyAsync(&h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  PSG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h_info != 0) fail(PSG_E_DOMAIN, "eigendecomposition did not converge");

  // descending, clamped (pca.cpp:72-77)
  std::vector<double> var(D, 0.0);
  double total = 0.0;
  for (int k = 0; k < ne; ++k) var[k] = std::max(0.0, h_eval[ne - 1 - k]);
  if (subset) {
    for (int j = 0; j < D; ++j) total += diag[j];
    total = std::max(total, 0.0);
  } else {
    for (int k = 0; k < D; ++k) total += var[k];
  }
  int retained = 0;
  if (cfg.d_fixed > 0) {
    retained = std::min(cfg.d_fixed, D);
  } else if (total > 0.0) {
    double cum = 0.0;
    for (retained = 1; retained <= ne; ++retained) {
      cum += var[retained - 1];
      if (cum >= cfg.variance_target * total) break;
    }
    retained = std::min(retained, ne);
    if (cfg.d_cap > 0) retained = std::min(retained, cfg.d_cap);
  }
  if (retained > kMaxDP) fail(PSG_E_DOMAIN, "retained PCA dimension > 128 is not supported");

  // eigenvector of the k-th largest: column (ne-1-k) of the column-major result
  std::vector<double> basis((size_t)retained * D);
  if (retained > 0) {
    std::vector<double> cols((size_t)retained * D);
    PSG_CUDA(cudaMemcpyAsync(cols.data(), cov.as<double>() + (size_t)(ne - retained) * D,
                             sizeof(double) * (size_t)retained * D, cudaMemcpyDeviceToHost,
                             ctx->stream));
    PSG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < retained; ++k) {
      const double* comp = cols.data() + (size_t)(retained - 1 - k) * D;
      int arg = 0;
      double best = -1.0;
      for (int j = 0; j < D; ++j)
        if (std::fabs(comp[j]) > best) {
          best = std::fabs(comp[j]);
          arg = j;
        }
      const double sgn = comp[arg] < 0.0 ? -1.0 : 1.0;
      for (int j = 0; j < D; ++j) basis[(size_t)k * D + j] = sgn * comp[j];
    }
  }
  tick("selection + basis download");
  ix.h_mean = std::move(h_mean);
  ix.h_basis = std::move(basis);
  ix.h_var = std::move(var);
  ix.d = retained;
}

}  // namespace psg
