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

struct DevMem {
  void* p = nullptr;
  explicit DevMem(size_t bytes) { PSG_CUDA(cudaMalloc(&p, bytes ? bytes : 1)); }
  ~DevMem() { cudaFree(p); }
  template <class T>
  T* as() { return static_cast<T*>(p); }
};
}  // namespace

void fit_pca_device(psg_ctx* ctx, Index& ix, const psg_index_cfg& cfg) {
  const int64_t n = ix.N;
  const int D = ix.D;
  if (n < 2) fail(PSG_E_DOMAIN, "PCA needs at least 2 points");
  if (cfg.d_fixed <= 0 && !(cfg.variance_target > 0.0 && cfg.variance_target <= 1.0))
    fail(PSG_E_DOMAIN, "variance target must be in (0, 1]");

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
  auto cb = static_cast<cublasHandle_t>(ctx->cublas);
  auto cs = static_cast<cusolverDnHandle_t>(ctx->cusolver);
  cublas_check(cublasSetStream(cb, ctx->stream), "cublasSetStream");
  cusolver_check(cusolverDnSetStream(cs, ctx->stream), "cusolverDnSetStream");

  const bool verbose = std::getenv("PERSYN_VERBOSE") != nullptr;
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
  int lwork = 0, meig = D;
  if (subset) {
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

  tick(subset ? "syevdx" : "syevd");
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
  if (retained > 64) fail(PSG_E_DOMAIN, "retained PCA dimension > 64 is not supported");

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
