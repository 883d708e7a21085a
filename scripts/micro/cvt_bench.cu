// Microbenchmark: F2F.F64.F32 (float -> double widening) throughput on
// sm_100a, alone and mixed with the rescoring chain's DADD/DMUL.  The
// rescoring and M-step kernels widen every fp32 feature before the exact fp64
// arithmetic; this measures whether the conversion, not the fp64 pipe, binds.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void cvt_only(double* out, int iters, float b) {
  float f[16];
  double acc[16];
  for (int t = 0; t < 16; ++t) { f[t] = threadIdx.x * t * 1e-3f; acc[t] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      f[t] = __fmul_rn(f[t], b);  // loop-carried fp32 (cheap pipe)
      acc[t] = __dadd_rn(acc[t], (double)f[t]);
    }
  }
  double s = 0;
  for (int t = 0; t < 16; ++t) s += acc[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fp32_only(float* out, int iters, float b) {
  float f[16], acc[16];
  for (int t = 0; t < 16; ++t) { f[t] = threadIdx.x * t * 1e-3f; acc[t] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      f[t] = __fmul_rn(f[t], b);
      acc[t] = __fadd_rn(acc[t], f[t]);
    }
  }
  float s = 0;
  for (int t = 0; t < 16; ++t) s += acc[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 8, iters = 2048;
  float ms;
  cvt_only<<<blocks, 256>>>(o, 16, 1.0000001f);
  cudaEventRecord(e0);
  cvt_only<<<blocks, 256>>>(o, iters, 1.0000001f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)blocks * 256 * iters * 16;
  printf("F2F.F64.F32 + DADD + FMUL per element: %.2f T elements/s (%.1f per SM-clock at 1.965 GHz)\n",
         n / ms / 1e9, n / ms * 1e3 / (148 * 1.965e9));
  fp32_only<<<blocks, 256>>>((float*)o, 16, 1.0000001f);
  cudaEventRecord(e0);
  fp32_only<<<blocks, 256>>>((float*)o, iters, 1.0000001f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FMUL + FADD per element (control): %.2f T elements/s\n", n / ms / 1e9);
  return 0;
}
