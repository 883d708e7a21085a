// Microbenchmark: fp64 DMUL + DADD (separate, no FMA: the exact projection's
// operation mix) throughput on sm_100a.  Both operations are loop-carried
// (an invariant product would be hoisted out of the loop by the compiler).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double b) {
  double acc[16], c[16];
  for (int t = 0; t < 16; ++t) { acc[t] = threadIdx.x * t; c[t] = 1.0 + t * 1e-3; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      c[t] = __dmul_rn(c[t], b);  // loop-carried: the multiply cannot be hoisted
      acc[t] = __dadd_rn(acc[t], c[t]);
    }
  }
  double s = 0;
  for (int t = 0; t < 16; ++t) s += acc[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocks : {148 * 2, 148 * 4, 148 * 8}) {
    int iters = 2048;
    k<<<blocks, 256>>>(o, 16, 1.0000001);
    cudaEventRecord(e0);
    k<<<blocks, 256>>>(o, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * 256 * iters * 16 * 2;
    printf("fp64 dmul+dadd: %d blocks x 256: %.2f T ops/s\n", blocks, ops / ms / 1e9);
  }
  return 0;
}
