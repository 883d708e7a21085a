// Microbenchmark: fp32 FFMA vs packed FFMA2 (f32x2) throughput on sm_100a —
// the measured denominator of the search kernel's fp32 roofline.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ffma(float* out, int iters, float b) {
  float acc[16];
  for (int t = 0; t < 16; ++t) acc[t] = threadIdx.x * t * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = __fmaf_rn(acc[t], b, 1e-7f);
  }
  float s = 0;
  for (int t = 0; t < 16; ++t) s += acc[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma2(float* out, int iters, float b) {
  float2 acc[16];
  for (int t = 0; t < 16; ++t) acc[t] = make_float2(threadIdx.x * t * 1e-3f, t * 1e-4f);
  const float2 bb = make_float2(b, b), cc = make_float2(1e-7f, 1e-7f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = __ffma2_rn(acc[t], bb, cc);
  }
  float s = 0;
  for (int t = 0; t < 16; ++t) s += acc[t].x + acc[t].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 8, iters = 4096;
  float ms;
  ffma<<<blocks, 256>>>(o, 16, 0.9999999f);
  cudaEventRecord(e0);
  ffma<<<blocks, 256>>>(o, iters, 0.9999999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * blocks * 256 * iters * 16;
  printf("FFMA : %.1f TFLOP/s\n", fl / ms / 1e9);
  ffma2<<<blocks, 256>>>(o, 16, 0.9999999f);
  cudaEventRecord(e0);
  ffma2<<<blocks, 256>>>(o, iters, 0.9999999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FFMA2: %.1f TFLOP/s\n", 2 * fl / ms / 1e9);
  return 0;
}
