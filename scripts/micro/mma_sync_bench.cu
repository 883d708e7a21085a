// Microbenchmark: legacy warp-level mma.sync (HMMA) throughput on sm_100a,
// bf16 m16n8k16 with fp32 accumulate, 8 independent accumulators per warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kf(float* out, int iters) {  // fp32 FFMA reference
  float c[16];
  for (int t = 0; t < 16; ++t) c[t] = threadIdx.x * t;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int t = 0; t < 16; ++t) c[t] = fmaf(c[t], 1.0001f, 0.5f);
  float s = 0;
  for (int t = 0; t < 16; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    int iters = 4096;
    k<<<148 * 4, 32 * warps>>>(o, 16);
    cudaEventRecord(e0);
    k<<<148 * 4, 32 * warps>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * 4 * warps * iters * 8 * (16.0 * 8 * 16 * 2);
    printf("mma.sync bf16 m16n8k16: %d warps/CTA, 4 CTA/SM: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  {
    int iters = 8192;
    kf<<<148 * 4, 256>>>(o, 16);
    cudaEventRecord(e0);
    kf<<<148 * 4, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 148.0 * 4 * 256 * iters * 16 * 2;
    printf("fp32 FFMA: %.1f TFLOP/s\n", flops / ms / 1e9);
  }
  return 0;
}
