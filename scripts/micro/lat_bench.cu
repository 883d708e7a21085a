// Microbenchmark: dependent-chain latency (cycles per op) of DADD, DMUL, FADD
// and F2F.F64.F32 on one warp of sm_100a (clock64 around 4096 chained ops).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double b, float fb) {
  double a = threadIdx.x * 1e-3;
  float f = threadIdx.x * 1e-3f;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) a = __dmul_rn(a, b);
  long long t2 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) f = __fadd_rn(f, fb);
  long long t3 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) a = (double)(float)a + b;  // F2F.F32.F64 + F2F.F64.F32 + DADD
  long long t4 = clock64();
  out[threadIdx.x] = a + f;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
}
int main() {
  double* o; long long* c; long long h[4];
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 4 * 8);
  k<<<1, 32>>>(o, c, 1e-9, 1e-9f);
  k<<<1, 32>>>(o, c, 1e-9, 1e-9f);
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("cycles/op: dadd %.2f dmul %.2f fadd %.2f (f2f+f2f+dadd) %.2f\n", h[0] / 4096.0, h[1] / 4096.0,
         h[2] / 4096.0, h[3] / 4096.0);
  return 0;
}
