// Dependent-chain latency of FP64 ops on this GPU (clock64 around 1024
// dependent ops in one thread): DFMA, DADD, sqrt, division, shfl of a double.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0) {
  double x = x0, y = 1.0000001;
  long long t0 = clock64();
#pragma unroll 32
  for (int i = 0; i < 1024; ++i) x = fma(x, y, 1e-300);
  long long t1 = clock64();
#pragma unroll 32
  for (int i = 0; i < 1024; ++i) x = x + 1e-300;
  long long t2 = clock64();
#pragma unroll 32
  for (int i = 0; i < 256; ++i) x = sqrt(x) + 1.0;
  long long t3 = clock64();
#pragma unroll 32
  for (int i = 0; i < 256; ++i) x = 1.0 / x + 1.0;
  long long t4 = clock64();
#pragma unroll 32
  for (int i = 0; i < 1024; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-300;
  long long t5 = clock64();
  float f = (float)x;
#pragma unroll 32
  for (int i = 0; i < 1024; ++i) f = fmaf(f, 1.0000001f, 1e-30f);
  long long t6 = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double* o; long long* c; long long h[6];
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 6 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 32>>>(o, c, 1.5);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  }
  printf("cycles per dependent op: DFMA %.1f  DADD %.1f  sqrt+add %.1f  rcp-div+add %.1f  shfl(double)+add %.1f  FFMA %.1f\n",
         h[0] / 1024.0, h[1] / 1024.0, h[2] / 256.0, h[3] / 256.0, h[4] / 1024.0, h[5] / 1024.0);
  return 0;
}
