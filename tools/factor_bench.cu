// Isolated timing of the spectral norm's 24-column factor step
// (snorm.cuh sn::factor_step / cta_chol_aug) in one 256-thread CTA, repeated,
// so ncu's source view gets enough samples: cycles per call and per column.
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include "../paper_1906_04572_b200/csrc/snorm.cuh"

__global__ void __launch_bounds__(256, 1) factor_bench(const double* G0, int b, int reps, sn::QrState* st,
                                                      long long* cyc) {
  __shared__ sn::RowSmem sm;
  for (int e = threadIdx.x; e < sn::B * sn::B; e += 256) sm.u.f.G[e] = G0[e];
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) { st->plain = 0; st->steps = 0; st->finish = 0; st->status = 0; }
    __syncthreads();
    sn::factor_step(sm.u.f.G, sn::B, b, 1e-14, 1e6, st, sm.u.f.W, sm.red, sm.rowj, sm.piv);
    __syncthreads();
    // restore G (factor_step's W aliases nothing in G here)
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
  const int b = 24;
  double h[32 * 32] = {0};
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) h[i * 32 + j] = (i == j ? 30.0 : 0.0) + 1.0 / (1.0 + i + j);
  double* d; long long* c; sn::QrState* st;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&c, 8); cudaMalloc(&st, sizeof(sn::QrState));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemset(st, 0, sizeof(sn::QrState));
  long long cy = 0;
  for (int rep = 0; rep < 3; ++rep) {
    factor_bench<<<1, 256>>>(d, b, 200, st, c);
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  }
  static sn::QrState hs;
  cudaMemcpy(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost);
  unsigned long long ck = 0;
  for (int e = 0; e < 32 * 32; ++e) {
    unsigned long long u;
    memcpy(&u, &hs.rinv[e], 8);
    ck = ck * 1099511628211ull + u;
  }
  printf("factor_step b=%d: %lld cycles per call (%.0f per column), rinv checksum %016llx kappa %.17g, err %s\n", b, cy,
         cy / (double)b, ck, hs.kappa, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
