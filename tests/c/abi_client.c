/* A plain C client of the drop-in boundary (include/corutv_b200.h): what a
 * non-Python host binds.  No Python, no torch: device memory from the CUDA
 * runtime, the decomposition through the C-ABI.
 *
 *   abi_client                 -> {"version": N}            (no GPU needed)
 *   abi_client IN OUT          -> decompose IN, write OUT, print a JSON line
 *
 * IN : int64 m, n, ell, q, variant; then A (m x n) and Omega (n x ell),
 *      row-major float64.
 * OUT: int64 passes; U (m x ell), T (ell x ell), V (n x ell) float64; perm
 *      (ell) int64.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "corutv_b200.h"

#define CHECK_CUDA(x)                                                        \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) {                                                 \
      fprintf(stderr, "cuda: %s (%s)\n", cudaGetErrorString(e_), #x);        \
      return 3;                                                              \
    }                                                                        \
  } while (0)

static int read_all(FILE* f, void* p, size_t bytes) { return fread(p, 1, bytes, f) == bytes ? 0 : -1; }

int main(int argc, char** argv) {
  if (argc == 1) {
    printf("{\"version\": %d}\n", corutv_version());
    return 0;
  }
  if (argc != 3) {
    fprintf(stderr, "usage: abi_client [IN OUT]\n");
    return 1;
  }
  FILE* fi = fopen(argv[1], "rb");
  if (!fi) return 1;
  int64_t hdr[5];
  if (read_all(fi, hdr, sizeof hdr)) return 1;
  const int64_t m = hdr[0], n = hdr[1], ell = hdr[2], q = hdr[3], variant = hdr[4];
  double* a = (double*)malloc(sizeof(double) * m * n);
  double* om = (double*)malloc(sizeof(double) * n * ell);
  if (read_all(fi, a, sizeof(double) * m * n) || read_all(fi, om, sizeof(double) * n * ell)) return 1;
  fclose(fi);

  corutv_handle* h = NULL;
  int rc = corutv_create(0, NULL, &h);
  if (rc) {
    fprintf(stderr, "corutv_create: %d\n", rc);
    return 2;
  }
  double *dA, *dO, *dU, *dT, *dV;
  int64_t* dP;
  CHECK_CUDA(cudaMalloc((void**)&dA, sizeof(double) * m * n));
  CHECK_CUDA(cudaMalloc((void**)&dO, sizeof(double) * n * ell));
  CHECK_CUDA(cudaMalloc((void**)&dU, sizeof(double) * m * ell));
  CHECK_CUDA(cudaMalloc((void**)&dT, sizeof(double) * ell * ell));
  CHECK_CUDA(cudaMalloc((void**)&dV, sizeof(double) * n * ell));
  CHECK_CUDA(cudaMalloc((void**)&dP, sizeof(int64_t) * ell));
  CHECK_CUDA(cudaMemcpy(dA, a, sizeof(double) * m * n, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(dO, om, sizeof(double) * n * ell, cudaMemcpyHostToDevice));

  int64_t passes = 0;
  rc = corutv_decompose(h, dA, m, n, n, (int)ell, (int)q, (int)variant, dO, dU, dT, dV, dP, &passes);
  if (rc) {
    printf("{\"rc\": %d, \"error\": \"%s\"}\n", rc, corutv_last_error(h));
    return 0;
  }
  double err = -1.0;
  rc = corutv_lowrank_error(h, dA, m, n, n, dU, dT, dV, (int)ell, &err);
  if (rc) {
    printf("{\"rc\": %d, \"error\": \"%s\"}\n", rc, corutv_last_error(h));
    return 0;
  }
  CHECK_CUDA(cudaDeviceSynchronize());

  double* u = (double*)malloc(sizeof(double) * m * ell);
  double* t = (double*)malloc(sizeof(double) * ell * ell);
  double* v = (double*)malloc(sizeof(double) * n * ell);
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * ell);
  CHECK_CUDA(cudaMemcpy(u, dU, sizeof(double) * m * ell, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(t, dT, sizeof(double) * ell * ell, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(v, dV, sizeof(double) * n * ell, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(perm, dP, sizeof(int64_t) * ell, cudaMemcpyDeviceToHost));
  FILE* fo = fopen(argv[2], "wb");
  if (!fo) return 1;
  fwrite(&passes, sizeof passes, 1, fo);
  fwrite(u, sizeof(double), (size_t)(m * ell), fo);
  fwrite(t, sizeof(double), (size_t)(ell * ell), fo);
  fwrite(v, sizeof(double), (size_t)(n * ell), fo);
  fwrite(perm, sizeof(int64_t), (size_t)ell, fo);
  fclose(fo);
  printf("{\"rc\": 0, \"passes\": %lld, \"err\": %.17g}\n", (long long)passes, err);
  cudaFree(dA);
  cudaFree(dO);
  cudaFree(dU);
  cudaFree(dT);
  cudaFree(dV);
  cudaFree(dP);
  corutv_destroy(h);
  free(a);
  free(om);
  free(u);
  free(t);
  free(v);
  free(perm);
  return 0;
}
