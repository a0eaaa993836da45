// Bandwidth-bound helper kernels: layout changes, split-K finalisation,
// deterministic reductions, gathers.
#pragma once
#include "common.cuh"

namespace aux {

// dst[c][r] = src[r][c]; src rows x cols (ld lds) -> dst cols x rows (ld ldd).
__global__ void transpose_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                 int64_t lds, double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][i];
  }
}

// dst (rows x cols, ld ldd) = src (ld lds)
__global__ void copy2d_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                              int64_t lds, double* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx % cols;
    dst[r * ldd + c] = src[r * lds + c];
  }
}

// C = sum_s ws[s] in fixed order (deterministic split-K); optional C^T.
__global__ void splitk_finalize_kernel(const double* __restrict__ ws, int splits,
                                       int64_t split_stride, int64_t M, int64_t N, int64_t ldw,
                                       double* __restrict__ C, int64_t ldc, double* __restrict__ Ct,
                                       int64_t ldct) {
  const int64_t total = M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / N, j = idx % N;
    // fixed summation order; loads batched so they are in flight together
    const double* src = ws + i * ldw + j;
    double s = 0.0;
    int k = 0;
    for (; k + 16 <= splits; k += 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = src[(int64_t)(k + u) * split_stride];
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
    for (; k < splits; ++k) s += src[(int64_t)k * split_stride];
    if (C) C[i * ldc + j] = s;
    if (Ct) Ct[j * ldct + i] = s;
  }
}

// V[i][k] = Q[i][perm[k]]  (sketch.py:206)
__global__ void gather_cols_kernel(const double* __restrict__ Q, int64_t rows, int ell,
                                   int64_t ldq, const int* __restrict__ perm,
                                   double* __restrict__ V, int64_t ldv) {
  const int64_t total = rows * ell;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / ell;
    const int k = idx % ell;
    V[i * ldv + k] = Q[i * ldq + perm[k]];
  }
}

// per-block partial sums of squares (stage 1 of a deterministic reduction)
__global__ void sumsq_partial_kernel(const double* __restrict__ A, int64_t rows, int64_t cols,
                                     int64_t lda, double* __restrict__ part, long long* __restrict__ bad) {
  __shared__ double red[32];
  __shared__ int redb[32];
  double s = 0.0;
  int nb = 0;  // non-finite entries seen (as_matrix's check, dense.py:48-49)
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx % cols;
    const double v = A[r * lda + c];
    s = fma(v, v, s);
    nb += isfinite(v) ? 0 : 1;
  }
  s = warp_sum(s);
  nb = __reduce_add_sync(0xffffffffu, (unsigned)nb);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = s;
    redb[threadIdx.x >> 5] = nb;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    s = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
    nb = (threadIdx.x < blockDim.x / 32) ? redb[threadIdx.x] : 0;
    s = warp_sum(s);
    nb = __reduce_add_sync(0xffffffffu, (unsigned)nb);
    if (threadIdx.x == 0) {
      part[blockIdx.x] = s;
      if (bad) bad[blockIdx.x] = nb;
    }
  }
}

// shrink (rpca.py:99-104): out = sign(x) max(|x| - delta, 0), counting
// non-finite inputs into bad[blockIdx.x] (grid-stride, fixed partition)
__global__ void shrink_kernel(const double* __restrict__ X, int64_t rows, int64_t cols, int64_t ldx,
                              double delta, double* out, int64_t ldo, long long* __restrict__ bad) {
  __shared__ int redb[32];
  int nb = 0;
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx % cols;
    const double x = X[r * ldx + c];
    nb += isfinite(x) ? 0 : 1;
    const double sg = (x > 0.0) ? 1.0 : ((x < 0.0) ? -1.0 : x);  // np.sign
    out[r * ldo + c] = sg * fmax(fabs(x) - delta, 0.0);
  }
  nb = __reduce_add_sync(0xffffffffu, (unsigned)nb);
  if ((threadIdx.x & 31) == 0) redb[threadIdx.x >> 5] = nb;
  __syncthreads();
  if (threadIdx.x < 32) {
    nb = (threadIdx.x < blockDim.x / 32) ? redb[threadIdx.x] : 0;
    nb = __reduce_add_sync(0xffffffffu, (unsigned)nb);
    if (threadIdx.x == 0) bad[blockIdx.x] = nb;
  }
}

// stage 2: one block sums n partials (doubles) and counts (int64) in a fixed
// order: out[0] = sum, out[1] = (double) count.
__global__ void finalize_sums_kernel(const double* __restrict__ part, const long long* cnt,
                                     int n, double* out) {
  __shared__ double red[32];
  __shared__ long long redc[32];
  double s = 0.0;
  long long c = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s += part[i];
    if (cnt) c += cnt[i];
  }
  s = warp_sum(s);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = s;
    redc[threadIdx.x >> 5] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    long long tc = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      t += red[w];
      tc += redc[w];
    }
    out[0] = t;
    out[1] = (double)tc;
  }
}

// spectral_norm start block (dense.py:421-424) written transposed:
// vt[j][i] = 1/sqrt(count_j) if i % b == j.
__global__ void snorm_init_kernel(double* vt, int b, int64_t n, int64_t ldv) {
  const int64_t total = (int64_t)b * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = idx / n;
    const int64_t i = idx % n;
    const int64_t count = (n - j + b - 1) / b;
    vt[j * ldv + i] = (i % b == j) ? 1.0 / sqrt((double)count) : 0.0;
  }
}

// rows of the left factor scaled for the pseudoinverse (dense.py:390-402):
// us[k][j] = ut[k][j] / sig_k when sig_k > max(len, nv) sig_0 1e-12, else 0
// (the one-CTA Jacobi kernel's (W / s) / s, with ut = W / s).
__global__ void pinv_scale_kernel(const double* __restrict__ ut, int64_t ldut, const double* __restrict__ sig,
                                  int nv, int len, double* __restrict__ us, int64_t ldus) {
  const double s0 = sig[0];
  const double cut = (double)max(len, nv) * s0 * 1e-12;
  const int64_t total = (int64_t)nv * len;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / len), j = (int)(idx % len);
    const double sk = sig[k];
    us[k * ldus + j] = (s0 > 0.0 && sk > cut) ? ut[k * ldut + j] / sk : 0.0;
  }
}

// C (M x N) = op(A) op(B) for small operands (SIMT).  ta/tb: use transpose.
__global__ void small_matmul_kernel(const double* __restrict__ A, int64_t lda, int ta,
                                    const double* __restrict__ B, int64_t ldb, int tb, int M,
                                    int N, int K, double* __restrict__ C, int64_t ldc) {
  const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
  if (i >= M || j >= N) return;
  double s = 0.0;
  for (int k = 0; k < K; ++k) {
    const double a = ta ? A[k * lda + i] : A[i * lda + k];
    const double b = tb ? B[j * ldb + k] : B[k * ldb + j];
    s = fma(a, b, s);
  }
  C[i * ldc + j] = s;
}

__global__ void fill2d_kernel(double* p, int64_t rows, int64_t cols, int64_t ld, double v) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    p[(idx / cols) * ld + idx % cols] = v;
}

__global__ void flag_to_double_kernel(const int* f, double* d) {
  if (threadIdx.x == 0) d[0] = (double)f[0];
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x)
    p[idx] = v;
}

// Singular value threshold of sorted sigma (rpca.py:150-156):
// kept = max(sigma - delta, 0), T = diag(kept) (k x k, ld ldt), *count +=
// #(kept > 0).  T feeds the fused ALM update as the core of U T V'.
__global__ void svt_kept_kernel(const double* sig, int k, double delta, double* kept, double* t, int64_t ldt,
                                int* count) {
  const int64_t total = (int64_t)k * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / k), j = (int)(idx % k);
    double v = 0.0;
    if (i == j) {
      v = fmax(sig[i] - delta, 0.0);
      kept[i] = v;
      if (v > 0.0) atomicAdd(count, 1);
    }
    t[i * ldt + j] = v;
  }
}

}  // namespace aux
