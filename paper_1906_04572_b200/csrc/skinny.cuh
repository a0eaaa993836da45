// Tall-skinny adaptive CholeskyQR in ONE cooperative launch, for the block
// power iteration of spectral_norm (dense.py:405-442: v = orth(A' w) every
// iteration, b <= 24 columns).  The multi-launch path (split-K Gram GEMM,
// finalize, Cholesky kernel, X R^-1 GEMM, a host decision per step) spends
// most of its time in launch and synchronisation latency at this size; here
// every step is three grid phases:
//
//   1. each CTA forms the Gram of its contiguous row chunk (FP64 FMA; the
//      chunk stays in shared memory for the whole launch);
//   2. the partials are summed entry-wise in CTA order (one warp per entry,
//      fixed shuffle tree: deterministic), then CTA 0 factors the Gram with
//      the one-CTA kernel's logic (small::chol_factor_block: the plain factor
//      is kept when kappa_F <= kappa_max, else the shifted one);
//   3. every CTA multiplies its rows by R^-1 and applies the step rule of
//      cholqr_multi (stop after two consecutive plain steps or a zero input)
//      -- the decision is read by all CTAs from the same global record, so it
//      is uniform without a host round trip.
//
// C4 spectral norm (10000^2, 352 iterations): 193.5 -> 179.1 ms.
//
// The final Q is written to `q` (rows x b, ld ldq) and transposed to `qT`
// (b x rows, ld ldqT); status[0] = 0 ok, 2 non-finite, 3 no convergence;
// status[1] = steps.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "small.cuh"

namespace skinny {

namespace cg = cooperative_groups;
constexpr int THREADS = 256;
constexpr int BMAX = 32;

__global__ void __launch_bounds__(THREADS) cholqr_kernel(const double* x0, int64_t rows, int b,
                                                         int64_t ldx, double shift_coeff, double kappa_max,
                                                         int max_steps, double* part, double* gsum,
                                                         double* rinvT, small::CholInfo* info, double* q,
                                                         int64_t ldq, double* qT, int64_t ldqT, int* status) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double xs[];  // this CTA's rows, chunk x b
  __shared__ double W[2 * BMAX * BMAX];
  __shared__ double red[small::NWARPS];
  __shared__ double R[BMAX * BMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bb = b * b;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int nr = (int)(r0 + chunk < rows ? chunk : (rows > r0 ? rows - r0 : 0));
  const double* cur = x0;
  int plain = 0, st = 3, steps = 0;
  // the CTA's rows stay in shared memory across steps (x R^-1 is row-local)
  if ((b & 1) == 0 && (ldx & 1) == 0) {
    // rows as double2 (b and ld even: 16-byte aligned)
    const int h2 = b >> 1;
    const double2* src = reinterpret_cast<const double2*>(cur);
    double2* dst = reinterpret_cast<double2*>(xs);
    for (int e = threadIdx.x; e < nr * h2; e += blockDim.x) dst[e] = src[(r0 + e / h2) * (ldx >> 1) + e % h2];
  } else {
    for (int e = threadIdx.x; e < nr * b; e += blockDim.x) xs[e] = cur[(r0 + e / b) * ldx + e % b];
  }
  __syncthreads();
  for (int step = 0; step < max_steps; ++step) {
    // 1. partial Gram of the CTA's rows (4 independent partial sums)
    for (int e = threadIdx.x; e < bb; e += blockDim.x) {
      const int i = e / b, j = e % b;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int r = 0;
      for (; r + 4 <= nr; r += 4) {
        a0 += xs[r * b + i] * xs[r * b + j];
        a1 += xs[(r + 1) * b + i] * xs[(r + 1) * b + j];
        a2 += xs[(r + 2) * b + i] * xs[(r + 2) * b + j];
        a3 += xs[(r + 3) * b + i] * xs[(r + 3) * b + j];
      }
      for (; r < nr; ++r) a0 += xs[r * b + i] * xs[r * b + j];
      part[(int64_t)blockIdx.x * bb + e] = (a0 + a1) + (a2 + a3);
    }
    grid.sync();
    // 2a. entry-wise reduction over the CTAs in CTA order, one warp per entry
    //     (lanes take strided CTAs, fixed-order shuffle tree: deterministic)
    for (int e = blockIdx.x * (blockDim.x >> 5) + warp; e < bb; e += gridDim.x * (blockDim.x >> 5)) {
      double acc = 0.0;
      for (int c = lane; c < (int)gridDim.x; c += 32) acc += part[(int64_t)c * bb + e];
      acc = warp_sum(acc);
      if (lane == 0) gsum[e] = acc;
    }
    grid.sync();
    // 2b. CTA 0 factors
    if (blockIdx.x == 0) small::chol_factor_block(gsum, b, b, shift_coeff, 1, kappa_max, rinvT, b, info, W, red);
    grid.sync();
    // 3. rows * R^-1 (in shared memory), step rule
    const int cst = *((volatile int*)&info->status);
    const int shifted = *((volatile int*)&info->shifted);
    steps = step + 1;
    if (cst == 2) {
      st = 2;
      break;
    }
    // R[k * b + c] = R^-1[k][c]  (rinvT[c][k] transposed: lanes read rows)
    for (int e = threadIdx.x; e < bb; e += blockDim.x) R[(e % b) * b + e / b] = rinvT[e];
    __syncthreads();
    // x_r <- x_r R^-1: a warp takes 4 rows at a time, lane c forms column c
    // (x_r[k] broadcast, k <= c); results stay in registers until the warp's
    // 4 rows are done, so the update is in place
    for (int rb = warp * 4; rb < nr; rb += (blockDim.x >> 5) * 4) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const int c = lane;
      for (int k = 0; k < b; ++k) {
        const double rk = (c < b && k <= c) ? R[k * b + c] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (rb + u < nr) acc[u] += xs[(rb + u) * b + k] * rk;
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (rb + u < nr && c < b) xs[(rb + u) * b + c] = acc[u];
      __syncwarp();
    }
    __syncthreads();
    plain = shifted ? 0 : plain + 1;
    const bool done = (cst == 1) || (plain == 2);
    if (done) {
      st = 0;
      break;
    }
  }
  if (st != 2) {
    for (int e = threadIdx.x; e < nr * b; e += blockDim.x) {
      const int64_t r = r0 + e / b;
      const int c = e % b;
      const double v = xs[e];
      q[r * ldq + c] = v;
      qT[(int64_t)c * ldqT + r] = v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    status[0] = st;
    status[1] = steps;
  }
}

}  // namespace skinny
