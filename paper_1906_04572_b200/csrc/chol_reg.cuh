// Register-resident step of the adaptive shifted CholeskyQR (small cores,
// l <= 64): the same contract as small::chol_factor_kernel (R'R = G [+ s I],
// the plain factor kept when it exists with kappa_F <= kappa_max, else the
// Fukaya shift s = shift_coeff tr(G); rinvT[j][k] = R^-1[k][j]; CholInfo),
// which stands in for householder_qr (dense.py:132-149) on the sketches.
//
// The augmented [G + s I | I] (l x 2l) is held by columns: G threads own one
// column, thread (k, g) keeps rows g + G m in registers.  Right-looking
// row-oriented Cholesky with ONE barrier per column: at the end of step j-1
// the owners publish the updated row j (unscaled) to shared memory; step j
// reads the pivot d = W[j][j] and the row from there, scales on the fly
// (W[j][k] * (1 / sqrt(d))) and applies the rank-1
// update to the rows it owns.  The row buffer is double-buffered by parity.
#pragma once
#include "common.cuh"
#include "small.cuh"

namespace creg {

template <int LM, int G>
__global__ void __launch_bounds__(2 * LM * G, 1)
    chol_reg_kernel(const double* __restrict__ Gm, int l, int64_t ldg, double shift_coeff, int allow_plain,
                    double kappa_max, double* __restrict__ rinvT, int64_t ldr, small::CholInfo* info,
                    int* qd) {
  constexpr int NC = 2 * LM, NT = NC * G, RPT = LM / G, NW = NT / 32;
  static_assert(32 % G == 0 && LM % G == 0, "shape");
  __shared__ double rowj[2][NC];
  __shared__ double red[2][NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col = tid / G, g = tid % G;
  const bool left = col < LM;
  const int k = left ? col : col - LM;  // column index within its half
  const bool live = k < l;
  // qd (optional, speculative schedule): {plain, done, status, steps} of
  // cholqr_multi's rule kept on the device.  Once done, the step is an exact
  // no-op: R^-1 = I (X I = X bit for bit in the following DMMA GEMM).
  if (qd && *((volatile int*)&qd[1])) {
    if (!left && live) {
#pragma unroll
      for (int m = 0; m < RPT; ++m) {
        const int i = g + G * m;
        if (i < l) rinvT[(int64_t)i * ldr + k] = (k == i) ? 1.0 : 0.0;
      }
    }
    return;
  }
  // trace (same value in every thread): one diagonal load per thread, then
  // the per-warp sums added in warp order
  double tr = warp_sum(tid < l ? Gm[(int64_t)tid * ldg + tid] : 0.0);
  if (lane == 0) red[0][warp] = tr;
  __syncthreads();
  tr = 0.0;
  for (int q = 0; q < NW; ++q) tr += red[0][q];
  __syncthreads();
  int shifted = allow_plain ? 0 : 1;
  int status = 0;
  double kappa = 0.0;
  double w[RPT];
  if (!(tr > 0.0) || !isfinite(tr)) {
    // exactly zero sketch (or garbage): R = I, Q = X
#pragma unroll
    for (int m = 0; m < RPT; ++m) w[m] = (!left && live && g + G * m == k) ? 1.0 : 0.0;
    status = isfinite(tr) ? 1 : 2;
    kappa = 1.0;
  } else {
    for (;;) {
      const double s = shifted ? shift_coeff * tr : 0.0;
#pragma unroll
      for (int m = 0; m < RPT; ++m) {
        const int i = g + G * m;
        double v = 0.0;
        if (live && i < l) {
          if (left) v = (k >= i) ? Gm[(int64_t)i * ldg + k] + (i == k ? s : 0.0) : 0.0;
          else v = (i == k) ? 1.0 : 0.0;
        }
        w[m] = v;
      }
      // publish row 0
      if (g == 0) rowj[0][col] = w[0];
      __syncthreads();
      bool fail = false;
      for (int j = 0; j < l; ++j) {
        const int cb = j & 1;
        const double d = rowj[cb][j];
        if (!(d > 0.0) || !isfinite(d)) {
          fail = true;  // uniform
          break;
        }
        const double r = sqrt(d), inv = 1.0 / r;
        // this column's entry of the scaled row j
        const double own = rowj[cb][col];
        const bool in_row = left ? (k > j && live) : (k <= j && live);
        const double bj = in_row ? own * inv : 0.0;
        const int jo = j % G, jm = j / G;
        if (g == jo) {
#pragma unroll
          for (int m = 0; m < RPT; ++m)
            if (m == jm) w[m] = (left && k == j) ? r : (in_row ? bj : w[m]);
        }
        // rank-1 update of the rows i > j (left: i <= k only)
#pragma unroll
        for (int m = 0; m < RPT; ++m) {
          const int i = g + G * m;
          if (i > j && i < l && in_row && (!left || i <= k)) {
            const double a = rowj[cb][i] * inv;
            w[m] = fma(-a, bj, w[m]);
          }
        }
        // publish row j + 1 (the owners of that row)
        if (j + 1 < l && g == (j + 1) % G) {
          const int m1 = (j + 1) / G;
          double v = 0.0;
#pragma unroll
          for (int m = 0; m < RPT; ++m)
            if (m == m1) v = w[m];
          rowj[cb ^ 1][col] = v;
        }
        __syncthreads();
      }
      if (fail) {
        __syncthreads();
        if (!shifted) {
          shifted = 1;
          continue;
        }
        status = 2;
        break;
      }
      // kappa_F = |R|_F |R^-1|_F (upper of the left half, lower of the right)
      double pr = 0.0, pi = 0.0;
#pragma unroll
      for (int m = 0; m < RPT; ++m) {
        const int i = g + G * m;
        if (!live || i >= l) continue;
        if (left && k >= i) pr = fma(w[m], w[m], pr);
        if (!left && k <= i) pi = fma(w[m], w[m], pi);
      }
      pr = warp_sum(pr);
      pi = warp_sum(pi);
      if (lane == 0) {
        red[0][warp] = pr;
        red[1][warp] = pi;
      }
      __syncthreads();
      double nr = 0.0, ni = 0.0;
      for (int q = 0; q < NW; ++q) {
        nr += red[0][q];
        ni += red[1][q];
      }
      __syncthreads();
      kappa = sqrt(nr) * sqrt(ni);
      if (!shifted && !(kappa <= kappa_max)) {
        shifted = 1;
        continue;
      }
      break;
    }
  }
  // rinvT = right half (lower): rinvT[i][k] = W[i][l + k] for k <= i
  if (!left && live) {
#pragma unroll
    for (int m = 0; m < RPT; ++m) {
      const int i = g + G * m;
      if (i < l) rinvT[(int64_t)i * ldr + k] = (k <= i) ? w[m] : 0.0;
    }
  }
  if (tid == 0) {
    info->shifted = shifted;
    info->status = status;
    info->kappa = kappa;
    info->trace = tr;
    if (qd) {
      const int plain = shifted ? 0 : qd[0] + 1;
      qd[0] = plain;
      qd[3] += 1;
      if (status == 2) qd[2] = 2;
      if (status != 0 || plain == 2) qd[1] = 1;
    }
  }
}

}  // namespace creg
