// Fused small kernels of the spectral-norm block power iteration
// (dense.py:405-442: w = A v; est = sigma_1(qr(w).r); v = qr(A' w).q, b <= 32
// columns).  Round 1 spent ~143 us of every 0.49 ms iteration in serial
// latency kernels between the two DMMA sweeps (a split-K finalize, a Gram
// GEMM and its finalize, a 41 us lambda_max, a 71 us cooperative
// CholeskyQR).  Here each sweep's split-K partials are consumed by ONE
// ordinary launch that also forms the Gram of the rows it finalises and, in
// its last CTA to finish (atomic ticket), reduces the per-CTA Grams in CTA
// order (deterministic) and either
//   * (w) takes lambda_max(w'w) -- est^2 -- with a one-warp register
//     Householder tridiagonalisation and a 256-way Sturm multisection, or
//   * (z) factors the Gram for the first CholeskyQR step (one-warp register
//     Cholesky and triangular inverse, lane = column).
// The remaining CholeskyQR steps are `apply` launches: rows <- rows R^-1 in
// place (plus the transposed copy the next A v sweep reads), the Gram of the
// new rows, and the next factor in the last CTA.  The step rule is
// cholqr_multi's (plain factor while it exists with kappa_F <= 1e6, else the
// Fukaya shift; two consecutive plain steps end it), decided on the device;
// the host launches a fixed number of apply kernels, which return at once
// when the state says done.  No grid barrier, no cooperative launch.
#pragma once
#include "common.cuh"

namespace sn {

constexpr int THREADS = 256;
constexpr int NW = THREADS / 32;
constexpr int B = 32;  // register tile (b <= 32, padded)

struct QrState {
  double rinv[B * B];     // R^-1 of the pending step, [k][c] (upper)
  double kappa;
  int plain;              // consecutive unshifted steps
  int finish;             // the pending apply is the last one
  int done;               // Q complete (apply launches return at once)
  int status;             // 0 ok, 2 non-finite, 3 not converged within the launched steps
  int steps;
  unsigned ticket;        // last-CTA election (reset by the last CTA)
};

struct WState {
  unsigned ticket;
};

// Cholesky G + shift I = R'R of the b x b matrix in smem (ld ldg), padded to
// 32 x 32 with the identity, lane c holding column c; then R^-1 (upper).
// Returns false when a pivot is not positive/finite.  nr2 / ni2: |R|_F^2,
// |R^-1|_F^2 (warp-uniform).
__device__ bool warp_chol_inv(const double* Gs, int ldg, int b, double shift, double (&x)[B], double& nr2,
                              double& ni2) {
  const int lane = threadIdx.x & 31;
  double a[B];
#pragma unroll
  for (int i = 0; i < B; ++i) {
    double g = (i < b && lane < b) ? Gs[i * ldg + lane] : (i == lane ? 1.0 : 0.0);
    if (i == lane && lane < b) g += shift;
    a[i] = g;
  }
  bool bad = false;
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const double djj = __shfl_sync(0xffffffffu, a[j], j);
    bad |= !(djj > 0.0) || !isfinite(djj);
    const double rjj = sqrt(djj);
    const double rj = (lane < j) ? 0.0 : ((lane == j) ? rjj : a[j] / rjj);
    a[j] = rj;  // R[j][lane]
#pragma unroll
    for (int i = j + 1; i < B; ++i) {
      const double rji = __shfl_sync(0xffffffffu, rj, i);
      if (lane >= i) a[i] = fma(-rji, rj, a[i]);
    }
  }
  // column `lane` of R^-1 by back substitution (row k of R from lanes >= k)
#pragma unroll
  for (int k = B - 1; k >= 0; --k) {
    const double rkk = __shfl_sync(0xffffffffu, a[k], k);
    double s = 0.0;
#pragma unroll
    for (int i = k + 1; i < B; ++i) {
      const double rki = __shfl_sync(0xffffffffu, a[k], i);
      if (i <= lane) s = fma(rki, x[i], s);
    }
    x[k] = (k == lane) ? 1.0 / rkk : ((k < lane) ? -s / rkk : 0.0);
  }
  double pr = 0.0, pi = 0.0;
  if (lane < b) {
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (k <= lane) {
        pr = fma(a[k], a[k], pr);
        pi = fma(x[k], x[k], pi);
      }
  }
  nr2 = warp_sum(pr);
  ni2 = warp_sum(pi);
  return !__any_sync(0xffffffffu, bad);
}

// One CholeskyQR step decision for the Gram G (smem, b x b, ld ldg), by
// warp 0 of the last CTA: cholqr_multi's rule (corutv_b200.cu) -- plain
// factor if it exists with kappa_F <= kappa_max, else G + s I with s =
// shift_coeff * tr(G); R^-1 -> st->rinv, state updated.
__device__ void factor_step(const double* Gs, int ldg, int b, double shift_coeff, double kappa_max,
                            QrState* st) {
  const int lane = threadIdx.x & 31;
  double tr = 0.0;
  for (int i = lane; i < b; i += 32) tr += Gs[i * ldg + i];
  tr = warp_sum(tr);
  double x[B];
  int shifted = 0, status = 0;
  double kappa = 1.0;
  if (!(tr > 0.0) || !isfinite(tr)) {
    // exactly zero input: R = I, Q = X, done (cholqr_multi's status 1); or garbage
#pragma unroll
    for (int k = 0; k < B; ++k) x[k] = (k == lane) ? 1.0 : 0.0;
    status = isfinite(tr) ? 1 : 2;
  } else {
    double nr2, ni2;
    bool ok = warp_chol_inv(Gs, ldg, b, 0.0, x, nr2, ni2);
    kappa = sqrt(nr2) * sqrt(ni2);
    if (!ok || !(kappa <= kappa_max)) {
      shifted = 1;
      ok = warp_chol_inv(Gs, ldg, b, shift_coeff * tr, x, nr2, ni2);
      kappa = sqrt(nr2) * sqrt(ni2);
      if (!ok) status = 2;
    }
  }
#pragma unroll
  for (int k = 0; k < B; ++k) st->rinv[k * B + lane] = x[k];
  if (lane == 0) {
    st->kappa = kappa;
    st->steps += 1;
    if (status == 2) {
      st->status = 2;
      st->done = 1;
    } else {
      st->plain = shifted ? 0 : st->plain + 1;
      st->finish = (status == 1 || st->plain == 2) ? 1 : 0;
    }
  }
}

// lambda_max of the symmetric b x b matrix in smem (ld ldg): warp 0 reduces
// it to tridiagonal form in registers (lane = column; dsytd2 / dlarfg
// conventions, zero-padded to 32), then all THREADS evaluate Sturm counts
// at THREADS shifts per round (8 bits) from the Gershgorin bracket.
__device__ double sym_lmax(const double* Gs, int ldg, int b, double* d, double* e, double* xs, int* cs) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {
    double a[B];
#pragma unroll
    for (int i = 0; i < B; ++i) a[i] = (i < b && lane < b) ? Gs[i * ldg + lane] : 0.0;
#pragma unroll
    for (int k = 0; k + 2 < B; ++k) {
      // x = A[k+1:, k] (column k = lane k's registers), broadcast
      double xv[B];
      double sigma = 0.0;
#pragma unroll
      for (int i = k + 1; i < B; ++i) {
        xv[i] = __shfl_sync(0xffffffffu, a[i], k);
        if (i > k + 1) sigma = fma(xv[i], xv[i], sigma);
      }
      const double akk = __shfl_sync(0xffffffffu, a[k], k);
      const double alpha = xv[k + 1];
      if (sigma == 0.0) {
        if (lane == 0) {
          d[k] = akk;
          e[k] = alpha;
        }
        continue;
      }
      const double nrm = sqrt(alpha * alpha + sigma);
      const double beta = (alpha >= 0.0) ? -nrm : nrm;
      const double tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      double v[B];
#pragma unroll
      for (int i = 0; i < B; ++i) v[i] = (i == k + 1) ? 1.0 : ((i > k + 1) ? xv[i] * scal : 0.0);
      // p_c = tau sum_i A[i][c] v_i (column c = row c: symmetric), w = p - (tau/2)(p'v) v
      double pc = 0.0;
#pragma unroll
      for (int i = k + 1; i < B; ++i) pc = fma(a[i], v[i], pc);
      pc *= tau;
      const double vc = (lane == k + 1) ? 1.0 : ((lane > k + 1) ? a[k] * scal : 0.0);
      const double kk = -0.5 * tau * warp_sum((lane > k) ? pc * vc : 0.0);
      const double wc = fma(kk, vc, pc);
#pragma unroll
      for (int i = k + 1; i < B; ++i) {
        const double wi = __shfl_sync(0xffffffffu, wc, i);
        if (lane > k) a[i] -= v[i] * wc + wi * vc;
      }
      if (lane == 0) {
        d[k] = akk;
        e[k] = beta;
      }
    }
    const double d30 = __shfl_sync(0xffffffffu, a[B - 2], B - 2);
    const double e30 = __shfl_sync(0xffffffffu, a[B - 1], B - 2);
    const double d31 = __shfl_sync(0xffffffffu, a[B - 1], B - 1);
    if (lane == 0) {
      d[B - 2] = d30;
      e[B - 2] = e30;
      d[B - 1] = d31;
    }
  }
  __syncthreads();
  double lo = 1e308, hi = -1e308, emax2 = 0.0;
  for (int i = 0; i < B; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < B ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    if (i + 1 < B) emax2 = fmax(emax2, e[i] * e[i]);
  }
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2);
  const double span = fmax(fabs(lo), fabs(hi));
  lo -= 4.0 * 2.220446049250313e-16 * span + pivmin;
  hi += 4.0 * 2.220446049250313e-16 * span + pivmin;
  for (int step = 0; step < 64; ++step) {
    const double x = lo + (hi - lo) * ((double)(tid + 1) / (double)(THREADS + 1));
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0.0);
#pragma unroll
    for (int i = 1; i < B; ++i) {
      q = (d[i] - x) - e[i - 1] * e[i - 1] / q;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += (q < 0.0);
    }
    xs[tid] = x;
    const unsigned above = __ballot_sync(0xffffffffu, cnt == B);
    if (lane == 0) cs[warp] = above ? warp * 32 + __ffs(above) - 1 : THREADS;
    __syncthreads();
    int f = THREADS;
    for (int w = 0; w < NW; ++w) f = min(f, cs[w]);
    double nlo = lo, nhi = hi;
    if (f < THREADS) {
      nhi = xs[f];
      if (f > 0) nlo = xs[f - 1];
    } else {
      nlo = xs[THREADS - 1];
    }
    __syncthreads();
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
    if (hi - lo <= 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi))) break;
  }
  return 0.5 * (lo + hi);
}

// Gram of the CTA's rows: lane i of every warp accumulates G[i][.] over the
// warp's rows (row values broadcast by shuffles), then the warps' partials
// are summed in warp order into part[blockIdx.x] (b x b, ld b).
struct GramAcc {
  double g[B];
  __device__ void zero() {
#pragma unroll
    for (int j = 0; j < B; ++j) g[j] = 0.0;
  }
  __device__ void add(double xi) {  // xi = row value of column `lane`
#pragma unroll
    for (int j = 0; j < B; ++j) g[j] = fma(xi, __shfl_sync(0xffffffffu, xi, j), g[j]);
  }
};

// the warps' Grams summed in warp order (deterministic) in smem gs (B x B+1),
// then stored as this CTA's partial part[blockIdx.x] (b x b, ld b)
__device__ void cta_gram_store(const GramAcc& acc, int b, double* gs, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int w = 0; w < NW; ++w) {
    if (warp == w && lane < b)
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (j < b) gs[lane * (B + 1) + j] = (w == 0 ? 0.0 : gs[lane * (B + 1) + j]) + acc.g[j];
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += THREADS) part[(int64_t)blockIdx.x * b * b + e] = gs[(e / b) * (B + 1) + e % b];
}

// last CTA to arrive (atomic ticket): sums the gridDim.x partials in CTA
// order into Gs (smem, ld b).  Returns false in every other CTA.
__device__ bool last_cta_reduce(const double* part, int b, unsigned* ticket, double* Gs) {
  __shared__ int am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  const int bb = b * b;
  for (int e = threadIdx.x; e < bb; e += THREADS) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int c = 0;
    const int nc = gridDim.x;
    for (; c + 4 <= nc; c += 4) {
      s0 += part[(int64_t)c * bb + e];
      s1 += part[(int64_t)(c + 1) * bb + e];
      s2 += part[(int64_t)(c + 2) * bb + e];
      s3 += part[(int64_t)(c + 3) * bb + e];
    }
    for (; c < nc; ++c) s0 += part[(int64_t)c * bb + e];
    Gs[e] = (s0 + s1) + (s2 + s3);
  }
  if (threadIdx.x == 0) *ticket = 0;
  __syncthreads();
  return true;
}

struct Smem {
  double gs[B * (B + 1)];
  double G[B * B];
  double d[B], e[B];
  double xs[THREADS];
  int cs[NW];
};

// rows [r0, r1) of this CTA (contiguous chunks)
__device__ __forceinline__ void cta_rows(int64_t rows, int64_t* r0, int64_t* r1) {
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  *r0 = min<int64_t>(rows, (int64_t)blockIdx.x * chunk);
  *r1 = min<int64_t>(rows, *r0 + chunk);
}

// MODE 0 (w = A v): finalize w from the split-K partials (ws, `splits`
// slices of stride sstride, ld ldw) into out (ld ldo), Gram, last CTA:
// lam[0] = lambda_max(w'w).
// MODE 1 (z = A' w): finalize z into out (the CholeskyQR buffer), Gram,
// last CTA: first factor step into st.
template <int MODE>
__global__ void __launch_bounds__(THREADS, 1)
    finalize_kernel(const double* __restrict__ ws, int splits, int64_t sstride, int64_t ldw, int64_t rows, int b,
                    double* __restrict__ out, int64_t ldo, double* __restrict__ part, unsigned* ticket,
                    double* lam, QrState* st, double shift_coeff, double kappa_max) {
  __shared__ Smem sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (MODE == 1 && blockIdx.x == 0 && threadIdx.x == 0) {
    // fresh CholeskyQR state (visible to the apply launches after this one)
    st->plain = 0;
    st->finish = 0;
    st->done = 0;
    st->status = 0;
    st->steps = 0;
  }
  int64_t r0, r1;
  cta_rows(rows, &r0, &r1);
  GramAcc acc;
  acc.zero();
  for (int64_t r = r0 + warp; r < r1; r += NW) {
    double v = 0.0;
    if (lane < b) {
      const double* src = ws + r * ldw + lane;
      int s = 0;
      for (; s + 4 <= splits; s += 4) {
        const double p0 = src[(int64_t)s * sstride], p1 = src[(int64_t)(s + 1) * sstride];
        const double p2 = src[(int64_t)(s + 2) * sstride], p3 = src[(int64_t)(s + 3) * sstride];
        v += p0;
        v += p1;
        v += p2;
        v += p3;
      }
      for (; s < splits; ++s) v += src[(int64_t)s * sstride];
      out[r * ldo + lane] = v;
    }
    acc.add(v);
  }
  cta_gram_store(acc, b, sm.gs, part);
  if (!last_cta_reduce(part, b, ticket, sm.G)) return;
  if (MODE == 0) {
    const double l = sym_lmax(sm.G, b, b, sm.d, sm.e, sm.xs, sm.cs);
    if (threadIdx.x == 0) lam[0] = l;
  } else {
    if (warp == 0) factor_step(sm.G, b, b, shift_coeff, kappa_max, st);
  }
}

// One CholeskyQR apply: x <- x R^-1 in place (rows x b, ld ldx) and the
// transposed copy xT (b x rows, ld ldxT); unless this was the last step,
// the Gram of the new rows and, in the last CTA, the next factor.
__global__ void __launch_bounds__(THREADS, 1)
    apply_kernel(double* __restrict__ x, int64_t ldx, double* __restrict__ xT, int64_t ldxT, int64_t rows, int b,
                 double* __restrict__ part, QrState* st, double shift_coeff, double kappa_max, int last_launch) {
  __shared__ Smem sm;
  __shared__ double Ri[B * (B + 1)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (*((volatile int*)&st->done)) return;  // uniform: written by an earlier launch
  const bool finish = *((volatile int*)&st->finish) != 0;
  for (int e = threadIdx.x; e < B * B; e += THREADS) Ri[(e / B) * (B + 1) + e % B] = st->rinv[e];
  __syncthreads();
  int64_t r0, r1;
  cta_rows(rows, &r0, &r1);
  GramAcc acc;
  acc.zero();
  for (int64_t r = r0 + warp; r < r1; r += NW) {
    const double xi = (lane < b) ? x[r * ldx + lane] : 0.0;
    double o = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const double xk = __shfl_sync(0xffffffffu, xi, k);
      if (k <= lane) o = fma(xk, Ri[k * (B + 1) + lane], o);
    }
    if (lane < b) {
      x[r * ldx + lane] = o;
      xT[(int64_t)lane * ldxT + r] = o;
    } else {
      o = 0.0;
    }
    if (!finish) acc.add(o);
  }
  if (finish) {
    // the last CTA to finish marks the state done: every CTA of this launch
    // has passed its `done` check by then
    __shared__ int am_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) am_last = (atomicAdd(&st->ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (am_last && threadIdx.x == 0) {
      st->ticket = 0;
      st->finish = 0;
      st->done = 1;
    }
    return;
  }
  cta_gram_store(acc, b, sm.gs, part);
  if (!last_cta_reduce(part, b, &st->ticket, sm.G)) return;
  if (warp == 0) {
    factor_step(sm.G, b, b, shift_coeff, kappa_max, st);
    // the launch budget is spent and another step would be needed
    if (lane == 0 && last_launch && !st->finish && st->status == 0) {
      st->status = 3;
      st->done = 1;
    }
  }
}

}  // namespace sn
