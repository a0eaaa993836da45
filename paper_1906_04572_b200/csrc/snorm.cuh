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
  double rtot[B * B];     // deferred mode: the product of every step's R^-1 so far (x_raw rtot = Q)
  double kappa;
  int plain;              // consecutive unshifted steps
  int finish;             // the pending apply is the last one
  int done;               // Q complete (apply launches return at once)
  int status;             // 0 ok, 2 non-finite, 3 not converged within the launched steps
  int steps;
  unsigned ticket;        // last-CTA election of a finishing apply (reset by it)
  unsigned tickets[16];   // two-level Gram reduction: [0] final, [1 + g] group g
  // %globaltimer stamps of the last launch (apply [0..3], finalize<1>
  // [4..7]): start, slowest CTA's rows done, reduction done, factor done
  unsigned long long prof[8];
  unsigned long long fprof[8];  // factor_step: entry, trace, attempt 1, attempt 2, R^-1 stored, end; shifted
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct WState {
  unsigned tickets[16];
};

constexpr int GS = 16;  // CTAs per first-level reduction group

// The serial 32 x 32 algorithms below run in ONE warp of the last CTA, once
// per launch: they keep the matrix in shared memory and use rolled loops, so
// the code stays small (fully unrolled register versions measured ~100 us a
// launch, dominated by instruction fetch of straight-line code run once).
constexpr int LDW = B + 1;

// CTA-wide Cholesky of the augmented [G + shift I | I] (32 x 64, identity-
// padded past b): the row operations that turn the left half into R (R'R =
// G + shift I) turn the right half into R^-T, so no separate triangular
// inverse (small.cuh chol_aug_unblocked).  Register-blocked: thread t owns
// row t/8, columns 8 (t%8) .. +7; per column j the pivot's owner publishes
// W[j][j], row j's owners scale and publish row j, every row below takes
// its rank-1 update -- two barriers per column.  Returns false (uniform) on
// a non-positive or non-finite pivot; nr2 / ni2 = |R|_F^2, |R^-1|_F^2 of the
// b x b block; on return the owners' registers are written to W (smem,
// 32 x LDA).
constexpr int LDA = 2 * B + 1;
static_assert(THREADS == 256, "cta_chol_aug: 32 rows x 8 threads");

__device__ bool cta_chol_aug(const double* Gs, int ldg, int b, double shift, double* W, double* red,
                             double* rowj, double* piv, double& nr2, double& ni2) {
  const int tid = threadIdx.x;
  const int i = tid >> 3, cb = (tid & 7) * 8;
  double w[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = cb + q;
    double g;
    if (c < B) {
      g = (i < b && c < b) ? Gs[i * ldg + c] : (i == c ? 1.0 : 0.0);
      if (i == c && i < b) g += shift;
    } else {
      g = (c - B == i) ? 1.0 : 0.0;
    }
    w[q] = g;
  }
  bool bad = false;
  // the padding (rows / columns b..31) is the identity and stays so: the
  // elimination stops after column b - 1 (b = 24 saves a quarter of the
  // serial chain)
  for (int j = 0; j < b; ++j) {
    if (i == j && (j >> 3) == (tid & 7)) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (cb + q == j) *piv = w[q];
    }
    __syncthreads();
    const double d = *piv;
    bad |= !(d > 0.0) || !isfinite(d);
    if (i == j) {
      // one reciprocal square root on the step's latency chain (as the
      // cluster Cholesky, chol_cluster.cuh) instead of a sqrt and a division
      const double ri = rsqrt(d), r = d * ri;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = cb + q;
        if (c == j) w[q] = r;
        else if (c > j) w[q] *= ri;
        rowj[c] = w[q];
      }
    }
    __syncthreads();
    if (i > j) {
      const double a = rowj[i];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (cb + q > j) w[q] = fma(-a, rowj[cb + q], w[q]);
    }
  }
  double pr = 0.0, pi = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = cb + q;
    W[i * LDA + c] = w[q];
    if (i < b && c < b && c >= i) pr = fma(w[q], w[q], pr);                   // R (upper)
    if (i < b && c >= B && c - B < b && c - B <= i) pi = fma(w[q], w[q], pi);  // R^-T (lower)
  }
  pr = warp_sum(pr);
  pi = warp_sum(pi);
  const int lane = tid & 31, warp = tid >> 5;
  if (lane == 0) {
    red[warp] = pr;
    red[NW + warp] = pi;
  }
  __syncthreads();
  nr2 = 0.0;
  ni2 = 0.0;
  for (int ww = 0; ww < NW; ++ww) {
    nr2 += red[ww];
    ni2 += red[NW + ww];
  }
  __syncthreads();
  return !bad;
}

// One CholeskyQR step decision for the Gram G (smem, b x b, ld ldg), by the
// whole last CTA: cholqr_multi's rule (corutv_b200.cu) -- plain factor if
// it exists with kappa_F <= kappa_max, else G + s I with s = shift_coeff *
// tr(G); R^-1 -> st->rinv ([k][c] upper), state updated.  W: smem 32 x LDA.
__device__ void factor_step(const double* Gs, int ldg, int b, double shift_coeff, double kappa_max,
                            QrState* st, double* W, double* red, double* rowj, double* piv) {
  const int tid = threadIdx.x;
  unsigned long long f0 = tid == 0 ? gtimer() : 0, f1 = 0, f2 = 0, f3 = 0;
  double tr = 0.0;
  for (int i = 0; i < b; ++i) tr += Gs[i * ldg + i];  // same order in every thread
  if (tid == 0) f1 = gtimer();
  int shifted = 0, status = 0;
  double kappa = 1.0;
  bool ident = false;
  if (!(tr > 0.0) || !isfinite(tr)) {
    // exactly zero input: R = I, Q = X, done (cholqr_multi's status 1); or garbage
    ident = true;
    status = isfinite(tr) ? 1 : 2;
  } else {
    double nr2, ni2;
    bool ok = cta_chol_aug(Gs, ldg, b, 0.0, W, red, rowj, piv, nr2, ni2);
    kappa = sqrt(nr2) * sqrt(ni2);
    if (tid == 0) f2 = gtimer();
    if (!ok || !(kappa <= kappa_max)) {
      shifted = 1;
      ok = cta_chol_aug(Gs, ldg, b, shift_coeff * tr, W, red, rowj, piv, nr2, ni2);
      kappa = sqrt(nr2) * sqrt(ni2);
      if (!ok) status = 2;
    }
    if (tid == 0) f3 = gtimer();
  }
  // R^-1[k][c] = (R^-T)[c][k]
  for (int e = tid; e < B * B; e += THREADS) {
    const int k = e / B, c = e % B;
    st->rinv[e] = ident ? (k == c ? 1.0 : 0.0) : ((k <= c) ? W[c * LDA + B + k] : 0.0);
  }
  if (tid == 0) {
    const unsigned long long f4 = gtimer();
    st->fprof[0] = f0;
    st->fprof[1] = f1;
    st->fprof[2] = f2;
    st->fprof[3] = f3;
    st->fprof[4] = f4;
    st->fprof[6] = shifted;
    st->kappa = kappa;
    st->steps = __ldcg(&st->steps) + 1;
    if (status == 2) {
      st->status = 2;
      st->done = 1;
    } else {
      const int plain = shifted ? 0 : __ldcg(&st->plain) + 1;
      st->plain = plain;
      st->finish = (status == 1 || plain == 2) ? 1 : 0;
    }
  }
}

// lambda_max of the symmetric b x b matrix in smem (ld ldg): warp 0 reduces
// it to tridiagonal form (dsytd2 / dlarfg conventions, zero-padded to 32,
// matrix in smem W, lane = column), then all THREADS evaluate Sturm counts
// at THREADS shifts per round (8 bits) from the Gershgorin bracket.
// vs, wsv: smem scratch vectors of B.
__device__ double sym_lmax(const double* Gs, int ldg, int b, double* d, double* e, double* xs, int* cs, double* W,
                           double* vs, double* wsv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {
    for (int i = 0; i < B; ++i) W[i * LDW + lane] = (i < b && lane < b) ? Gs[i * ldg + lane] : 0.0;
    __syncwarp();
    for (int k = 0; k + 2 < B; ++k) {
      const double xl = W[lane * LDW + k];  // A[lane][k]
      const double sigma = warp_sum(lane > k + 1 ? xl * xl : 0.0);
      const double akk = W[k * LDW + k];
      const double alpha = W[(k + 1) * LDW + k];
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
      const double vl = (lane == k + 1) ? 1.0 : ((lane > k + 1) ? xl * scal : 0.0);
      vs[lane] = vl;
      __syncwarp();
      // p = tau A22 v (column lane = row lane: symmetric), w = p - (tau/2)(p'v) v
      double pc = 0.0;
#pragma unroll 4
      for (int i = k + 1; i < B; ++i) pc = fma(W[i * LDW + lane], vs[i], pc);
      pc *= tau;
      const double kk = -0.5 * tau * warp_sum((lane > k) ? pc * vl : 0.0);
      const double wl = fma(kk, vl, pc);
      wsv[lane] = wl;
      __syncwarp();
      if (lane > k) {
#pragma unroll 4
        for (int i = k + 1; i < B; ++i) W[i * LDW + lane] -= vs[i] * wl + wsv[i] * vl;
      }
      __syncwarp();
      if (lane == 0) {
        d[k] = akk;
        e[k] = beta;
      }
    }
    if (lane == 0) {
      d[B - 2] = W[(B - 2) * LDW + B - 2];
      e[B - 2] = W[(B - 1) * LDW + B - 2];
      d[B - 1] = W[(B - 1) * LDW + B - 1];
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

// Two-level deterministic reduction of the gridDim.x per-CTA Gram partials
// (32 x 32, ld B, symmetric; only the upper triangle of the leading b x b
// block is summed): the last CTA of each group of GS (atomic ticket) sums
// its group in CTA order into part2[group]; the last group reducer sums the
// groups in order into Gs (smem, 32 x 32, both triangles, zero past b) and
// returns true; every other CTA returns false.  A thread's loads (all its
// entries x all CTAs of a group) are issued before any add.
constexpr int UMAX = (B * (B + 1) / 2 + THREADS - 1) / THREADS;  // upper entries per thread

__device__ __forceinline__ void upper_ij(int u, int b, int* i, int* j) {
  // u-th entry of the row-major upper triangle of a b x b matrix
  int r = 0, rem = u;
  while (rem >= b - r) {
    rem -= b - r;
    ++r;
  }
  *i = r;
  *j = r + rem;
}

// slot / count: this contributor's slot and the number of slots (the CTA
// index and grid size for the row kernels; the tile index and tile count
// for the fused sweep epilogue of gemm_snorm_kernel).
__device__ bool last_cta_reduce(const double* part, double* part2, int b, unsigned* tickets, double* Gs, int slot,
                                int count) {
  __shared__ int am_last;
  constexpr int bb = B * B;
  const int nu = b * (b + 1) / 2;
  const int group = slot / GS, ngroups = (count + GS - 1) / GS;
  const int gsize = min(GS, count - group * GS);
  int idx[UMAX];
#pragma unroll
  for (int q = 0; q < UMAX; ++q) {
    const int u = threadIdx.x + q * THREADS;
    int i = 0, j = 0;
    if (u < nu) upper_ij(u, b, &i, &j);
    idx[q] = (u < nu) ? i * B + j : -1;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = (atomicAdd(&tickets[1 + group], 1u) == (unsigned)gsize - 1);
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  {
    double v[UMAX][GS];
#pragma unroll
    for (int q = 0; q < UMAX; ++q)
#pragma unroll
      for (int c = 0; c < GS; ++c)
        v[q][c] = (idx[q] >= 0 && c < gsize) ? __ldcg(part + (int64_t)(group * GS + c) * bb + idx[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < UMAX; ++q) {
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < GS; ++c) sum += v[q][c];
      if (idx[q] >= 0) {
        if (ngroups == 1) Gs[idx[q]] = sum;
        else part2[(int64_t)group * bb + idx[q]] = sum;
      }
    }
  }
  if (threadIdx.x == 0) tickets[1 + group] = 0;
  if (ngroups > 1) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) am_last = (atomicAdd(&tickets[0], 1u) == (unsigned)ngroups - 1);
    __syncthreads();
    if (!am_last) return false;
    __threadfence();
    double v[UMAX][GS];
#pragma unroll
    for (int q = 0; q < UMAX; ++q)
#pragma unroll
      for (int g = 0; g < GS; ++g) v[q][g] = (idx[q] >= 0 && g < ngroups) ? __ldcg(part2 + (int64_t)g * bb + idx[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < UMAX; ++q) {
      double sum = 0.0;
#pragma unroll
      for (int g = 0; g < GS; ++g) sum += v[q][g];
      if (idx[q] >= 0) Gs[idx[q]] = sum;
    }
    if (threadIdx.x == 0) tickets[0] = 0;
  }
  __syncthreads();
  // mirror to the lower triangle, zero outside the b x b block
  for (int e = threadIdx.x; e < bb; e += THREADS) {
    const int i = e / B, j = e % B;
    if (i >= b || j >= b) Gs[e] = 0.0;
    else if (i > j) Gs[e] = Gs[j * B + i];
  }
  __syncthreads();
  return true;
}

// Deferred mode (spectral_norm_fused): the sweep after a CholeskyQR reads the
// un-normalised rows, and the product of all the steps' R^-1 is applied to
// its result instead (A (x R1^-1 R2^-1) = (A x) R1^-1 R2^-1), so the QR
// chain runs beside the sweep.  After a factor step stored st->rinv:
// rtot <- rinv (first step) or rtot rinv.  Called by the whole CTA that ran
// factor_step; tmp: smem B x B.
__device__ void compose_rtot(QrState* st, int first, double* tmp) {
  __syncthreads();  // st->rinv written by this CTA's threads
  for (int e = threadIdx.x; e < B * B; e += THREADS) tmp[e] = first ? 0.0 : st->rtot[e];
  __syncthreads();
  for (int e = threadIdx.x; e < B * B; e += THREADS) {
    const int k = e / B, c = e % B;
    double v;
    if (first) {
      v = st->rinv[e];
    } else {
      v = 0.0;
      for (int j = k; j <= c; ++j) v = fma(tmp[k * B + j], st->rinv[j * B + c], v);  // upper x upper
    }
    st->rtot[e] = v;
  }
  __syncthreads();
}

// last_cta_reduce's sums (groups of GS partials in slot order, then the
// groups in order: the same floating-point sequence) by ONE CTA, for a Gram
// whose partials a previous launch left in `part`.
__device__ void single_cta_reduce(const double* part, int b, int count, double* Gs) {
  constexpr int bb = B * B;
  const int nu = b * (b + 1) / 2;
  const int ngroups = (count + GS - 1) / GS;
  for (int u = threadIdx.x; u < nu; u += THREADS) {
    int i, j;
    upper_ij(u, b, &i, &j);
    const int idx = i * B + j;
    double total = 0.0;
    for (int g = 0; g < ngroups; ++g) {
      const int gsize = min(GS, count - g * GS);
      double v[GS];
#pragma unroll
      for (int c = 0; c < GS; ++c) v[c] = c < gsize ? __ldcg(part + (int64_t)(g * GS + c) * bb + idx) : 0.0;
      double sum = 0.0;
#pragma unroll
      for (int c = 0; c < GS; ++c) sum += v[c];
      if (ngroups == 1) total = sum;
      else total += sum;
    }
    Gs[idx] = total;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < bb; e += THREADS) {
    const int i = e / B, j = e % B;
    if (i >= b || j >= b) Gs[e] = 0.0;
    else if (i > j) Gs[e] = Gs[j * B + i];
  }
  __syncthreads();
}

// rows [r0, r1) of this CTA (contiguous chunks)
__device__ __forceinline__ void cta_rows(int64_t rows, int64_t* r0, int64_t* r1) {
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t a = (int64_t)blockIdx.x * chunk;
  *r0 = a < rows ? a : rows;
  *r1 = *r0 + chunk < rows ? *r0 + chunk : rows;
}

// The row kernels stage RCH rows at a time in shared memory (row stride
// LDX, columns b..31 and rows past the end zero): every global access is a
// coalesced sweep by the whole CTA, and the CTA's Gram partial is formed on
// the tensor pipe (DMMA.884: 16 8x8 blocks of the padded 32 x 32 Gram, two
// per warp, K = the chunk's rows).
constexpr int RCH = 96;
constexpr int LDX = 36;

struct RowSmem {
  union {
    double x[RCH * LDX];
    struct {
      double G[B * B];
      double W[B * LDA];
    } f;
  } u;
  double Ri[B * (B + 1)];
  double red[2 * NW];
  double rowj[2 * B];
  double piv[2];
};

__device__ __forceinline__ void gram_chunk(const double* x, int nr4, double (&acc)[2][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r8 = lane >> 2, c4 = lane & 3;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int q = 2 * warp + t, bi = q >> 2, bj = q & 3;
    for (int k0 = 0; k0 < nr4; k0 += 4) {
      const double a = x[(k0 + c4) * LDX + bi * 8 + r8];
      const double bb = x[(k0 + c4) * LDX + bj * 8 + r8];
      dmma884(acc[t][0], acc[t][1], a, bb);
    }
  }
}

__device__ __forceinline__ void gram_store(const double (&acc)[2][2], double* part, int idx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r8 = lane >> 2, c4 = lane & 3;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int q = 2 * warp + t, bi = q >> 2, bj = q & 3;
#pragma unroll
    for (int e = 0; e < 2; ++e) part[(int64_t)idx * B * B + (bi * 8 + r8) * B + bj * 8 + 2 * c4 + e] = acc[t][e];
  }
}

// x (RCH x 32 in smem, zero past nr / b) <- x R^-1 (Ri: smem [k][c] upper,
// ld B + 1) in place, on the tensor pipe: 12 x 4 output blocks of 8 x 8
// (K = 32), six per warp, held in registers until every warp has read x
__device__ __forceinline__ void apply_rinv_chunk(double* x, const double* Ri, int nr4) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r8 = lane >> 2, c4 = lane & 3;
  constexpr int NBLK = (RCH / 8) * (B / 8);       // 48
  constexpr int PERW = NBLK / NW;                 // 6
  double o[PERW][2];
#pragma unroll
  for (int t = 0; t < PERW; ++t) {
    const int q = warp * PERW + t, bi = q / (B / 8), bj = q % (B / 8);
    o[t][0] = o[t][1] = 0.0;
    if (bi * 8 < nr4) {
#pragma unroll
      for (int k0 = 0; k0 < B; k0 += 4) {
        const double a = x[(bi * 8 + r8) * LDX + k0 + c4];
        const double bb = Ri[(k0 + c4) * (B + 1) + bj * 8 + r8];
        dmma884(o[t][0], o[t][1], a, bb);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < PERW; ++t) {
    const int q = warp * PERW + t, bi = q / (B / 8), bj = q % (B / 8);
    if (bi * 8 < nr4) {
      x[(bi * 8 + r8) * LDX + bj * 8 + 2 * c4] = o[t][0];
      x[(bi * 8 + r8) * LDX + bj * 8 + 2 * c4 + 1] = o[t][1];
    }
  }
  __syncthreads();
}

// write the chunk to out (rows, ld ldo; coalesced along columns) and outT
// (b x rows, ld ldoT; coalesced along rows)
__device__ __forceinline__ void store_chunk(const double* x, int nr, int b, int64_t row0, double* out, int64_t ldo,
                                            double* outT, int64_t ldoT) {
  for (int e = threadIdx.x; e < nr * b; e += THREADS) {
    const int r = e / b, c = e % b;
    out[(row0 + r) * ldo + c] = x[r * LDX + c];
  }
  if (outT)
    for (int e = threadIdx.x; e < nr * b; e += THREADS) {
      const int c = e / nr, r = e % nr;
      outT[(int64_t)c * ldoT + row0 + r] = x[r * LDX + c];
    }
}

// MODE 0 (w = A v): finalize w from the split-K partials (ws, `splits`
// slices of stride sstride, ld ldw), times the pending R^-1 of the previous
// CholeskyQR (its last apply folded in: A (v' R^-1) = (A v') R^-1;
// identity on the first iteration), into out (+ outT); Gram; the last CTA
// writes the reduced Gram w'w (32 x 32, padded) to lam for lmax_kernel.
// MODE 1 (z = A' w): finalize z into out (the CholeskyQR buffer) + outT;
// Gram; the last CTA takes the first factor step into st.
// Rows [r0, r1) of a finalize: the split-K sum of the nr x b elements in
// fixed slice order (per thread 4 elements x up to 16 slices of loads in
// flight before any add), times the pending R^-1 for MODE 0, stored to out
// (+ outT), and their Gram accumulated into acc.  Ends with a barrier.
template <int MODE>
__device__ __forceinline__ void finalize_rows(RowSmem& sm, const double* __restrict__ ws, int splits, int64_t sstride,
                                              int64_t ldw, int64_t r0, int64_t r1, int b, double* __restrict__ out,
                                              int64_t ldo, double* __restrict__ outT, int64_t ldoT,
                                              double (&acc)[2][2]) {
  for (int64_t c0 = r0; c0 < r1; c0 += RCH) {
    const int nr = (int)min((int64_t)RCH, r1 - c0), nr4 = (nr + 3) & ~3;
    // zero the padding (rows nr..nr4, columns b..32)
    for (int e = threadIdx.x; e < nr4 * B; e += THREADS) {
      const int r = e / B, c = e % B;
      if (r >= nr || c >= b) sm.u.x[r * LDX + c] = 0.0;
    }
    const int ne = nr * b;
    for (int e0 = threadIdx.x; e0 < ne; e0 += 4 * THREADS) {
      int64_t off[4];
      int sidx[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = e0 + k * THREADS, r = e / b, c = e % b;
        off[k] = (c0 + r) * ldw + c;
        sidx[k] = (e < ne) ? r * LDX + c : -1;
      }
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      for (int s0 = 0; s0 < splits; s0 += 16) {
        double p[16][4];
#pragma unroll
        for (int q = 0; q < 16; ++q)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            p[q][k] = (sidx[k] >= 0 && s0 + q < splits) ? __ldcg(ws + (int64_t)(s0 + q) * sstride + off[k]) : 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (s0 + q < splits) v[k] += p[q][k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (sidx[k] >= 0) sm.u.x[sidx[k]] = v[k];
    }
    __syncthreads();
    if (MODE == 0) apply_rinv_chunk(sm.u.x, sm.Ri, nr4);
    store_chunk(sm.u.x, nr, b, c0, out, ldo, outT, ldoT);
    gram_chunk(sm.u.x, nr4, acc);
    __syncthreads();
  }
}

__device__ __forceinline__ void load_pending_rinv(RowSmem& sm, const QrState* st, int use_pending) {
  for (int e = threadIdx.x; e < B * B; e += THREADS)
    sm.Ri[(e / B) * (B + 1) + e % B] = use_pending == 2 ? __ldcg(st->rtot + e)
                                       : use_pending  ? __ldcg(st->rinv + e)
                                                      : ((e / B == e % B) ? 1.0 : 0.0);
}

__device__ __forceinline__ void reset_qr_state(QrState* st) {
  st->plain = 0;
  st->finish = 0;
  st->done = 0;
  st->status = 0;
  st->steps = 0;
}

// MODE 0 (w = A v): finalize w from the split-K partials (ws, `splits`
// slices of stride sstride, ld ldw), times the pending R^-1 of the previous
// CholeskyQR (its last apply folded in: A (v' R^-1) = (A v') R^-1;
// identity on the first iteration), into out (+ outT); Gram; the last CTA
// writes the reduced Gram w'w (32 x 32, padded) to lam for lmax_kernel.
// MODE 1 (z = A' w): finalize z into out (the CholeskyQR buffer) + outT;
// Gram; the last CTA takes the first factor step into st.
template <int MODE>
__global__ void __launch_bounds__(THREADS, 1)
    finalize_kernel(const double* __restrict__ ws, int splits, int64_t sstride, int64_t ldw, int64_t rows, int b,
                    double* __restrict__ out, int64_t ldo, double* __restrict__ outT, int64_t ldoT,
                    double* __restrict__ part, double* __restrict__ part2, unsigned* tickets, double* lam,
                    QrState* st, double shift_coeff, double kappa_max, int use_pending) {
  __shared__ RowSmem sm;
  if (MODE == 0) load_pending_rinv(sm, st, use_pending);
  if (MODE >= 1 && blockIdx.x == 0 && threadIdx.x == 0) {
    reset_qr_state(st);  // visible to the later applies
    st->prof[4] = gtimer();
    st->prof[1] = 0;
  }
  int64_t r0, r1;
  cta_rows(rows, &r0, &r1);
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  __syncthreads();
  finalize_rows<MODE>(sm, ws, splits, sstride, ldw, r0, r1, b, out, ldo, outT, ldoT, acc);
  gram_store(acc, part, blockIdx.x);
  if (MODE == 2) return;  // deferred mode: reduce_factor_kernel (side stream) takes it from here
  if (MODE == 1 && threadIdx.x == 0) atomicMax(&st->prof[5], gtimer());
  if (!last_cta_reduce(part, part2, b, tickets, sm.u.f.G, blockIdx.x, gridDim.x)) return;
  if (MODE == 0) {
    for (int e = threadIdx.x; e < B * B; e += THREADS) lam[e] = sm.u.f.G[e];
  } else {
    if (threadIdx.x == 0) st->prof[6] = gtimer();
    factor_step(sm.u.f.G, B, b, shift_coeff, kappa_max, st, sm.u.f.W, sm.red, sm.rowj, sm.piv);
    __syncthreads();
    if (threadIdx.x == 0) st->prof[7] = gtimer();
  }
}

struct LmaxSmem {
  double G[B * B];
  double W[B * LDW];
  double d[B], e[B];
  double xs[THREADS];
  int cs[NW];
  double vs[B], wsv[B];
};

// lambda_max of the b x b Gram G (global, ld ldg) -> lam[0]; one CTA.
__global__ void __launch_bounds__(THREADS, 1) lmax_kernel(const double* __restrict__ G, int ldg, int b, double* lam) {
  __shared__ LmaxSmem sm;
  for (int e = threadIdx.x; e < b * b; e += THREADS) sm.G[e] = G[(e / b) * ldg + e % b];
  __syncthreads();
  const double l = sym_lmax(sm.G, b, b, sm.d, sm.e, sm.xs, sm.cs, sm.W, sm.vs, sm.wsv);
  if (threadIdx.x == 0) lam[0] = l;
}

// One CholeskyQR apply: x <- x R^-1 in place (rows x b, ld ldx) with the
// pending factor, plus the transposed copy xT (b x rows, ld ldxT), the Gram
// of the new rows and, in the last CTA, the next factor.  Returns at once
// when the pending factor is the final one (the next finalize_kernel<0>
// applies it) or on an error status.
// Deferred mode (defer != 0): the rows are read from xin (the raw sketch the
// concurrent sweep also reads; later steps pass xin == x) and written to x,
// and the new factor is folded into st->rtot.
__global__ void __launch_bounds__(THREADS, 1)
    apply_kernel(const double* xin, double* x, int64_t ldx, double* __restrict__ xT, int64_t ldxT, int64_t rows,
                 int b, double* __restrict__ part, double* __restrict__ part2, QrState* st, double shift_coeff,
                 double kappa_max, int last_launch, int defer) {
  __shared__ RowSmem sm;
  if (*((volatile int*)&st->finish) || *((volatile int*)&st->status)) return;  // uniform: earlier launches
  if (blockIdx.x == 0 && threadIdx.x == 0) st->prof[0] = gtimer();
  for (int e = threadIdx.x; e < B * B; e += THREADS) sm.Ri[(e / B) * (B + 1) + e % B] = __ldcg(st->rinv + e);
  int64_t r0, r1;
  cta_rows(rows, &r0, &r1);
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t c0 = r0; c0 < r1; c0 += RCH) {
    const int nr = (int)min((int64_t)RCH, r1 - c0), nr4 = (nr + 3) & ~3;
    constexpr int PER = (RCH * B + THREADS - 1) / THREADS;  // 12: all loads in flight
    double xv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = threadIdx.x + q * THREADS, r = e / B, c = e % B;
      xv[q] = (r < nr && c < b) ? xin[(c0 + r) * ldx + c] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = threadIdx.x + q * THREADS, r = e / B, c = e % B;
      if (r < nr4) sm.u.x[r * LDX + c] = xv[q];
    }
    __syncthreads();
    apply_rinv_chunk(sm.u.x, sm.Ri, nr4);
    store_chunk(sm.u.x, nr, b, c0, x, ldx, xT, ldxT);
    gram_chunk(sm.u.x, nr4, acc);
    __syncthreads();
  }
  gram_store(acc, part, blockIdx.x);
  if (threadIdx.x == 0) atomicMax(&st->prof[1], gtimer());
  if (!last_cta_reduce(part, part2, b, st->tickets, sm.u.f.G, blockIdx.x, gridDim.x)) return;
  if (threadIdx.x == 0) st->prof[2] = gtimer();
  factor_step(sm.u.f.G, B, b, shift_coeff, kappa_max, st, sm.u.f.W, sm.red, sm.rowj, sm.piv);
  __syncthreads();
  if (defer) compose_rtot(st, 0, sm.u.f.G);
  if (threadIdx.x == 0) {
    st->prof[3] = gtimer();
    st->prof[5] = 0;  // the next finalize<1>'s max-stamp starts over
  }
  // the launch budget is spent and another step would be needed
  if (threadIdx.x == 0 && last_launch && !__ldcg(&st->finish) && __ldcg(&st->status) == 0) st->status = 3;
}

// Deferred mode: the first CholeskyQR factor from the Gram partials a
// finalize_kernel<2> launch left in `part` (count slots); one CTA.
__global__ void __launch_bounds__(THREADS, 1)
    reduce_factor_kernel(const double* __restrict__ part, int count, int b, QrState* st, double shift_coeff,
                         double kappa_max) {
  __shared__ RowSmem sm;
  single_cta_reduce(part, b, count, sm.u.f.G);
  factor_step(sm.u.f.G, B, b, shift_coeff, kappa_max, st, sm.u.f.W, sm.red, sm.rowj, sm.piv);
  __syncthreads();
  // the Gram is consumed: its storage is the scratch of the composition
  compose_rtot(st, 1, sm.u.f.G);
}

}  // namespace sn
