// Small dense kernels on l x l matrices, one CTA each.  The Cholesky and QRCP
// kernels work entirely in shared memory (larger cores go to the cluster
// versions); the Jacobi kernel is compiled for shared or (L2-resident)
// global scratch as a template parameter, so every access has a known
// address space (LDS/STS, never generic LD/ST).
//
//   chol_factor_kernel : R = chol(G [+ s I]), R^-1, kappa_F — one step of the
//                        adaptive shifted CholeskyQR that replaces
//                        householder_qr (dense.py:132-149) for the sketches.
//   qrcp_kernel        : Businger-Golub QRCP of the compressed core
//                        (dense.py:152-192), explicit Q by reverse
//                        accumulation (dense.py:117-129).
//   jacobi_kernel      : one-sided Jacobi (dense.py:223-282) for singular
//                        values / pseudoinverse of small matrices.
#pragma once
#include "common.cuh"

namespace small {

constexpr int THREADS = 1024;
constexpr int NWARPS = THREADS / 32;
constexpr int LMAX = 640;  // largest core dimension supported

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// ----------------------------------------------------------- Cholesky step
struct CholInfo {
  int shifted;   // 1 if the shift was applied
  int status;    // 0 ok, 1 zero matrix (R = I), 2 failure (non-finite)
  double kappa;  // |R|_F |R^-1|_F of the applied factor
  double trace;
};

// The augmented matrix [G | I] (row-major, ld = 2l): the row operations
// that turn G into R (R'R = G) turn I into R^-T, so the right half ends up
// holding rinvT[j][k] = R^-1[k][j] -- exactly the Bt operand of the X * R^-1
// GEMM -- without a separate triangular inverse.  NB: panel height of the
// cluster version (chol_cluster.cuh).
constexpr int NB = 32;

// Unblocked right-looking Cholesky of [G | I] in shared memory (l < 64):
// two barriers per column, the trailing update spread over warps (rows) and
// lanes (columns) with no serial chains -- latency-optimal for small cores.
__device__ bool chol_aug_unblocked(double* W, int l) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nw = nt >> 5;
  const int ld = 2 * l;
  for (int j = 0; j < l; ++j) {
    const double d = W[j * ld + j];
    if (!(d > 0.0) || !isfinite(d)) return true;  // uniform
    const double r = sqrt(d);
    const int nl = l - j - 1;
    for (int t = tid; t < nl + j + 1; t += nt) {
      const int k = (t < nl) ? (j + 1 + t) : (l + (t - nl));
      W[j * ld + k] = W[j * ld + k] / r;
    }
    __syncthreads();
    if (tid == 0) W[j * ld + j] = r;
    for (int i = j + 1 + warp; i < l; i += nw) {
      const double a = W[j * ld + i];
      double* wi = W + i * ld;
      const double* wj = W + j * ld;
      for (int k = i + lane; k < l; k += 32) wi[k] -= a * wj[k];
      for (int k = lane; k <= j; k += 32) wi[l + k] -= a * wj[l + k];
    }
    __syncthreads();
  }
  return false;
}

__device__ double upper_sumsq(const double* W, int l, int ld, int col0, bool lower, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x >> 5; i < l; i += blockDim.x >> 5)
    for (int k = threadIdx.x & 31; k < l; k += 32) {
      if (lower ? (k > i) : (k < i)) continue;
      const double v = W[(int64_t)i * ld + col0 + k];
      s += v * v;
    }
  return block_sum(s, red);
}

// G: l x l (ld ldg).  shift_coeff = 11 (m l + l (l + 1)) u  (shifted
// CholeskyQR, Fukaya et al. 2020).  allow_plain: try the unshifted factor
// first and keep it when it succeeds with kappa_F <= kappa_max.
// Output rinvT (l x l, ld ldr): rinvT[j][k] = R^-1[k][j] (the Bt operand of
// the X * R^-1 GEMM).  Work: [G | I], 2 l^2 doubles of shared memory.
// The factorisation itself, for one whole CTA (any block size) with W =
// 2 l^2 doubles and red = NWARPS doubles of shared memory; also called by
// the fused tall-skinny CholeskyQR (skinny.cuh).
__device__ void chol_factor_block(const double* G, int l, int64_t ldg, double shift_coeff, int allow_plain,
                                  double kappa_max, double* rinvT, int64_t ldr, CholInfo* info, double* W,
                                  double* red) {
  const int ld = 2 * l;
  double tr = 0.0;
  for (int i = threadIdx.x; i < l; i += blockDim.x) tr += G[i * ldg + i];
  tr = block_sum(tr, red);
  int shifted = allow_plain ? 0 : 1;
  int status = 0;
  double kappa = 0.0;
  if (!(tr > 0.0) || !isfinite(tr)) {
    // exactly zero sketch (or garbage): R = I, Q = X.
    for (int i = threadIdx.x >> 5; i < l; i += blockDim.x >> 5)
      for (int k = threadIdx.x & 31; k < l; k += 32) W[(int64_t)i * ld + l + k] = (i == k) ? 1.0 : 0.0;
    status = isfinite(tr) ? 1 : 2;
    kappa = 1.0;
    __syncthreads();
  } else {
    for (;;) {
      const double s = shifted ? shift_coeff * tr : 0.0;
      for (int i = threadIdx.x >> 5; i < l; i += blockDim.x >> 5)
        for (int k = threadIdx.x & 31; k < 2 * l; k += 32) {
          double g;
          if (k < l) {
            g = (k >= i) ? G[i * ldg + k] : 0.0;
            if (i == k) g += s;
          } else {
            g = (k - l == i) ? 1.0 : 0.0;
          }
          W[(int64_t)i * ld + k] = g;
        }
      __syncthreads();
      const bool fail = chol_aug_unblocked(W, l);
      __syncthreads();
      if (fail) {
        if (!shifted) { shifted = 1; continue; }
        status = 2;
        break;
      }
      const double nr = upper_sumsq(W, l, ld, 0, false, red);
      const double ni = upper_sumsq(W, l, ld, l, true, red);
      kappa = sqrt(nr) * sqrt(ni);
      if (!shifted && !(kappa <= kappa_max)) { shifted = 1; __syncthreads(); continue; }
      break;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x >> 5; j < l; j += blockDim.x >> 5)  // rinvT = right half (lower)
    for (int k = threadIdx.x & 31; k < l; k += 32) rinvT[j * ldr + k] = (k <= j) ? W[(int64_t)j * ld + l + k] : 0.0;
  if (threadIdx.x == 0) {
    info->shifted = shifted;
    info->status = status;
    info->kappa = kappa;
    info->trace = tr;
  }
}

__global__ void __launch_bounds__(512, 1)
    chol_factor_kernel(const double* __restrict__ G, int l, int64_t ldg, double shift_coeff,
                       int allow_plain, double kappa_max, double* __restrict__ rinvT,
                       int64_t ldr, double* gwork, int use_smem, CholInfo* info, int* qd) {
  extern __shared__ double dsm[];
  __shared__ double red[NWARPS];
  // [G | I] always in shared memory here (the host launches this kernel only
  // when it fits; larger cores use the cluster kernel), so every access is
  // an LDS/STS rather than a generic LD/ST
  (void)use_smem;
  (void)gwork;
  // qd (optional, speculative schedule): {plain, done, status, steps} of
  // cholqr_multi's rule on the device (as creg::chol_reg_kernel); once done
  // the step is an exact no-op, R^-1 = I
  if (qd && *((volatile int*)&qd[1])) {
    for (int e = threadIdx.x; e < l * l; e += blockDim.x) {
      const int i = e / l, k = e % l;
      rinvT[(int64_t)i * ldr + k] = (i == k) ? 1.0 : 0.0;
    }
    return;
  }
  chol_factor_block(G, l, ldg, shift_coeff, allow_plain, kappa_max, rinvT, ldr, info, dsm, red);
  if (qd && threadIdx.x == 0) {
    const int plain = info->shifted ? 0 : qd[0] + 1;
    qd[0] = plain;
    qd[3] += 1;
    if (info->status == 2) qd[2] = 2;
    if (info->status != 0 || plain == 2) qd[1] = 1;
  }
}

// ------------------------------------------------------------------- QRCP
// D: l x l (ld ldd).  Outputs: T (ld ldt) = triu(R); qtT (ld ldq):
// qtT[j][i] = Q[i][j]; perm (int64) and perm32.
//
// Businger-Golub exactly as dense.py:152-192, organised for one CTA with a
// single barrier per pivot step: columns never move physically (a
// logical->physical map is double-buffered by step parity, so the
// lowest-LOGICAL-index tie-break of dense.py:169 is kept), every warp
// redundantly computes the pivot argmax and the reflector norm (no barrier
// needed to broadcast them), and a group of G lanes owns each physical
// column: it forms the column's reflector coefficient (G-way split dot +
// shuffle reduction), applies the update and downdates / refreshes the
// column norm (dense.py:181-190).  The new diagonal goes to diag[] so the
// pivot column stays read-only within a step.  R / Q live in shared memory
// when they fit (smem_R / smem_Q), else in L2-resident global scratch.
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G, int LM>
__device__ int qrcp_body(double* R, double* Q, int l, double* nrm, double* ref, double* tau,
                         double* vhead, double* diag, int (*l2p)[LM], int* done, int* has_ref,
                         const int** fin_out, double delta, int* rcount_out) {
  const int lane = threadIdx.x & 31;
  const int nt = blockDim.x;
  const int gid = threadIdx.x / G, gl = threadIdx.x % G;
  const int ngroups = nt / G;
  int kend = l;
  int rcount = 0;  // #(|diag T| > delta) over the steps taken (rpca.py:123-124)
  for (int j = 0; j < l; ++j) {
    const int* cur = l2p[j & 1];
    int* nxt = l2p[(j + 1) & 1];
    // pivot = first logical position of the max downdated norm (every warp)
    double best = -1.0;
    int bq = l;
    for (int q = j + lane; q < l; q += 32) {
      const double v = nrm[cur[q]];
      if (v > best) { best = v; bq = q; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
      if (ov > best || (ov == best && oq < bq)) { best = ov; bq = oq; }
    }
    // truncation (delta >= 0): stop once no remaining column can give
    // |diag T| > delta -- the largest downdated norm^2 (within 1e-3 of the
    // true one: refreshed below 1e-10 of its reference) is below delta^2.
    // The reference counts the whole diagonal (rpca.py:123-124), which may
    // be slightly non-monotone around delta; steps up to here are counted
    if (delta >= 0.0 && best * 1.001 < delta * delta) {
      kend = j;
      break;
    }
    const int p = bq;
    const int pc = cur[p];
    // reflector of x = R[j:, pc] (dense.py:104-114), every warp
    const double x0 = R[j * l + pc];
    double t2 = 0.0;
    for (int i = j + 1 + lane; i < l; i += 32) t2 += R[i * l + pc] * R[i * l + pc];
    t2 = warp_sum(t2);
    const double nx = sqrt(x0 * x0 + t2);
    const bool refl = nx != 0.0;
    const double v0 = refl ? x0 + (x0 >= 0.0 ? nx : -nx) : 0.0;
    const double tj = refl ? 2.0 / (v0 * v0 + t2) : 0.0;
    const double dj = refl ? x0 - v0 * (tj * (v0 * x0 + t2)) : x0;
    rcount += (fabs(dj) > delta) ? 1 : 0;
    for (int q = threadIdx.x; q < l; q += nt) nxt[q] = (q == j) ? cur[p] : ((q == p) ? cur[j] : cur[q]);
    if (threadIdx.x == 0) {
      diag[j] = dj;
      tau[j] = tj;
      vhead[j] = v0;
      has_ref[j] = refl;
    }
    // apply H_j to the other active columns: group per physical column
    for (int cb = 0; cb < l; cb += ngroups) {
      const int c = cb + gid;
      const bool act = c < l && c != pc && !done[c];
      const int cc = act ? c : pc;  // inactive lanes read a valid column
      double s = 0.0;
      if (refl) {
        for (int i = j + 1 + gl; i < l; i += G) s += R[i * l + pc] * R[i * l + cc];
        if (gl == 0) s += v0 * R[j * l + cc];
        s = group_sum<G>(s);
        const double w = tj * s;
        if (act) {
          for (int i = j + 1 + gl; i < l; i += G) R[i * l + c] -= R[i * l + pc] * w;
          if (gl == 0) R[j * l + c] -= v0 * w;
        }
      }
      // norm downdate (dense.py:181-185), refresh when stale (dense.py:185-190)
      double nv = 0.0;
      bool stale = false;
      if (act && j + 1 < l) {
        const double rj = R[j * l + c];  // gl == 0 wrote it; same lane reads
        nv = fmax(nrm[c] - rj * rj, 0.0);
        stale = nv < 1e-10 * ref[c];
      }
      stale = __shfl_sync(0xffffffffu, stale ? 1 : 0, (lane / G) * G) != 0;
      if (__any_sync(0xffffffffu, stale)) {
        double f = 0.0;
        for (int i = j + 1 + gl; i < l; i += G) f += R[i * l + cc] * R[i * l + cc];
        f = group_sum<G>(f);
        if (stale) nv = f;
        if (stale && gl == 0) ref[c] = f;
      }
      if (act && gl == 0 && j + 1 < l) nrm[c] = nv;
    }
    if (threadIdx.x == 0) done[pc] = 1;
    __syncthreads();
  }
  __syncthreads();
  const int* fin = l2p[kend & 1];
  *fin_out = fin;
  *rcount_out = delta >= 0.0 ? rcount : kend;

  // explicit Q by reverse accumulation on the identity (dense.py:117-129)
  for (int i = threadIdx.x >> 5; i < l; i += nt >> 5)
    for (int c = lane; c < l; c += 32) Q[i * l + c] = (i == c) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = kend - 1; j >= 0; --j) {
    if (has_ref[j]) {
      const int pc = fin[j];
      const double v0 = vhead[j], tj = tau[j];
      for (int cb = j; cb < l; cb += ngroups) {
        const int c = cb + gid;
        const bool act = c < l;
        const int cc = act ? c : j;
        double s = 0.0;
        for (int i = j + 1 + gl; i < l; i += G) s += R[i * l + pc] * Q[i * l + cc];
        if (gl == 0) s += v0 * Q[j * l + cc];
        s = group_sum<G>(s);
        const double w = tj * s;
        if (act) {
          for (int i = j + 1 + gl; i < l; i += G) Q[i * l + c] -= R[i * l + pc] * w;
          if (gl == 0) Q[j * l + c] -= v0 * w;
        }
      }
    }
    __syncthreads();
  }
  return kend;
}

// LM: capacity of the per-column arrays (the core must satisfy l <= LM);
// G: lanes per column.  The host launches ~G * l threads so the redundant
// per-warp pivot/norm work stays small (few warps) for small cores.
template <int LM, int G>
__global__ void __launch_bounds__(1024, 1)
    qrcp_kernel(const double* __restrict__ D, int l, int64_t ldd, double* __restrict__ T,
                int64_t ldt, double* __restrict__ qtT, int64_t ldq, long long* perm_out,
                int* perm32, double* gwork, int smem_R, int smem_Q, double delta, int* r_out) {
  extern __shared__ double dsm[];
  __shared__ double nrm[LM];
  __shared__ double ref[LM];
  __shared__ double tau[LM];
  __shared__ double vhead[LM];
  __shared__ double diag[LM];
  __shared__ int l2p[2][LM];
  __shared__ int done[LM];
  __shared__ int has_ref[LM];
  const int lane = threadIdx.x & 31;
  const int nt = blockDim.x;
  // R and Q always in shared memory here (the host launches this kernel
  // only when they fit); a pointer chosen at run time between shared and
  // global memory would compile every access to a generic LD/ST
  (void)smem_R;
  (void)smem_Q;
  (void)gwork;
  double* R = dsm;
  double* Q = dsm + l * l;

  for (int i = threadIdx.x >> 5; i < l; i += nt >> 5)
    for (int c = lane; c < l; c += 32) R[i * l + c] = D[i * ldd + c];
  __syncthreads();
  // initial column norms^2 (dense.py:165-166)
  for (int c = threadIdx.x >> 5; c < l; c += nt >> 5) {
    double s = 0.0;
    for (int i = lane; i < l; i += 32) s += R[i * l + c] * R[i * l + c];
    s = warp_sum(s);
    if (lane == 0) {
      nrm[c] = s;
      ref[c] = s;
      l2p[0][c] = c;
      done[c] = 0;
    }
  }
  __syncthreads();
  const int* fin = nullptr;
  int rcount = 0;
  const int kend = qrcp_body<G, LM>(R, Q, l, nrm, ref, tau, vhead, diag, l2p, done, has_ref, &fin, delta, &rcount);
  __syncthreads();
  for (int i = threadIdx.x >> 5; i < l; i += nt >> 5)
    for (int c = lane; c < l; c += 32) {
      T[i * ldt + c] = (i >= kend) ? 0.0 : ((c > i) ? R[i * l + fin[c]] : ((c == i) ? diag[i] : 0.0));
      qtT[c * ldq + i] = Q[i * l + c];
    }
  if (threadIdx.x == 0 && r_out) *r_out = rcount;
  for (int c = threadIdx.x; c < l; c += nt) {
    if (perm_out) perm_out[c] = fin[c];
    perm32[c] = fin[c];
  }
}

// Left-factor completion for zero singular values (dense.py:285-310), one
// warp: row j of ut (sorted order, sig_sorted[j] == 0) is replaced by the
// first unit-vector candidate e_cand that keeps norm > 0.1 after two
// Gram-Schmidt passes against the kept rows (index order) and the earlier
// fills.  Returns true when the candidates run out.
__device__ bool complete_left(double* ut_out, int64_t ldut, const double* sig_sorted, int nv, int len,
                              int lane) {
  int cand = 0;
  for (int j = 0; j < nv; ++j) {
    if (sig_sorted[j] > 0.0) continue;
    for (;;) {
      if (cand >= len) return true;
      for (int i = lane; i < len; i += 32) ut_out[j * ldut + i] = (i == cand) ? 1.0 : 0.0;
      ++cand;
      __syncwarp();
      for (int pass = 0; pass < 2; ++pass) {
        // basis: kept vectors (sig > 0) in index order, then earlier fills
        for (int b = 0; b < 2 * nv; ++b) {
          const int kb = b < nv ? b : b - nv;
          const bool kept = sig_sorted[kb] > 0.0;
          if (b < nv ? !kept : (kept || kb >= j)) continue;
          double d = 0.0;
          for (int i = lane; i < len; i += 32) d += ut_out[kb * ldut + i] * ut_out[j * ldut + i];
          d = warp_sum(d);
          for (int i = lane; i < len; i += 32) ut_out[j * ldut + i] -= d * ut_out[kb * ldut + i];
          __syncwarp();
        }
      }
      double nw = 0.0;
      for (int i = lane; i < len; i += 32) nw += ut_out[j * ldut + i] * ut_out[j * ldut + i];
      nw = sqrt(warp_sum(nw));
      if (nw > 0.1) {
        for (int i = lane; i < len; i += 32) ut_out[j * ldut + i] /= nw;
        __syncwarp();
        break;
      }
    }
  }
  return false;
}

// ---------------------------------------------------------------- Jacobi
// One-sided Jacobi on the nv rows (length len, ld ldx) of X: orthogonalises
// them by plane rotations in the round-robin order of dense.py:200-210,
// until every pair has |<xa,xb>| <= tol |xa||xb| (dense.py:223-282).
// One warp per pair (pairs of a round are disjoint), pairs computed
// arithmetically by each warp, one barrier per round.
// sig (device, nv, descending).  pinv != nullptr: B = X^T (len x nv) and
// pinv(B) (nv x len, ld ldp) is written with the cutoff
// max(len, nv) * sig0 * 1e-12 (dense.py:390-402).
template <bool USE_SMEM>
__global__ void __launch_bounds__(THREADS, 1)
    jacobi_kernel(const double* __restrict__ X, int nv, int len, int64_t ldx, double tol,
                  int max_sweeps, double* sig_out, double* pinv, int64_t ldp, double* ut_out,
                  int64_t ldut, double* vt_out, int64_t ldvt, double* gwork, int use_smem,
                  int* status) {
  extern __shared__ double dsm[];
  __shared__ double offmax[NWARPS];
  __shared__ double sig[LMAX];
  __shared__ int order[LMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int nt = blockDim.x;
  const int n = nv + (nv > 1 && (nv & 1));  // pad odd counts with a zero row
  const bool want_v = pinv != nullptr || vt_out != nullptr;
  (void)use_smem;
  double* W = USE_SMEM ? dsm : gwork;          // n x len (compile-time address space)
  double* V = W + (int64_t)n * len;            // n x n (row a = column a of V)
  for (int r = warp; r < n; r += nwarps)
    for (int c = lane; c < len; c += 32) W[(int64_t)r * len + c] = (r < nv) ? X[r * ldx + c] : 0.0;
  if (want_v)
    for (int r = warp; r < n; r += nwarps)
      for (int c = lane; c < n; c += 32) V[(int64_t)r * n + c] = (r == c) ? 1.0 : 0.0;
  __syncthreads();
  int st = 0;
  if (n > 1) {
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
      double off = 0.0;
      for (int round = 0; round < n - 1; ++round) {
        for (int pi = warp; pi < n / 2; pi += nwarps) {
          // ring position -> player: position 0 fixed, the others rotate
          auto ring = [&](int pos) -> int {
            if (pos == 0) return 0;
            int q = (pos - 1 - round) % (n - 1);
            if (q < 0) q += n - 1;
            return 1 + q;
          };
          const int a = ring(pi), b = ring(n - 1 - pi);
          double* xa = W + (int64_t)a * len;
          double* xb = W + (int64_t)b * len;
          double al = 0.0, be = 0.0, ga = 0.0;
          for (int i = lane; i < len; i += 32) {
            const double u = xa[i], v = xb[i];
            al += u * u;
            be += v * v;
            ga += u * v;
          }
          al = warp_sum(al);
          be = warp_sum(be);
          ga = warp_sum(ga);
          const double den = sqrt(al * be);
          const double rel = den > 0.0 ? fabs(ga) / den : 0.0;
          off = fmax(off, rel);
          if (rel > tol) {
            const double zeta = (be - al) / (2.0 * ga);
            const double sgn = zeta >= 0.0 ? 1.0 : -1.0;
            const double t = sgn / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t);
            const double s = c * t;
            for (int i = lane; i < len; i += 32) {
              const double u = xa[i], v = xb[i];
              xa[i] = c * u - s * v;
              xb[i] = s * u + c * v;
            }
            if (want_v) {
              double* va = V + (int64_t)a * n;
              double* vb = V + (int64_t)b * n;
              for (int i = lane; i < n; i += 32) {
                const double u = va[i], v = vb[i];
                va[i] = c * u - s * v;
                vb[i] = s * u + c * v;
              }
            }
          }
        }
        __syncthreads();
      }
      if (lane == 0) offmax[warp] = off;
      __syncthreads();
      double mm = 0.0;
      for (int w = 0; w < nwarps; ++w) mm = fmax(mm, offmax[w]);
      __syncthreads();
      if (mm <= tol) break;
    }
    if (sweep == max_sweeps) st = 1;
  }
  // singular values and stable descending order (dense.py:339-341)
  for (int r = warp; r < nv; r += nwarps) {
    double s = 0.0;
    for (int i = lane; i < len; i += 32) s += W[(int64_t)r * len + i] * W[(int64_t)r * len + i];
    s = warp_sum(s);
    if (lane == 0) sig[r] = sqrt(s);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nv; r += nt) {
    int rank = 0;
    for (int q = 0; q < nv; ++q) rank += (sig[q] > sig[r]) || (sig[q] == sig[r] && q < r);
    order[rank] = r;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nv; k += nt) sig_out[k] = sig[order[k]];
  if (pinv) {
    // B = X^T = U S V^T with U[:, k] = W[k] / sig_k.  pinv = V S^+ U^T.
    const double s0 = sig[order[0]];
    const double cut = (double)max(len, nv) * s0 * 1e-12;
    for (int i = warp; i < nv; i += nwarps)
      for (int j = lane; j < len; j += 32) {
        double acc = 0.0;
        if (s0 > 0.0) {
          for (int k = 0; k < nv; ++k) {
            const double sk = sig[k];
            if (sk > cut) acc += V[(int64_t)k * n + i] * (W[(int64_t)k * len + j] / sk) / sk;
          }
        }
        pinv[i * ldp + j] = acc;
      }
  }
  if (ut_out || vt_out) {
    // economy SVD of B = X^T (dense.py:339-352): B[:, order[k]] / sig_k is
    // left vector k (row k of ut_out), column order[k] of the accumulated
    // rotations right vector k (row k of vt_out)
    for (int k = warp; k < nv; k += nwarps) {
      const int r = order[k];
      const double sk = sig[r];
      if (ut_out)
        for (int i = lane; i < len; i += 32)
          ut_out[k * ldut + i] = (sk > 0.0) ? W[(int64_t)r * len + i] / sk : 0.0;
      if (vt_out)
        for (int i = lane; i < nv; i += 32) vt_out[k * ldvt + i] = V[(int64_t)r * n + i];
    }
    __syncthreads();
    // zero singular values: complete the left factor (dense.py:285-310)
    if (ut_out && warp == 0 && complete_left(ut_out, ldut, sig_out, nv, len, lane)) st = 2;
  }
  if (threadIdx.x == 0 && status) *status = st;
}

// Largest eigenvalue of a symmetric b x b matrix G (b <= 32; the lower
// triangle is read), one warp: Householder tridiagonalisation (LAPACK
// dsytd2 / dlarfg conventions) then multisection on the tridiagonal with
// Sturm counts, 32 shifts per step.  Both stages are backward stable, so
// lambda_max is accurate to a few u ||G|| -- what the block power iteration
// of spectral_norm needs from sigma_1(w)^2 = lambda_max(w'w) (dense.py:425-431
// takes sigma_1 of the QR factor of w; same value to rounding).
constexpr int LMAX_THREADS = 256;

__global__ void __launch_bounds__(LMAX_THREADS) sym_lmax_kernel(const double* __restrict__ G, int b, int64_t ldg,
                                                                double* __restrict__ out) {
  // 8 warps: rows of the Householder updates are spread over the warps
  // (warp w owns rows i = w mod 8), and the multisection evaluates 256
  // shifts per step (8 bits) instead of 32
  __shared__ double A[32][33];
  __shared__ double ps[32], d[32], e[32];
  __shared__ double xs[LMAX_THREADS];
  __shared__ int cs[LMAX_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = LMAX_THREADS / 32;
  for (int idx = tid; idx < b * b; idx += LMAX_THREADS) {
    const int i = idx / b, j = idx % b;
    A[i][j] = (i >= j) ? G[i * ldg + j] : G[j * ldg + i];
  }
  __syncthreads();
  for (int k = 0; k + 2 < b; ++k) {
    // reflector for x = A[k+1:b, k]:  H x = beta e1, H = I - tau v v', v[0] = 1
    // (every warp forms the same scalars and v from shared memory)
    const double alpha = A[k + 1][k];
    const double xt = (lane > k + 1 && lane < b) ? A[lane][k] : 0.0;
    const double sigma = warp_sum(xt * xt);
    if (sigma == 0.0) {
      if (tid == 0) {
        d[k] = A[k][k];
        e[k] = alpha;
      }
      __syncthreads();
      continue;
    }
    const double nrm = sqrt(alpha * alpha + sigma);
    const double beta = (alpha >= 0.0) ? -nrm : nrm;
    const double tau = (beta - alpha) / beta;
    const double scal = 1.0 / (alpha - beta);
    const double vi = (lane == k + 1) ? 1.0 : ((lane > k + 1 && lane < b) ? A[lane][k] * scal : 0.0);
    // p = tau A22 v, one warp-reduced row at a time
    for (int i = k + 1 + warp; i < b; i += NW) {
      const double pr = warp_sum((lane > k && lane < b) ? A[i][lane] * vi : 0.0);
      if (lane == 0) ps[i] = tau * pr;
    }
    __syncthreads();
    const double pi = (lane > k && lane < b) ? ps[lane] : 0.0;
    // w = p - (tau/2)(p'v) v ; A22 -= v w' + w v'
    const double kk = -0.5 * tau * warp_sum(pi * vi);
    const double wi = fma(kk, vi, pi);
    if (tid == 0) {
      d[k] = A[k][k];
      e[k] = beta;
    }
    for (int i = k + 1 + warp; i < b; i += NW) {
      const double vr = __shfl_sync(0xffffffffu, vi, i), wr = __shfl_sync(0xffffffffu, wi, i);
      if (lane > k && lane < b) A[i][lane] -= vr * wi + wr * vi;
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (b >= 2) {
      d[b - 2] = A[b - 2][b - 2];
      e[b - 2] = A[b - 1][b - 2];
    }
    d[b - 1] = A[b - 1][b - 1];
  }
  __syncthreads();
  // Gershgorin bracket of lambda_max
  double lo = 1e308, hi = -1e308, emax2 = 0.0;
  for (int i = 0; i < b; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < b ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    if (i + 1 < b) emax2 = fmax(emax2, e[i] * e[i]);
  }
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2);
  const double span = fmax(fabs(lo), fabs(hi));
  lo -= 4.0 * 2.220446049250313e-16 * span + pivmin;
  hi += 4.0 * 2.220446049250313e-16 * span + pivmin;
  // multisection: count(x) = #eigenvalues < x; lambda_max in [lo, hi)
  for (int step = 0; step < 64; ++step) {
    const double x = lo + (hi - lo) * ((double)(tid + 1) / (double)(LMAX_THREADS + 1));
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0.0);
    for (int i = 1; i < b; ++i) {
      q = (d[i] - x) - e[i - 1] * e[i - 1] / q;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += (q < 0.0);
    }
    xs[tid] = x;
    // smallest shift above lambda_max (cnt == b); counts are monotone in x
    const unsigned above = __ballot_sync(0xffffffffu, cnt == b);
    if (lane == 0) cs[warp] = above ? warp * 32 + __ffs(above) - 1 : LMAX_THREADS;
    __syncthreads();
    int f = LMAX_THREADS;
    for (int w = 0; w < NW; ++w) f = min(f, cs[w]);
    double nlo = lo, nhi = hi;
    if (f < LMAX_THREADS) {
      nhi = xs[f];
      if (f > 0) nlo = xs[f - 1];
    } else {
      nlo = xs[LMAX_THREADS - 1];
    }
    __syncthreads();
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
    if (hi - lo <= 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi))) break;
  }
  if (tid == 0) out[0] = 0.5 * (lo + hi);
}

}  // namespace small
