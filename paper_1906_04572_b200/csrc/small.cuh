// Small dense kernels on l x l (l <= ~600) matrices, one CTA each, working in
// shared memory when the matrix fits and in (L2-resident) global scratch
// otherwise — the pointer is generic either way.
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
    t = (lane < NWARPS) ? red[lane] : 0.0;
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

// Returns true on failure.  W holds G's upper triangle (row-major, ld l).
__device__ bool chol_upper_inplace(double* W, int l, double* red) {
  for (int j = 0; j < l; ++j) {
    __syncthreads();
    const double d = W[j * l + j];
    if (!(d > 0.0) || !isfinite(d)) return true;
    const double r = sqrt(d);
    for (int k = j + 1 + threadIdx.x; k < l; k += THREADS) W[j * l + k] = W[j * l + k] / r;
    __syncthreads();
    if (threadIdx.x == 0) W[j * l + j] = r;
    const int T = l - j - 1;
    for (int idx = threadIdx.x; idx < T * T; idx += THREADS) {
      const int i = j + 1 + idx / T, k = j + 1 + idx % T;
      if (k >= i) W[i * l + k] -= W[j * l + i] * W[j * l + k];
    }
  }
  __syncthreads();
  return false;
}

__device__ double upper_sumsq(const double* W, int l, double* red) {
  double s = 0.0;
  for (int idx = threadIdx.x; idx < l * l; idx += THREADS) {
    const int i = idx / l, k = idx % l;
    if (k >= i) s += W[idx] * W[idx];
  }
  return block_sum(s, red);
}

// In-place inverse of an upper-triangular matrix, column by column.
__device__ void inv_upper_inplace(double* W, int l, double* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < l; ++j) {
    __syncthreads();
    const double invd = 1.0 / W[j * l + j];
    for (int i = warp; i < j; i += NWARPS) {
      double s = 0.0;
      for (int k = i + lane; k < j; k += 32) s += W[i * l + k] * W[k * l + j];
      s = warp_sum(s);
      if (lane == 0) tmp[i] = -s * invd;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < j; i += THREADS) W[i * l + j] = tmp[i];
    if (threadIdx.x == 0) W[j * l + j] = invd;
  }
  __syncthreads();
}

// G: l x l (ld ldg).  shift_coeff = 11 (m l + l (l + 1)) u  (shifted
// CholeskyQR, Fukaya et al. 2020).  allow_plain: try the unshifted factor
// first and keep it when it succeeds with kappa_F <= kappa_max.
// Output rinvT (l x l, ld ldr): rinvT[j][k] = R^-1[k][j] (the Bt operand of
// the X * R^-1 GEMM).
__global__ void __launch_bounds__(THREADS, 1)
    chol_factor_kernel(const double* __restrict__ G, int l, int64_t ldg, double shift_coeff,
                       int allow_plain, double kappa_max, double* __restrict__ rinvT,
                       int64_t ldr, double* gwork, int use_smem, CholInfo* info) {
  extern __shared__ double dsm[];
  __shared__ double red[NWARPS];
  __shared__ double tmp[LMAX];
  double* W = use_smem ? dsm : gwork;
  double tr = 0.0;
  for (int i = threadIdx.x; i < l; i += THREADS) tr += G[i * ldg + i];
  tr = block_sum(tr, red);
  int shifted = allow_plain ? 0 : 1;
  int status = 0;
  double kappa = 0.0;
  if (!(tr > 0.0) || !isfinite(tr)) {
    // exactly zero sketch (or garbage): R = I, Q = X.
    for (int idx = threadIdx.x; idx < l * l; idx += THREADS) W[idx] = (idx / l == idx % l) ? 1.0 : 0.0;
    status = isfinite(tr) ? 1 : 2;
    kappa = 1.0;
    __syncthreads();
  } else {
    for (;;) {
      const double s = shifted ? shift_coeff * tr : 0.0;
      for (int idx = threadIdx.x; idx < l * l; idx += THREADS) {
        const int i = idx / l, k = idx % l;
        double g = (k >= i) ? G[i * ldg + k] : 0.0;
        if (i == k) g += s;
        W[idx] = g;
      }
      __syncthreads();
      const bool fail = chol_upper_inplace(W, l, red);
      if (fail) {
        if (!shifted) { shifted = 1; __syncthreads(); continue; }
        status = 2;
        break;
      }
      const double nr = upper_sumsq(W, l, red);
      inv_upper_inplace(W, l, tmp);
      const double ni = upper_sumsq(W, l, red);
      kappa = sqrt(nr) * sqrt(ni);
      if (!shifted && !(kappa <= kappa_max)) { shifted = 1; __syncthreads(); continue; }
      break;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < l * l; idx += THREADS) {
    const int k = idx / l, j = idx % l;  // rinvT[j][k] = Rinv[k][j]
    rinvT[j * ldr + k] = (j >= k) ? W[k * l + j] : 0.0;
  }
  if (threadIdx.x == 0) {
    info->shifted = shifted;
    info->status = status;
    info->kappa = kappa;
    info->trace = tr;
  }
}

// ------------------------------------------------------------------- QRCP
// D: l x l (ld ldd).  Outputs: T (ld ldt) = triu(R); qtT (ld ldq):
// qtT[j][i] = Q[i][j]; perm (int64) and perm32.
// WR / WQ: l x l work (smem or global).  Small per-column state lives in
// static shared arrays of LMAX.
__global__ void __launch_bounds__(THREADS, 1)
    qrcp_kernel(const double* __restrict__ D, int l, int64_t ldd, double* __restrict__ T,
                int64_t ldt, double* __restrict__ qtT, int64_t ldq, long long* perm_out,
                int* perm32, double* gwork, int smem_R, int smem_Q) {
  extern __shared__ double dsm[];
  __shared__ double red[NWARPS];
  __shared__ double nrm[LMAX];
  __shared__ double ref[LMAX];
  __shared__ double tau[LMAX];
  __shared__ double vhead[LMAX];
  __shared__ int perm[LMAX];
  __shared__ int has_ref[LMAX];
  __shared__ int piv_idx[NWARPS];
  __shared__ double piv_val[NWARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* R = smem_R ? dsm : gwork;
  double* Q = smem_Q ? (smem_R ? dsm + l * l : dsm) : gwork + (int64_t)l * l;

  for (int idx = threadIdx.x; idx < l * l; idx += THREADS) R[idx] = D[(idx / l) * ldd + idx % l];
  __syncthreads();
  // initial column norms^2 (dense.py:165-166)
  for (int c = warp; c < l; c += NWARPS) {
    double s = 0.0;
    for (int i = lane; i < l; i += 32) s += R[i * l + c] * R[i * l + c];
    s = warp_sum(s);
    if (lane == 0) { nrm[c] = s; ref[c] = s; perm[c] = c; }
  }
  __syncthreads();

  for (int j = 0; j < l; ++j) {
    // pivot: argmax nrm[j:], first index on ties (dense.py:169)
    double best = -1.0;
    int bi = l;
    for (int c = j + threadIdx.x; c < l; c += THREADS) {
      const double v = nrm[c];
      if (v > best) { best = v; bi = c; }  // increasing c: keeps first max
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { piv_val[warp] = best; piv_idx[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = piv_val[lane];
      bi = piv_idx[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) piv_idx[0] = bi;
    }
    __syncthreads();
    const int p = piv_idx[0];
    if (p != j) {
      for (int i = threadIdx.x; i < l; i += THREADS) {
        const double t = R[i * l + j];
        R[i * l + j] = R[i * l + p];
        R[i * l + p] = t;
      }
      if (threadIdx.x == 0) {
        int ti = perm[j]; perm[j] = perm[p]; perm[p] = ti;
        double t = nrm[j]; nrm[j] = nrm[p]; nrm[p] = t;
        t = ref[j]; ref[j] = ref[p]; ref[p] = t;
      }
    }
    __syncthreads();
    // reflector of x = R[j:, j] (dense.py:104-114)
    double part = 0.0;
    for (int i = j + threadIdx.x; i < l; i += THREADS) part += R[i * l + j] * R[i * l + j];
    const double nx2 = block_sum(part, red);
    const double x0 = R[j * l + j];
    __syncthreads();  // x0 is overwritten below by the warp owning column j
    const bool refl = (sqrt(nx2) != 0.0);
    double v0 = 0.0, tj = 0.0;
    if (refl) {
      const double nx = sqrt(nx2);
      v0 = x0 + (x0 >= 0.0 ? nx : -nx);
      // v'v = v0^2 + sum_{i>j} x_i^2
      tj = 2.0 / (v0 * v0 + (nx2 - x0 * x0));
    }
    if (threadIdx.x == 0) { has_ref[j] = refl; tau[j] = tj; vhead[j] = v0; }
    // apply H to columns c >= j; warp per column.  Column j keeps v below
    // the diagonal (LAPACK-style storage); only its diagonal is updated.
    if (refl) {
      for (int c = j + warp; c < l; c += NWARPS) {
        double s = (lane == 0) ? v0 * R[j * l + c] : 0.0;
        for (int i = j + 1 + lane; i < l; i += 32) s += R[i * l + j] * R[i * l + c];
        s = warp_sum(s);
        const double w = tj * s;
        if (c == j) {
          if (lane == 0) R[j * l + j] = x0 - v0 * w;
        } else {
          for (int i = j + 1 + lane; i < l; i += 32) R[i * l + c] -= R[i * l + j] * w;
          if (lane == 0) R[j * l + c] -= v0 * w;
        }
      }
    }
    __syncthreads();
    // norm downdate + exact refresh of stale norms (dense.py:181-190)
    if (j + 1 < l) {
      for (int c = j + 1 + warp; c < l; c += NWARPS) {
        double nv = 0.0;
        if (lane == 0) {
          const double rj = R[j * l + c];
          nv = nrm[c] - rj * rj;
          nv = fmax(nv, 0.0);
        }
        nv = __shfl_sync(0xffffffffu, nv, 0);
        if (nv < 1e-10 * ref[c]) {
          double s = 0.0;
          for (int i = j + 1 + lane; i < l; i += 32) s += R[i * l + c] * R[i * l + c];
          s = warp_sum(s);
          if (lane == 0) { nrm[c] = s; ref[c] = s; }
        } else if (lane == 0) {
          nrm[c] = nv;
        }
      }
    }
    __syncthreads();
  }

  // explicit Q by reverse accumulation on the identity (dense.py:117-129)
  for (int idx = threadIdx.x; idx < l * l; idx += THREADS) Q[idx] = (idx / l == idx % l) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = l - 1; j >= 0; --j) {
    if (has_ref[j]) {
      const double v0 = vhead[j], tj = tau[j];
      for (int c = j + warp; c < l; c += NWARPS) {
        double s = (lane == 0) ? v0 * Q[j * l + c] : 0.0;
        for (int i = j + 1 + lane; i < l; i += 32) s += R[i * l + j] * Q[i * l + c];
        s = warp_sum(s);
        const double w = tj * s;
        for (int i = j + 1 + lane; i < l; i += 32) Q[i * l + c] -= R[i * l + j] * w;
        if (lane == 0) Q[j * l + c] -= v0 * w;
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < l * l; idx += THREADS) {
    const int i = idx / l, c = idx % l;
    T[i * ldt + c] = (c >= i) ? R[idx] : 0.0;
    qtT[c * ldq + i] = Q[idx];
  }
  for (int c = threadIdx.x; c < l; c += THREADS) {
    if (perm_out) perm_out[c] = perm[c];
    perm32[c] = perm[c];
  }
}

// ---------------------------------------------------------------- Jacobi
// One-sided Jacobi on the nv rows (length len, ld ldx) of X: orthogonalises
// them by plane rotations in the round-robin order of dense.py:200-210,
// until every pair has |<xa,xb>| <= tol |xa||xb| (dense.py:223-282).
// sig (device, nv, descending).  want_pinv: X holds B^T for an nv x nv ...
// (general: B = X^T, len x nv); writes pinv(B) (nv x len, ld ldp) with the
// cutoff max(len, nv) * sig0 * 1e-12 (dense.py:390-402).
__global__ void __launch_bounds__(THREADS, 1)
    jacobi_kernel(const double* __restrict__ X, int nv, int len, int64_t ldx, double tol,
                  int max_sweeps, double* sig_out, double* pinv, int64_t ldp, double* gwork,
                  int use_smem, int* status) {
  extern __shared__ double dsm[];
  __shared__ int pair_a[LMAX / 2 + 1], pair_b[LMAX / 2 + 1];
  __shared__ double offmax[NWARPS];
  __shared__ double sig[LMAX];
  __shared__ int order[LMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = nv + (nv > 1 && (nv & 1));  // pad odd counts with a zero row
  const bool want_v = pinv != nullptr;
  double* W = use_smem ? dsm : gwork;          // n x len
  double* V = W + (int64_t)n * len;            // n x n (row a = column a of V)
  for (int64_t idx = threadIdx.x; idx < (int64_t)n * len; idx += THREADS) {
    const int r = idx / len, c = idx % len;
    W[idx] = (r < nv) ? X[r * ldx + c] : 0.0;
  }
  if (want_v)
    for (int64_t idx = threadIdx.x; idx < (int64_t)n * n; idx += THREADS)
      V[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
  __syncthreads();
  int st = 0;
  if (n > 1) {
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
      double off = 0.0;
      for (int round = 0; round < n - 1; ++round) {
        // round-robin pairing: ring[0] fixed, others rotate
        if (threadIdx.x < n / 2) {
          const int t = threadIdx.x;
          auto ring = [&](int pos) -> int {
            if (pos == 0) return 0;
            int q = (pos - 1 - round) % (n - 1);
            if (q < 0) q += n - 1;
            return 1 + q;
          };
          pair_a[t] = ring(t);
          pair_b[t] = ring(n - 1 - t);
        }
        __syncthreads();
        for (int pi = warp; pi < n / 2; pi += NWARPS) {
          const int a = pair_a[pi], b = pair_b[pi];
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
      // block max of off
      double m = off;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) offmax[warp] = m;
      __syncthreads();
      if (threadIdx.x == 0) {
        double mm = 0.0;
        for (int w = 0; w < NWARPS; ++w) mm = fmax(mm, offmax[w]);
        offmax[0] = mm;
      }
      __syncthreads();
      const bool done = offmax[0] <= tol;
      __syncthreads();
      if (done) break;
    }
    if (sweep == max_sweeps) st = 1;
  }
  // singular values and stable descending order (dense.py:339-341)
  for (int r = warp; r < nv; r += NWARPS) {
    double s = 0.0;
    for (int i = lane; i < len; i += 32) s += W[(int64_t)r * len + i] * W[(int64_t)r * len + i];
    s = warp_sum(s);
    if (lane == 0) sig[r] = sqrt(s);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nv; r += THREADS) {
    int rank = 0;
    for (int q = 0; q < nv; ++q) rank += (sig[q] > sig[r]) || (sig[q] == sig[r] && q < r);
    order[rank] = r;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nv; k += THREADS) sig_out[k] = sig[order[k]];
  if (want_v) {
    // B = X^T = U S V^T with U[:, k] = W[k] / sig_k.  pinv = V S^+ U^T.
    const double s0 = sig[order[0]];
    const double cut = (double)max(len, nv) * s0 * 1e-12;
    for (int64_t idx = threadIdx.x; idx < (int64_t)nv * len; idx += THREADS) {
      const int i = idx / len, j = idx % len;
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
  if (threadIdx.x == 0 && status) *status = st;
}

}  // namespace small
