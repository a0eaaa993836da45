// Grid-wide one-sided Jacobi SVD for matrices whose working set does not fit
// one CTA's shared memory (the InexactALM baseline's n x n iterates, large
// jacobi_svd calls).  Same algorithm as dense.py:223-282 -- round-robin
// pairing (dense.py:200-210), cached squared column norms updated by the
// rotation identities and clamped at 0, exact refresh after every sweep,
// stop when max |<xa,xb>| / sqrt(|xa|^2 |xb|^2) <= tol over a sweep -- spread
// over a cooperative grid: one CTA per column pair (the n/2 pairs of a round
// are disjoint; the CTA's warps split the rows and reduce through shared
// memory, four 16-B loads per operand in flight per thread), one grid
// barrier per round.  Columns live as rows of W
// (length len, 16-B aligned, ld even) and rotations of V as rows of V, both
// in global memory: a 1000 x 1000 problem is 16 MB, L2-resident.  No
// __restrict__ / read-only loads here: every buffer is rewritten by other
// CTAs between grid barriers.
//
// After convergence the same launch computes sigma, the stable descending
// order (dense.py:339-341), the sorted factors (rows of ut / vt) and the
// zero-sigma completion of the left factor (dense.py:285-310).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "small.cuh"

namespace jg {

namespace cg = cooperative_groups;
constexpr int THREADS = 128;

__device__ __forceinline__ double row_dot(const double* a, const double* b, int len,
                                          int lane) {
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double s0 = 0.0, s1 = 0.0;
  const int h = len >> 1;
  for (int i = lane; i < h; i += 32) {
    const double2 x = a2[i], y = b2[i];
    s0 += x.x * y.x;
    s1 += x.y * y.y;
  }
  if ((len & 1) && lane == 0) s0 += a[len - 1] * b[len - 1];
  return warp_sum(s0 + s1);
}

__device__ __forceinline__ void row_rotate(double* a, double* b, int len, int lane, double c, double s) {
  double2* a2 = reinterpret_cast<double2*>(a);
  double2* b2 = reinterpret_cast<double2*>(b);
  const int h = len >> 1;
  for (int i = lane; i < h; i += 32) {
    const double2 u = a2[i], v = b2[i];
    a2[i] = make_double2(c * u.x - s * v.x, c * u.y - s * v.y);
    b2[i] = make_double2(s * u.x + c * v.x, s * u.y + c * v.y);
  }
  if ((len & 1) && lane == 0) {
    const double u = a[len - 1], v = b[len - 1];
    a[len - 1] = c * u - s * v;
    b[len - 1] = s * u + c * v;
  }
}

// Block-wide dot product of two rows (all THREADS threads; result in every
// thread).  Four double2 loads per operand in flight per thread.
__device__ __forceinline__ double block_row_dot(const double* a, const double* b, int len, double* red) {
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  const int h = len >> 1;
  double s0 = 0.0, s1 = 0.0;
  for (int i0 = threadIdx.x; i0 < h; i0 += 4 * THREADS) {
    double2 x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * THREADS;
      x[u] = i < h ? a2[i] : make_double2(0.0, 0.0);
      y[u] = i < h ? b2[i] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s0 += x[u].x * y[u].x;
      s1 += x[u].y * y[u].y;
    }
  }
  if ((len & 1) && threadIdx.x == 0) s0 += a[len - 1] * b[len - 1];
  const double w = warp_sum(s0 + s1);
  __syncthreads();  // red[] is reused across calls
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < THREADS / 32; ++k) t += red[k];
  return t;
}

__device__ __forceinline__ void block_row_rotate(double* a, double* b, int len, double c, double s) {
  double2* a2 = reinterpret_cast<double2*>(a);
  double2* b2 = reinterpret_cast<double2*>(b);
  const int h = len >> 1;
  for (int i0 = threadIdx.x; i0 < h; i0 += 4 * THREADS) {
    double2 u[4], v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k * THREADS;
      if (i < h) {
        u[k] = a2[i];
        v[k] = b2[i];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k * THREADS;
      if (i < h) {
        a2[i] = make_double2(c * u[k].x - s * v[k].x, c * u[k].y - s * v[k].y);
        b2[i] = make_double2(s * u[k].x + c * v[k].x, s * u[k].y + c * v[k].y);
      }
    }
  }
  if ((len & 1) && threadIdx.x == 0) {
    const double u = a[len - 1], v = b[len - 1];
    a[len - 1] = c * u - s * v;
    b[len - 1] = s * u + c * v;
  }
}

// W: n x len (ld ldw), rows nv..n-1 zero (odd nv padded to even n);
// V: n x n (ld ldv) scratch, set to I here.  offs: max_sweeps zeroed slots.
// Outputs: sig_out[nv] descending; ut_out row k = column order[k] / sigma;
// vt_out row k = rotation column order[k] (first nv entries).
// status[0]: 0 ok, 1 no convergence, 2 completion ran out; status[1]: sweeps.
__global__ void __launch_bounds__(THREADS) jacobi_grid_kernel(
    double* W, int64_t ldw, double* V, int64_t ldv, int nv, int n, int len, double tol,
    int max_sweeps, double* nrm, unsigned long long* offs, double* sig,
    int* order, double* sig_out, double* ut_out, int64_t ldut,
    double* vt_out, int64_t ldvt, int* status) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[THREADS / 32];
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int ntot = gridDim.x * blockDim.x;
  const bool want_v = vt_out != nullptr;
  if (want_v)
    for (int r = gw; r < n; r += nw)
      for (int c = lane; c < n; c += 32) V[r * ldv + c] = (r == c) ? 1.0 : 0.0;
  for (int c = gw; c < n; c += nw) {
    const double s = row_dot(W + c * ldw, W + c * ldw, len, lane);
    if (lane == 0) nrm[c] = s;
  }
  grid.sync();
  int st = 0, sweeps = 0;
  if (n > 1) {
    st = 1;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
      double off = 0.0;
      for (int round = 0; round < n - 1; ++round) {
        // one CTA per pair: the CTA's warps share the row (block reduce)
        for (int pi = blockIdx.x; pi < n / 2; pi += gridDim.x) {
          // ring position -> player (dense.py:200-210): position 0 fixed
          auto ring = [&](int pos) -> int {
            if (pos == 0) return 0;
            int q = (pos - 1 - round) % (n - 1);
            if (q < 0) q += n - 1;
            return 1 + q;
          };
          const int a = ring(pi), b = ring(n - 1 - pi);
          double* xa = W + a * ldw;
          double* xb = W + b * ldw;
          const double al = nrm[a], be = nrm[b];
          const double ga = block_row_dot(xa, xb, len, red);
          const double den = sqrt(al * be);
          const double rel = den > 0.0 ? fabs(ga) / den : 0.0;
          off = fmax(off, rel);
          if (rel > tol) {
            // np.sign: an exact tie (al == be) gives t = 0, no rotation
            const double zeta = (be - al) / (2.0 * ga);
            const double sgn = zeta > 0.0 ? 1.0 : (zeta < 0.0 ? -1.0 : 0.0);
            const double t = sgn / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t);
            const double s = c * t;
            block_row_rotate(xa, xb, len, c, s);
            if (want_v) block_row_rotate(V + a * ldv, V + b * ldv, n, c, s);
            if (threadIdx.x == 0) {
              nrm[a] = fmax(al - t * ga, 0.0);
              nrm[b] = fmax(be + t * ga, 0.0);
            }
          }
        }
        grid.sync();
      }
      if (threadIdx.x == 0 && off > 0.0) atomicMax(offs + sweep, (unsigned long long)__double_as_longlong(off));
      grid.sync();
      sweeps = sweep + 1;
      const double o = __longlong_as_double((long long)*((volatile unsigned long long*)(offs + sweep)));
      if (o <= tol) {
        st = 0;
        break;
      }
      for (int c = gw; c < n; c += nw) {
        const double s = row_dot(W + c * ldw, W + c * ldw, len, lane);
        if (lane == 0) nrm[c] = s;
      }
      grid.sync();
    }
  }
  // sigma, stable descending order, sorted factors
  for (int c = gw; c < nv; c += nw) {
    const double s = row_dot(W + c * ldw, W + c * ldw, len, lane);
    if (lane == 0) sig[c] = sqrt(s);
  }
  grid.sync();
  for (int c = gt; c < nv; c += ntot) {
    const double sc = sig[c];
    int rank = 0;
    for (int q = 0; q < nv; ++q) {
      const double sq = sig[q];
      rank += (sq > sc) || (sq == sc && q < c);
    }
    order[rank] = c;
    sig_out[rank] = sc;
  }
  grid.sync();
  for (int k = gw; k < nv; k += nw) {
    const int r = order[k];
    const double sk = sig[r];
    if (ut_out)
      for (int i = lane; i < len; i += 32) ut_out[k * ldut + i] = (sk > 0.0) ? W[r * ldw + i] / sk : 0.0;
    if (want_v)
      for (int i = lane; i < nv; i += 32) vt_out[k * ldvt + i] = V[r * ldv + i];
  }
  if (ut_out) {
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x < 32 && sig_out[nv - 1] <= 0.0)
      if (small::complete_left(ut_out, ldut, sig_out, nv, len, lane)) st = 2;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    status[0] = st;
    status[1] = sweeps;
  }
}

}  // namespace jg
