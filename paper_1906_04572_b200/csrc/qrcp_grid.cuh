// Grid QRCP: Businger-Golub column-pivoted Householder QR (dense.py:152-192)
// of an m x n matrix too large for one thread-block cluster's shared memory
// (cores l > 640, the harness's full-matrix "qrcp" method, rectangular
// inputs).  One cooperative launch; the matrix lives column-major in an
// L2-resident global scratch R (a 1000 x 1000 core is 8 MB of the 126 MB L2).
//
// Column c is owned by global warp c % (gridDim.x * NW): every update,
// downdate and refresh of a column is done by its owner alone, so the only
// cross-CTA traffic per pivot step is
//   * one grid barrier,
//   * each CTA's pivot candidate (max downdated norm^2, lowest LOGICAL
//     position on ties -- the position the reference's physical swaps give
//     the column), double-buffered by step parity,
//   * the pivot column, read by every CTA into shared memory.
// Every CTA then reduces the candidates, swaps its own copy of the
// logical<->physical maps and computes the reflector (v0, tau) with the same
// thread->data mapping, so all CTAs agree bit for bit.  The pivot column is
// never modified after it is chosen: rows j+1.. keep the reflector tail and
// the new diagonal goes to diag[].  Explicit Q (dense.py:117-129) needs no
// barrier at all: column c of Q is transformed only by H_j with j <= c, by
// its owner warp, reading the (read-only) reflectors from L2.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace qg {

namespace cg = cooperative_groups;

constexpr int THREADS = 256;
constexpr int NW = THREADS / 32;

struct Params {
  const double* a;      // m x n row-major input (ld lda)
  int64_t lda;
  int m, n, k;          // k = min(m, n)
  double* R;            // m x n column-major scratch (ld m)
  double* nrm;          // n: downdated column norms^2 (owner warp only)
  double* ref;          // n: reference norms^2 of the last exact refresh
  int* done;            // n: column already pivoted
  double* cand_v;       // 2 x gridDim.x candidates (value)
  int* cand_q;          // 2 x gridDim.x candidates (logical position)
  double* diag;         // k: R_jj
  double* tau;          // k
  double* vhead;        // k: v0 of reflector j
  int* has_ref;         // k: reflector j exists (nonzero column)
  double* T;            // k x n row-major (ld ldt), upper; rows >= kend zero
  int64_t ldt;
  double* qtT;          // k x m: row c = column c of Q (ld ldq)
  int64_t ldq;
  long long* perm_out;  // n (nullable)
  int* perm32;          // n
  double delta;         // >= 0: ALM truncation (see small.cuh qrcp_body)
  int* r_out;           // #(|diag| > delta), or kend when delta < 0 (nullable)
};

__host__ __device__ inline size_t smem_bytes(int m, int n) {
  return (size_t)m * 8 + (size_t)2 * n * 4 + 16;
}

__device__ __forceinline__ void better(double& bv, int& bq, double v, int q) {
  if (v > bv || (v == bv && q < bq)) {
    bv = v;
    bq = q;
  }
}

// this CTA's best active owned column (by logical position) -> slot `par`
__device__ void candidate(const Params& P, const int* p2l, int par, double* wv, int* wq) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int GW = gridDim.x * NW, gw = blockIdx.x * NW + warp;
  double bv = -1.0;
  int bq = P.n;
  for (int c = gw; c < P.n; c += GW)
    if (!P.done[c]) better(bv, bq, P.nrm[c], p2l[c]);  // lane-uniform (one column per warp step)
  (void)lane;
  if (lane == 0) {
    wv[warp] = bv;
    wq[warp] = bq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = -1.0;
    int q = P.n;
    for (int w = 0; w < NW; ++w) better(v, q, wv[w], wq[w]);
    P.cand_v[par * gridDim.x + blockIdx.x] = v;
    P.cand_q[par * gridDim.x + blockIdx.x] = q;
  }
}

__global__ void __launch_bounds__(THREADS) qrcp_grid_kernel(Params P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dsm[];
  double* pv = dsm;                                  // pivot column (rows j..m)
  int* l2p = reinterpret_cast<int*>(dsm + P.m);      // logical -> physical
  int* p2l = l2p + P.n;                              // physical -> logical
  __shared__ double wv[NW], red[NW];
  __shared__ int wq[NW];
  __shared__ double s_best;
  __shared__ int s_p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = gridDim.x, GW = G * NW, gw = blockIdx.x * NW + warp;
  const int m = P.m, n = P.n, k = P.k;

  // owned columns: copy, initial norms^2 (dense.py:165-166)
  for (int c = gw; c < n; c += GW) {
    double* col = P.R + (int64_t)c * m;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) {
      const double v = P.a[(int64_t)i * P.lda + c];
      col[i] = v;
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) {
      P.nrm[c] = s;
      P.ref[c] = s;
      P.done[c] = 0;
    }
  }
  for (int q = threadIdx.x; q < n; q += THREADS) {
    l2p[q] = q;
    p2l[q] = q;
  }
  __syncthreads();
  candidate(P, p2l, 0, wv, wq);

  int kend = k, rcount = 0;
  for (int j = 0; j < k; ++j) {
    const int par = j & 1;
    grid.sync();
    // global pivot: identical reduction in every CTA
    if (warp == 0) {
      double bv = -1.0;
      int bq = n;
      for (int b = lane; b < G; b += 32) better(bv, bq, P.cand_v[par * G + b], P.cand_q[par * G + b]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
        better(bv, bq, ov, oq);
      }
      if (lane == 0) {
        s_best = bv;
        s_p = bq;
      }
    }
    __syncthreads();
    const double best = s_best;
    const int p = s_p;
    // truncation: no remaining column can give |diag| > delta (small.cuh)
    if (P.delta >= 0.0 && best * 1.001 < P.delta * P.delta) {
      kend = j;
      break;
    }
    const int pc = l2p[p];
    for (int i = j + threadIdx.x; i < m; i += THREADS) pv[i] = P.R[(int64_t)pc * m + i];
    __syncthreads();  // every thread has read l2p[p] / l2p[j]
    if (threadIdx.x == 0) {
      const int cj = l2p[j];
      l2p[j] = pc;
      l2p[p] = cj;
      p2l[pc] = j;
      p2l[cj] = p;
    }
    // reflector of x = R[j:, pc] (dense.py:104-114), same order in every CTA
    double t2 = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += THREADS) t2 += pv[i] * pv[i];
    t2 = warp_sum(t2);
    if (lane == 0) red[warp] = t2;
    __syncthreads();
    t2 = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t2 += red[w];
    const double x0 = pv[j];
    const double nx = sqrt(x0 * x0 + t2);
    const bool refl = nx != 0.0;
    const double v0 = refl ? x0 + (x0 >= 0.0 ? nx : -nx) : 0.0;
    const double tj = refl ? 2.0 / (v0 * v0 + t2) : 0.0;
    const double dj = refl ? x0 - v0 * (tj * (v0 * x0 + t2)) : x0;
    rcount += (fabs(dj) > P.delta) ? 1 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      P.diag[j] = dj;
      P.tau[j] = tj;
      P.vhead[j] = v0;
      P.has_ref[j] = refl;
    }
    // owned active columns: apply H_j, downdate (dense.py:181-185), refresh
    // when stale (dense.py:185-190)
    for (int c = gw; c < n; c += GW) {
      if (c == pc || P.done[c]) continue;
      double* col = P.R + (int64_t)c * m;
      if (refl) {
        double s = (lane == 0) ? v0 * col[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) s += pv[i] * col[i];
        s = warp_sum(s);
        const double w = tj * s;
        for (int i = j + 1 + lane; i < m; i += 32) col[i] -= pv[i] * w;
        if (lane == 0) col[j] -= v0 * w;
      }
      __syncwarp();
      if (j + 1 < n) {
        const double rj = col[j];
        double nv = fmax(P.nrm[c] - rj * rj, 0.0);
        if (nv < 1e-10 * P.ref[c]) {
          double f = 0.0;
          for (int i = j + 1 + lane; i < m; i += 32) f += col[i] * col[i];
          nv = warp_sum(f);
          if (lane == 0) P.ref[c] = nv;
        }
        if (lane == 0) P.nrm[c] = nv;
      }
      __syncwarp();
    }
    if (lane == 0 && gw == pc % GW) P.done[pc] = 1;
    __syncthreads();  // map swap and this CTA's column state
    candidate(P, p2l, par ^ 1, wv, wq);
  }
  grid.sync();

  // T: logical column cq is physical column l2p[cq]
  for (int cq = gw; cq < n; cq += GW) {
    const double* col = P.R + (int64_t)l2p[cq] * m;
    for (int i = lane; i < k; i += 32)
      P.T[(int64_t)i * P.ldt + cq] = (i >= kend) ? 0.0 : ((i < cq) ? col[i] : ((i == cq) ? P.diag[i] : 0.0));
  }
  if (blockIdx.x == 0) {
    for (int q = threadIdx.x; q < n; q += THREADS) {
      if (P.perm_out) P.perm_out[q] = l2p[q];
      P.perm32[q] = l2p[q];
    }
    if (threadIdx.x == 0 && P.r_out) *P.r_out = P.delta >= 0.0 ? rcount : kend;
  }
  // explicit Q = H_0 ... H_{kend-1} I[:, :k], column by column
  for (int c = gw; c < k; c += GW) {
    double* qc = P.qtT + (int64_t)c * P.ldq;
    for (int i = lane; i < m; i += 32) qc[i] = (i == c) ? 1.0 : 0.0;
    __syncwarp();
    for (int jj = min(kend, c + 1) - 1; jj >= 0; --jj) {
      if (!P.has_ref[jj]) continue;
      const double* vj = P.R + (int64_t)l2p[jj] * m;
      const double v0 = P.vhead[jj], tj = P.tau[jj];
      double s = (lane == 0) ? v0 * qc[jj] : 0.0;
      for (int i = jj + 1 + lane; i < m; i += 32) s += vj[i] * qc[i];
      s = warp_sum(s);
      const double w = tj * s;
      for (int i = jj + 1 + lane; i < m; i += 32) qc[i] -= vj[i] * w;
      if (lane == 0) qc[jj] -= v0 * w;
      __syncwarp();
    }
  }
}

}  // namespace qg
