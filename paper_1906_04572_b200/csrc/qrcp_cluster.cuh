// Cluster QRCP: Businger-Golub column-pivoted Householder QR of the l x l
// compressed core (dense.py:152-192) spread over a thread-block cluster of
// CS CTAs (CS <= 16).  CTA r owns physical columns [r*cw, (r+1)*cw) in its
// shared memory (column-major, so a warp's lanes stride down a column); the
// whole core stays on chip for l <= 640 (16 x 205 KB).
//
// Per pivot step j (ONE cluster barrier):
//   1. each CTA finds its best (downdated norm, lowest logical position) and
//      stores it into every CTA's candidate slot (DSMEM st, slots
//      double-buffered by step parity);  cluster barrier;
//   2. every CTA reduces the CS candidates identically -> pivot p / column pc,
//      copies column pc (rows j..l) from its owner over DSMEM, and computes
//      the reflector (v0, tau) redundantly and bit-identically;
//   3. warp per owned active column: dot, update, norm downdate and exact
//      refresh when stale (dense.py:181-190).
// Columns never move; a replicated logical->physical map keeps the
// lowest-logical-index tie-break.  The new diagonal of the pivot column goes
// to diag[] so the owner never modifies a column another CTA is reading.
// Explicit Q (dense.py:117-129): reflectors are read-only after the
// factorization, so each CTA accumulates its own Q columns with only CTA
// barriers, fetching v_j from its owner over DSMEM.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace qc {

namespace cg = cooperative_groups;

constexpr int THREADS = 1024;
constexpr int NW = THREADS / 32;
constexpr int LMAX = 640;
constexpr int MAXCW = 64;  // columns owned per CTA (host picks CS accordingly)

struct Shared {
  double nrm[MAXCW], ref[MAXCW];
  int done[MAXCW];
  double cand_v[2][16];
  int cand_q[2][16];
  int l2p[2][LMAX];
  double pv[LMAX];
  double tau[LMAX], vhead[LMAX], diag[LMAX];
  int has_ref[LMAX];
};

// dyn smem: R cols [cw][l], then (optional) Q cols [cw][l]
__global__ void __launch_bounds__(THREADS, 1)
    qrcp_cluster_kernel(const double* __restrict__ D, int l, int64_t ldd, int cw,
                        double* __restrict__ T, int64_t ldt, double* __restrict__ qtT, int64_t ldq,
                        long long* perm_out, int* perm32, double* qglobal, int q_in_smem, double delta,
                        int* r_out) {
  extern __shared__ double dsm[];
  __shared__ Shared sh;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int CS = (int)cluster.num_blocks();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c_lo = rank * cw;
  const int nown = max(0, min(cw, l - c_lo));
  double* Rl = dsm;                                             // [cw][l]
  double* Ql = q_in_smem ? dsm + (size_t)cw * l : qglobal + (size_t)rank * cw * l;

  // load owned columns of D (column-major), norms, maps
  for (int cl = warp; cl < nown; cl += NW) {
    const int c = c_lo + cl;
    double s = 0.0;
    for (int i = lane; i < l; i += 32) {
      const double v = D[i * ldd + c];
      Rl[cl * l + i] = v;
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) {
      sh.nrm[cl] = s;
      sh.ref[cl] = s;
      sh.done[cl] = 0;
    }
  }
  for (int q = threadIdx.x; q < l; q += THREADS) sh.l2p[0][q] = q;
  cluster.sync();

  int kend = l;
  int rcount = 0;  // #(|diag T| > delta) over the steps taken (rpca.py:123-124)
  for (int j = 0; j < l; ++j) {
    const int par = j & 1;
    const int* cur = sh.l2p[par];
    int* nxt = sh.l2p[par ^ 1];
    // 1. local candidate: first logical position of the max norm among owned
    if (warp == 0) {
      double best = -1.0;
      int bq = l;
      for (int q = j + lane; q < l; q += 32) {
        const int c = cur[q];
        if (c >= c_lo && c < c_lo + nown) {
          const double v = sh.nrm[c - c_lo];
          if (v > best) { best = v; bq = q; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
        if (ov > best || (ov == best && oq < bq)) { best = ov; bq = oq; }
      }
      if (lane < CS) {
        Shared* rs = cluster.map_shared_rank(&sh, lane);
        rs->cand_v[par][rank] = best;
        rs->cand_q[par][rank] = bq;
      }
    }
    cluster.sync();
    // 2. global pivot (identical in every CTA)
    double best = -1.0;
    int bq = l;
    for (int r = 0; r < CS; ++r) {
      const double v = sh.cand_v[par][r];
      const int q = sh.cand_q[par][r];
      if (v > best || (v == best && q < bq)) { best = v; bq = q; }
    }
    // truncation: stop once no remaining column can give |diag T| > delta
    // (small.cuh qrcp_body; identical in every CTA)
    if (delta >= 0.0 && best * 1.001 < delta * delta) {
      kend = j;
      break;
    }
    const int p = bq;
    const int pc = cur[p];
    const int owner = pc / cw;
    {
      const double* src = cluster.map_shared_rank(Rl, owner) + (size_t)(pc - owner * cw) * l;
      for (int i = j + threadIdx.x; i < l; i += THREADS) sh.pv[i] = src[i];
    }
    for (int q = threadIdx.x; q < l; q += THREADS) nxt[q] = (q == j) ? cur[p] : ((q == p) ? cur[j] : cur[q]);
    __syncthreads();
    // reflector (dense.py:104-114), every warp identically
    const double x0 = sh.pv[j];
    double t2 = 0.0;
    for (int i = j + 1 + lane; i < l; i += 32) t2 += sh.pv[i] * sh.pv[i];
    t2 = warp_sum(t2);
    const double nx = sqrt(x0 * x0 + t2);
    const bool refl = nx != 0.0;
    const double v0 = refl ? x0 + (x0 >= 0.0 ? nx : -nx) : 0.0;
    const double tj = refl ? 2.0 / (v0 * v0 + t2) : 0.0;
    const double dj = refl ? x0 - v0 * (tj * (v0 * x0 + t2)) : x0;
    rcount += (fabs(dj) > delta) ? 1 : 0;
    if (threadIdx.x == 0) {
      sh.diag[j] = dj;
      sh.tau[j] = tj;
      sh.vhead[j] = v0;
      sh.has_ref[j] = refl;
    }
    // 3. owned active columns: warp per column
    for (int cl = warp; cl < nown; cl += NW) {
      const int c = c_lo + cl;
      if (c == pc || sh.done[cl]) continue;
      double* col = Rl + (size_t)cl * l;
      if (refl) {
        double s = (lane == 0) ? v0 * col[j] : 0.0;
        for (int i = j + 1 + lane; i < l; i += 32) s += sh.pv[i] * col[i];
        s = warp_sum(s);
        const double w = tj * s;
        for (int i = j + 1 + lane; i < l; i += 32) col[i] -= sh.pv[i] * w;
        if (lane == 0) col[j] -= v0 * w;
      }
      __syncwarp();
      if (j + 1 < l) {
        const double rj = col[j];
        double nv = fmax(sh.nrm[cl] - rj * rj, 0.0);
        if (nv < 1e-10 * sh.ref[cl]) {
          double f = 0.0;
          for (int i = j + 1 + lane; i < l; i += 32) f += col[i] * col[i];
          f = warp_sum(f);
          nv = f;
          if (lane == 0) sh.ref[cl] = f;
        }
        if (lane == 0) sh.nrm[cl] = nv;
      }
    }
    if (threadIdx.x == 0 && pc >= c_lo && pc < c_lo + nown) sh.done[pc - c_lo] = 1;
    __syncthreads();
  }
  cluster.sync();
  const int* fin = sh.l2p[kend & 1];

  // outputs owned by this CTA: T columns whose pivot column it owns, perm
  for (int cq = warp; cq < l; cq += NW) {
    const int c = fin[cq];
    if (c < c_lo || c >= c_lo + nown) continue;
    const double* col = Rl + (size_t)(c - c_lo) * l;
    for (int i = lane; i < l; i += 32)
      T[i * ldt + cq] = (i >= kend) ? 0.0 : ((i < cq) ? col[i] : ((i == cq) ? sh.diag[cq] : 0.0));
  }
  if (rank == 0) {
    for (int c = threadIdx.x; c < l; c += THREADS) {
      if (perm_out) perm_out[c] = fin[c];
      perm32[c] = fin[c];
    }
    if (threadIdx.x == 0 && r_out) *r_out = delta >= 0.0 ? rcount : kend;
  }

  // explicit Q: this CTA's Q columns [c_lo, c_lo + nown)
  for (int cl = warp; cl < nown; cl += NW)
    for (int i = lane; i < l; i += 32) Ql[(size_t)cl * l + i] = (i == c_lo + cl) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = kend - 1; j >= 0; --j) {
    if (!sh.has_ref[j]) continue;  // uniform
    if (c_lo + nown <= j) continue;  // no owned column c >= j (uniform)
    const int pc = fin[j];
    const int owner = pc / cw;
    const double* src = cluster.map_shared_rank(Rl, owner) + (size_t)(pc - owner * cw) * l;
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < l; i += THREADS) sh.pv[i] = src[i];
    __syncthreads();
    const double v0 = sh.vhead[j], tj = sh.tau[j];
    for (int cl = warp; cl < nown; cl += NW) {
      if (c_lo + cl < j) continue;
      double* col = Ql + (size_t)cl * l;
      double s = (lane == 0) ? v0 * col[j] : 0.0;
      for (int i = j + 1 + lane; i < l; i += 32) s += sh.pv[i] * col[i];
      s = warp_sum(s);
      const double w = tj * s;
      for (int i = j + 1 + lane; i < l; i += 32) col[i] -= sh.pv[i] * w;
      if (lane == 0) col[j] -= v0 * w;
    }
  }
  __syncthreads();
  // qtT[c][i] = Q[i][c]: row c of qtT is this CTA's column
  for (int cl = warp; cl < nown; cl += NW)
    for (int i = lane; i < l; i += 32) qtT[(size_t)(c_lo + cl) * ldq + i] = Ql[(size_t)cl * l + i];
  cluster.sync();  // keep shared memory alive until every remote read is done
}

}  // namespace qc
