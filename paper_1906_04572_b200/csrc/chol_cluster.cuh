// Cluster-parallel adaptive Cholesky step for cores l >= 64 (the one-CTA
// kernel in small.cuh handles smaller ones).  Same algorithm as
// chol_factor_kernel: blocked Cholesky of the augmented matrix
// [G (+ sI) | I], whose right half becomes R^-T (= the Bt operand of the
// X * R^-1 GEMM).  The matrix lives in L2-resident global scratch; a
// thread-block cluster of CS CTAs shares every 32-row panel:
//   (a) the diagonal block is factored redundantly in every CTA (identical
//       inputs -> identical result, nothing crosses CTAs), one panel ahead:
//       warp 0 updates and factors the next diagonal block while the other
//       warps run the trailing update (lookahead);
//   (b) the panel rows get R_kk^-T by forward substitution, a thread per
//       column;
//   (c) each CTA stages the panel with cp.async and the trailing Schur
//       update runs as 32 x 32 DMMA tiles over all warps of the cluster.
// Two cluster barriers per panel.  kappa_F sums are reduced across the
// cluster through DSMEM in rank order (deterministic).  CHOL_PROF builds
// print per-phase times (tools/ell600_probe.py with CORUTV_LIB).
#pragma once
#include <cooperative_groups.h>

#include "small.cuh"

namespace chc {

namespace cg = cooperative_groups;
using small::CholInfo;
using small::NB;

constexpr int THREADS = 256;

#ifdef CHOL_PROF
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CHOL_T(i) if (rank == 0 && tid == 0) tp[i] = gtime();
#else
#define CHOL_T(i)
#endif

// shared memory (doubles): the diagonal block R_kk (32 x 33), 1/diag(R_kk),
// and the 32 panel rows staged with a padded stride (stride % 16 == 8:
// the 4 rows a DMMA fragment touches fall on different bank halves)
__host__ __device__ inline int stage_stride(int l) { return (l + 15) / 16 * 16 + 8; }
__host__ __device__ inline int smem_doubles(int l) { return 2 * 32 * 33 + 32 * stage_stride(l); }
// cores whose panel stage does not fit shared memory (l >~ 840) read the
// panel straight from the L2-resident W instead (GSTAGE): after step (b)
// the panel row kb + p, columns c0.., IS the stage row p (left block then
// right half, contiguous), so only the pointer and the stride change
__host__ __device__ inline int smem_doubles_gstage() { return 2 * 32 * 33; }

// Warp-level Cholesky of the identity-padded 32 x 32 block in Ds (upper,
// stride 33), in place, lane = column; Rinv[k] = 1 / R[k][k].  Returns the
// warp-uniform failure flag (non-positive or non-finite pivot).
__device__ bool factor_diag32(double* Ds, double* Rinv) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  for (int j = 0; j < 32; ++j) {
    const double d = Ds[j * 33 + j];
    bad |= !(d > 0.0) || !isfinite(d);
    // one reciprocal square root per step instead of a sqrt and a division
    // per lane: the step's latency chain is the factor's critical path
    const double ri = rsqrt(d);
    const double rjk = (lane > j) ? Ds[j * 33 + lane] * ri : d * ri;
    __syncwarp();
    if (lane >= j) Ds[j * 33 + lane] = rjk;
    __syncwarp();
    // all loads of the step first (stores could alias them), then the
    // rank-1 update of column `lane`
    double rowj[32], colv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      rowj[i] = Ds[j * 33 + i];
      colv[i] = Ds[i * 33 + lane];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i > j && lane >= i) Ds[i * 33 + lane] = fma(-rowj[i], rjk, colv[i]);
    __syncwarp();
  }
  Rinv[lane] = 1.0 / Ds[lane * 33 + lane];
  __syncwarp();
  return bad;
}

// Blocked right-looking Cholesky of the augmented [G | I] (l x 2l, global,
// L2-resident, ld = 2l), panels of 32 rows, over a thread-block cluster:
//  (a) every CTA loads the 32 x 32 diagonal block into shared memory; its
//      warp 0 factors it (lane = column, rank-1 updates) and inverts the
//      factor (lane = column, back substitution) -- identical inputs give
//      identical results in every CTA, so nothing crosses CTAs;
//  (b) the panel rows become R_kk^-T times themselves: a thread per column
//      multiplies by the explicit inverse (no sequential division chain);
//  (c) each CTA stages the transformed panel rows (one cluster barrier
//      after (b)) and the trailing Schur update W -= P' P runs as 32 x 32
//      DMMA tiles (K = 32) spread over every warp of the cluster: the upper
//      triangle of the left block and the nonzero band of the right half.
// Two cluster barriers per panel.
template <bool GSTAGE>
__device__ bool chol_aug_cluster(cg::cluster_group& cluster, double* W, int l, double* smem, int* s_flag) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int nwarp = nt >> 5;
  const int ld = 2 * l;
  const int wp = GSTAGE ? ld : stage_stride(l);
  double* Ds = smem;             // R_kk (upper), 32 x 33
  double* Rinv = smem + 32 * 33;  // 1 / diag(R_kk)

  double* stage = smem + 2 * 32 * 33;
  const int r8 = lane >> 2, c4 = lane & 3;
#ifdef CHOL_PROF
  unsigned long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long acc_t[6] = {0, 0, 0, 0, 0, 0};
#endif
  // prologue: the first diagonal block (later ones are factored one panel
  // ahead, by warp 0 while the other warps run the trailing update)
  {
    const int nb0 = min(NB, l);
    for (int e = tid; e < 32 * 32; e += nt) {
      const int i = e >> 5, k = e & 31;
      double v;
      if (i < nb0 && k < nb0) v = (k >= i) ? W[(int64_t)i * ld + k] : 0.0;
      else v = (i == k) ? 1.0 : 0.0;
      Ds[i * 33 + k] = v;
    }
    __syncthreads();
    if (warp == 0) {
      const bool bad = factor_diag32(Ds, Rinv);
      if (lane == 0) *s_flag = bad ? 1 : 0;
    }
  }
  for (int kb = 0; kb < l; kb += NB) {
    const int nb = min(NB, l - kb);
    CHOL_T(0)
    __syncthreads();
    CHOL_T(1)
    if (*s_flag) return true;  // identical in every CTA
    if (rank == 0)
      for (int e = tid; e < nb * nb; e += nt) {
        const int i = e / nb, k = e % nb;
        if (k >= i) W[(int64_t)(kb + i) * ld + kb + k] = Ds[i * 33 + k];
      }
    const int c0 = kb + nb;
    const int nleft = l - c0, nright = kb + nb, ncols = nleft + nright;
    // (b) panel rows := R_kk^-T panel rows: a thread per column, forward
    // substitution with R_kk' (backward stable, the unblocked step's
    // arithmetic); the column lives in registers, R_kk rows are shared-
    // memory broadcasts (a compiler barrier per row bounds load hoisting)
    for (int t = rank * nt + tid; t < ncols; t += CS * nt) {
      const int64_t col = (t < nleft) ? c0 + t : l + (t - nleft);
      double x[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) x[q] = (q < nb) ? W[(int64_t)(kb + q) * ld + col] : 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        double sacc = x[i];
#pragma unroll
        for (int q = 0; q < i; ++q) sacc -= Ds[q * 33 + i] * x[q];
        x[i] = sacc * Rinv[i];
        asm volatile("" ::: "memory");
      }
#pragma unroll
      for (int i = 0; i < NB; ++i)
        if (i < nb) W[(int64_t)(kb + i) * ld + col] = x[i];
    }
    CHOL_T(2)
    cluster.sync();
    CHOL_T(3)
    if (c0 >= l) break;
    // (c) stage the panel (rows >= nb zero) with asynchronous 8-byte copies
    // (all of a thread's loads in flight at once), then update the trailing
    // matrix.  GSTAGE: the panel rows in W are the stage (nb == 32 here:
    // only the last panel is short, and it ends the loop above)
    if (GSTAGE) stage = W + (int64_t)kb * ld + c0;
    for (int e = tid; !GSTAGE && e < 32 * ncols; e += nt) {
      const int p = e / ncols, t = e % ncols;
      if (p < nb) {
        const int64_t col = (t < nleft) ? c0 + t : l + (t - nleft);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(stage + p * wp + t)),
                     "l"(W + (int64_t)(kb + p) * ld + col)
                     : "memory");
      } else {
        stage[p * wp + t] = 0.0;
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    const int TI = (nleft + 31) / 32, TR = (nright + 31) / 32;
    const int nup = TI * (TI + 1) / 2;
    if (warp == 0) {
      // lookahead: the next diagonal block = its current W values (tile 0 of
      // the update is left to this warp, so nobody else touches it) minus
      // the panel's contribution, then factored for the next iteration
      const int nbn = min(NB, nleft);
      // P' P for the 32 x 32 block on the tensor pipe (same fragments as
      // the update tiles, srow = scol = 0)
      double acc[4][4][2];
#pragma unroll
      for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) acc[a2][b2][0] = acc[a2][b2][1] = 0.0;
#pragma unroll
      for (int p0 = 0; p0 < 32; p0 += 4) {
        const double* row = stage + (p0 + c4) * wp;
        double av[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) av[mi] = (mi * 8 + r8 < nleft) ? row[mi * 8 + r8] : 0.0;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], av[mi], av[nj]);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = mi * 8 + r8, k = nj * 8 + 2 * c4 + e;
            double v;
            if (i < nbn && k < nbn) v = (k >= i) ? W[(int64_t)(c0 + i) * ld + c0 + k] - acc[mi][nj][e] : 0.0;
            else v = (i == k) ? 1.0 : 0.0;
            Ds[i * 33 + k] = v;
          }
      __syncwarp();
      const bool bad = factor_diag32(Ds, Rinv);
      if (lane == 0) *s_flag = bad ? 1 : 0;
    }
    const int uw = rank * (nwarp - 1) + (warp - 1), uwn = CS * (nwarp - 1);
    for (int tile = (warp == 0) ? nup + TI * TR : uw; tile < nup + TI * TR; tile += uwn) {
      if (tile == 0) continue;  // the next diagonal block (lookahead above)
      int ti, tk;
      bool left;
      if (tile < nup) {
        tk = (int)((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
        while ((tk + 1) * (tk + 2) / 2 <= tile) ++tk;
        while (tk * (tk + 1) / 2 > tile) --tk;
        ti = tile - tk * (tk + 1) / 2;
        left = true;
      } else {
        ti = (tile - nup) / TR;
        tk = (tile - nup) % TR;
        left = false;
      }
      const int srow = 32 * ti;                              // stage column of the tile's rows
      const int scol = left ? 32 * tk : nleft + 32 * tk;     // stage column of the tile's columns
      const int slim = left ? nleft : ncols;
      double acc[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
      for (int p0 = 0; p0 < 32; p0 += 4) {
        const double* row = stage + (p0 + c4) * wp;
        double av[4], bv[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int sc = srow + mi * 8 + r8;
          av[mi] = (sc < nleft) ? row[sc] : 0.0;
        }
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) {
          const int sc = scol + nj * 8 + r8;
          bv[nj] = (sc < slim) ? row[sc] : 0.0;
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 4; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], av[mi], bv[nj]);
      }
      // read-modify-write of the tile: every old value is loaded before any
      // store (stores could alias later loads), so the 32 L2 reads overlap
      auto elem = [&](int mi, int nj, int e) -> double* {
        const int i = c0 + srow + mi * 8 + r8;
        const int sc = scol + nj * 8 + 2 * c4 + e;
        if (i >= l || sc >= slim || (left && c0 + sc < i)) return nullptr;
        return left ? W + (int64_t)i * ld + c0 + sc : W + (int64_t)i * ld + l + (sc - nleft);
      };
      double old[4][4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double* q = elem(mi, nj, e);
            old[mi][nj][e] = q ? *q : 0.0;
          }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 4; ++nj)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (double* q = elem(mi, nj, e)) *q = old[mi][nj][e] - acc[mi][nj][e];
    }
    CHOL_T(4)
    cluster.sync();
    CHOL_T(5)
#ifdef CHOL_PROF
    if (rank == 0 && tid == 0)
      for (int q = 0; q < 5; ++q) acc_t[q] += tp[q + 1] - tp[q];
#endif
  }
#ifdef CHOL_PROF
  if (rank == 0 && tid == 0)
    printf("chol l=%d CS=%d: diag-sync %.1f us, trsm %.1f us, sync1 %.1f us, update+lookahead %.1f us, sync2 %.1f us\n", l, CS,
           acc_t[0] * 1e-3, acc_t[1] * 1e-3, acc_t[2] * 1e-3, acc_t[3] * 1e-3, acc_t[4] * 1e-3);
#endif
  return false;
}

// cluster-wide deterministic sum: every CTA gets sum_r part_r in rank order
__device__ double cluster_sum(cg::cluster_group& cluster, double v, double* slot, double* red) {
  v = small::block_sum(v, red);
  if (threadIdx.x == 0) *slot = v;
  cluster.sync();
  double s = 0.0;
  for (int r = 0; r < (int)cluster.num_blocks(); ++r) s += *cluster.map_shared_rank(slot, r);
  cluster.sync();
  return s;
}

template <bool GSTAGE>
__global__ void __launch_bounds__(THREADS, 1)
    chol_factor_cluster_kernel(const double* __restrict__ G, int l, int64_t ldg, double shift_coeff,
                               int allow_plain, double kappa_max, double* __restrict__ rinvT,
                               int64_t ldr, double* W, CholInfo* info) {
  extern __shared__ double dsm[];
  __shared__ double red[32];
  __shared__ double slot;
  __shared__ int s_flag;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int gt = rank * blockDim.x + threadIdx.x, gn = CS * blockDim.x;
  const int ld = 2 * l;
  double tr = 0.0;
  for (int i = threadIdx.x; i < l; i += blockDim.x) tr += G[i * ldg + i];
  tr = small::block_sum(tr, red);  // identical in every CTA
  int shifted = allow_plain ? 0 : 1;
  int status = 0;
  double kappa = 1.0;
  if (!(tr > 0.0) || !isfinite(tr)) {
    for (int64_t e = gt; e < (int64_t)l * l; e += gn) {
      const int i = (int)(e / l), k = (int)(e % l);
      W[(int64_t)i * ld + l + k] = (i == k) ? 1.0 : 0.0;
    }
    status = isfinite(tr) ? 1 : 2;
    cluster.sync();
  } else {
    for (;;) {
      const double s = shifted ? shift_coeff * tr : 0.0;
      for (int64_t e = gt; e < (int64_t)l * 2 * l; e += gn) {
        const int i = (int)(e / (2 * l)), k = (int)(e % (2 * l));
        double g;
        if (k < l) {
          g = (k >= i) ? G[i * ldg + k] : 0.0;
          if (i == k) g += s;
        } else {
          g = (k - l == i) ? 1.0 : 0.0;
        }
        W[(int64_t)i * ld + k] = g;
      }
      cluster.sync();
      const bool fail = chol_aug_cluster<GSTAGE>(cluster, W, l, dsm, &s_flag);
      cluster.sync();
      if (fail) {
        if (!shifted) { shifted = 1; continue; }
        status = 2;
        break;
      }
      double nr = 0.0, ni = 0.0;
      for (int64_t e = gt; e < (int64_t)l * l; e += gn) {
        const int i = (int)(e / l), k = (int)(e % l);
        const double a = (k >= i) ? W[(int64_t)i * ld + k] : 0.0;
        const double b = (k <= i) ? W[(int64_t)i * ld + l + k] : 0.0;
        nr += a * a;
        ni += b * b;
      }
      nr = cluster_sum(cluster, nr, &slot, red);
      ni = cluster_sum(cluster, ni, &slot, red);
      kappa = sqrt(nr) * sqrt(ni);
      if (!shifted && !(kappa <= kappa_max)) { shifted = 1; continue; }
      break;
    }
  }
  for (int64_t e = gt; e < (int64_t)l * l; e += gn) {
    const int j = (int)(e / l), k = (int)(e % l);
    rinvT[j * ldr + k] = (k <= j) ? W[(int64_t)j * ld + l + k] : 0.0;
  }
  if (rank == 0 && threadIdx.x == 0) {
    info->shifted = shifted;
    info->status = status;
    info->kappa = kappa;
    info->trace = tr;
  }
  cluster.sync();
}

}  // namespace chc
