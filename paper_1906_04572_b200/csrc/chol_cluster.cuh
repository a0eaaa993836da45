// Cluster-parallel adaptive Cholesky step for large cores (l > 113, where
// [G | I] no longer fits one CTA's shared memory).  Same algorithm as
// chol_factor_kernel (small.cuh): blocked Cholesky of the augmented matrix
// [G (+ sI) | I], whose right half becomes R^-T (= the Bt operand of the
// X * R^-1 GEMM).  The matrix lives in L2-resident global scratch; a
// thread-block cluster of CS CTAs shares every panel step:
//   (a) every CTA's warp 0 factors the 32 x 32 diagonal block redundantly
//       in registers (identical inputs -> identical result, so no flag or
//       factor needs to cross CTAs); rank 0 writes it back;
//   (b) the panel's forward substitution is split over all cluster threads;
//   (c) each CTA stages the panel rows in its shared memory and updates its
//       share of the trailing 4 x 4 tiles.
// Two cluster barriers per 32-row panel.  kappa_F sums are reduced across
// the cluster through DSMEM in rank order (deterministic).
#pragma once
#include <cooperative_groups.h>

#include "small.cuh"

namespace chc {

namespace cg = cooperative_groups;
using small::CholInfo;
using small::NB;

constexpr int THREADS = 512;

__device__ bool chol_aug_cluster(cg::cluster_group& cluster, double* W, int l, double* Dsm,
                                 double* stage, int* s_flag) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int gt = rank * nt + tid, gn = CS * nt;
  const int ld = 2 * l;
  for (int kb = 0; kb < l; kb += NB) {
    const int nb = min(NB, l - kb);
    if (warp == 0) {
      double c[32];
      const bool bad =
          small::warp_chol32(c, nb, [&](int i, int k) { return W[(int64_t)(kb + i) * ld + kb + k]; });
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        Dsm[i * 32 + lane] = (i <= lane) ? c[i] : 0.0;
        if (rank == 0 && i <= lane && lane < nb) W[(int64_t)(kb + i) * ld + kb + lane] = c[i];
      }
      if (lane == 0) *s_flag = bad ? 1 : 0;
    }
    __syncthreads();
    if (*s_flag) return true;  // identical in every CTA
    const int c0 = kb + nb;
    const int nleft = l - c0, nright = kb + nb;
    for (int t = gt; t < nleft + nright; t += gn) {
      const int c = (t < nleft) ? c0 + t : l + (t - nleft);
      double x[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) x[i] = (i < nb) ? W[(int64_t)(kb + i) * ld + c] : 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        if (i < nb) {
          double sacc = x[i];
#pragma unroll
          for (int q = 0; q < i; ++q) sacc -= Dsm[q * 32 + i] * x[q];
          x[i] = sacc / Dsm[i * 32 + i];
        }
      }
#pragma unroll
      for (int i = 0; i < NB; ++i)
        if (i < nb) W[(int64_t)(kb + i) * ld + c] = x[i];
    }
    cluster.sync();
    if (c0 >= l) break;
    const int w = nleft + nright;
    for (int p = warp; p < nb; p += nt >> 5)
      for (int c = lane; c < w; c += 32) stage[p * w + c] = W[(int64_t)(kb + p) * ld + c0 + c];
    __syncthreads();
    const int TI = (nleft + 3) / 4;
    const int nup = TI * (TI + 1) / 2;
    const int TR = (nright + 3) / 4;
    for (int t = gt; t < nup + TI * TR; t += gn) {
      if (t < nup) {
        int tk = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
        while ((tk + 1) * (tk + 2) / 2 <= t) ++tk;
        while (tk * (tk + 1) / 2 > t) --tk;
        const int ti = t - tk * (tk + 1) / 2;
        small::tile_update(W, ld, stage, w, c0, nb, c0 + 4 * ti, c0 + 4 * tk, l, l, true, 0);
      } else {
        const int u = t - nup;
        small::tile_update(W, ld, stage, w, c0, nb, c0 + 4 * (u / TR), l + 4 * (u % TR), l, l + nright,
                           false, 0);
      }
    }
    cluster.sync();
  }
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
  double* Dsm = dsm;            // 32 x 32
  double* stage = dsm + 1024;   // NB x (l + NB)
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
      const bool fail = chol_aug_cluster(cluster, W, l, Dsm, stage, &s_flag);
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
