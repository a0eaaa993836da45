// Register-resident Businger-Golub QRCP of a small core (l <= 64): the
// latency path of every CoR-UTV call with a narrow sketch (C1 l = 15, C2
// l = 50, the ALM iterations' l = 1..64 cores).
//
// Same algorithm and decisions as small::qrcp_body (dense.py:152-192 /
// dense.py:104-129): pivot = first LOGICAL position of the largest downdated
// norm^2, Householder reflector x0 + sign(x0) |x|, norm downdate with the
// refresh rule (dense.py:181-190), the delta truncation of _truncate_utv
// (rpca.py:122-132), explicit Q by reverse accumulation on the identity.
//
// Layout: G threads own one physical column; thread (c, g) keeps rows
// i = g + G k (k < LM / G) of column c in registers, so a step's dot
// products and updates never touch shared memory.  One __syncthreads per
// step: at its end every live column publishes its rows >= j + 1 (the
// next pivot column is read from there) and its norm^2; every warp then
// finds the pivot redundantly (lane-parallel argmax over the published
// norms).  The logical <-> physical maps and the norms are double-buffered
// by step parity, so a warp still reading step j never sees step j + 1's
// writes.  Q is accumulated afterwards in the same registers from the
// reflector tails left in shared memory (no barrier per reflector).
#pragma once
#include "common.cuh"

namespace qreg {

template <int LM>
struct Shared {
  double rs[LM][LM + 1];   // rows >= current step of every column (pivot tails stay)
  double nrm[2][LM];       // published norm^2, -1 once pivoted
  int at[2][LM];           // logical position -> physical column
  int lpos[2][LM];         // physical column -> logical position
  double diag[LM], tau[LM], vhead[LM];
  int has_ref[LM];
};

template <int G>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// D (l x l, ld ldd) -> T (l x l, ld ldt; rows >= kend zero), qtT (row c =
// column c of Q, ld ldq), perm (logical -> physical), *r_out: with
// delta >= 0 the count of |diag T| > delta over the steps taken, else kend.
template <int LM, int G>
__global__ void __launch_bounds__(LM * G, 1)
    qrcp_reg_kernel(const double* __restrict__ D, int l, int64_t ldd, double* __restrict__ T, int64_t ldt,
                    double* __restrict__ qtT, int64_t ldq, long long* perm_out, int* perm32, double delta,
                    int* r_out) {
  constexpr int NT = LM * G, RPT = LM / G, NWP = NT / 32;
  static_assert(LM % 32 == 0 && 32 % G == 0 && LM % G == 0 && G > 1, "shape");
  __shared__ Shared<LM> sm;
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = tid / G, g = tid % G;
  const bool live_col = c < l;
  double r[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int i = g + G * k;
    r[k] = (live_col && i < l) ? D[(int64_t)i * ldd + c] : 0.0;
    sm.rs[i][c] = r[k];
  }
  // initial norms^2 (dense.py:165-166)
  double part = 0.0;
#pragma unroll
  for (int k = 0; k < RPT; ++k) part = fma(r[k], r[k], part);
  double nrm = gsum<G>(part);
  double ref = nrm;
  if (g == 0) {
    sm.nrm[0][c] = live_col ? nrm : -1.0;
    sm.at[0][c] = c;
    sm.lpos[0][c] = c;
  }
  bool done = !live_col;
  int rcount = 0, kend = l;
  __syncthreads();

  for (int j = 0; j < l; ++j) {
    const int cb = j & 1, nb = cb ^ 1;
    // pivot: first logical position of the max published norm^2, every warp
    double best = -1.0;
    int bq = LM, bc = 0;
#pragma unroll
    for (int h = 0; h < LM / 32; ++h) {
      const int cc = lane + 32 * h;
      const double v = sm.nrm[cb][cc];
      const int q = sm.lpos[cb][cc];
      if (cc < l && (v > best || (v == best && q < bq))) {
        best = v;
        bq = q;
        bc = cc;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > best || (ov == best && oq < bq)) {
        best = ov;
        bq = oq;
        bc = oc;
      }
    }
    if (delta >= 0.0 && best * 1.001 < delta * delta) {  // qrcp_body's truncation rule
      kend = j;
      break;
    }
    const int p = bq < l ? bq : j, pc = bq < l ? bc : sm.at[cb][j];
    const int cj = sm.at[cb][j];
    // reflector of x = R[j:, pc] (every thread, from the published tail)
    double xr[RPT];
    double t2p = 0.0;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int i = g + G * k;
      xr[k] = (i > j && i < l) ? sm.rs[i][pc] : 0.0;
      t2p = fma(xr[k], xr[k], t2p);
    }
    const double t2 = gsum<G>(t2p);
    const double x0 = sm.rs[j][pc];
    const double nx = sqrt(x0 * x0 + t2);
    const bool refl = nx != 0.0;
    const double v0 = refl ? x0 + (x0 >= 0.0 ? nx : -nx) : 0.0;
    const double tj = refl ? 2.0 / (v0 * v0 + t2) : 0.0;
    const double dj = refl ? x0 - v0 * (tj * (v0 * x0 + t2)) : x0;
    rcount += (fabs(dj) > delta) ? 1 : 0;
    if (tid == 0) {
      sm.diag[j] = dj;
      sm.tau[j] = tj;
      sm.vhead[j] = v0;
      sm.has_ref[j] = refl ? 1 : 0;
    }
    // logical maps for step j + 1 (swap positions j and p)
    if (tid < l) {
      sm.at[nb][tid] = (tid == j) ? pc : ((tid == p) ? cj : sm.at[cb][tid]);
      sm.lpos[nb][tid] = (tid == pc) ? j : ((tid == cj) ? p : sm.lpos[cb][tid]);
    }
    const int jo = j % G, jk = j / G;  // owner sub-lane / register slot of row j
    const bool act = !done && c != pc;
    if (c == pc) done = true;
    if (refl) {  // uniform; the group sums run in every lane (shuffles)
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < RPT; ++k) s = fma(xr[k], r[k], s);
      if (g == jo) {
#pragma unroll
        for (int k = 0; k < RPT; ++k)
          if (k == jk) s = fma(v0, r[k], s);
      }
      const double w = tj * gsum<G>(s);
      if (act) {
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int i = g + G * k;
          if (i > j) r[k] = fma(-xr[k], w, r[k]);
          else if (i == j) r[k] = fma(-v0, w, r[k]);
        }
      }
    }
    // norm downdate / refresh (dense.py:181-190); rows of this column
    // below j are final from here on
    double rjv = 0.0;
#pragma unroll
    for (int k = 0; k < RPT; ++k)
      if (k == jk) rjv = r[k];
    rjv = __shfl_sync(0xffffffffu, rjv, (lane / G) * G + jo);
    bool stale = false;
    double nv = nrm;
    if (act && j + 1 < l) {
      nv = fmax(nrm - rjv * rjv, 0.0);
      stale = nv < 1e-10 * ref;
    }
    if (__any_sync(0xffffffffu, stale)) {
      double f = 0.0;
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int i = g + G * k;
        if (i > j) f = fma(r[k], r[k], f);
      }
      f = gsum<G>(f);
      if (stale) {
        nv = f;
        ref = f;
      }
    }
    if (act && j + 1 < l) nrm = nv;
    // publish rows >= j + 1 and the norm for the next step
    if (act) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int i = g + G * k;
        if (i > j) sm.rs[i][c] = r[k];
      }
    }
    if (g == 0 && c < LM) sm.nrm[nb][c] = act ? nrm : -1.0;
    __syncthreads();
  }
  __syncthreads();
  const int fb = kend & 1;
  // this column's final logical position and its R rows -> T (row-major)
  if (live_col) {
    const int q = sm.lpos[fb][c];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int i = g + G * k;
      if (i >= l) continue;
      double v = 0.0;
      if (i < kend) v = (i < q) ? r[k] : ((i == q) ? sm.diag[i] : 0.0);
      T[(int64_t)i * ldt + q] = v;
    }
  }
  // explicit Q by reverse accumulation on the identity (dense.py:117-129):
  // thread (c, g) now holds rows g + G k of column c of Q
#pragma unroll
  for (int k = 0; k < RPT; ++k) r[k] = (g + G * k == c) ? 1.0 : 0.0;
  for (int j = kend - 1; j >= 0; --j) {
    if (!sm.has_ref[j]) continue;  // uniform
    const bool upd = live_col && c >= j;  // per column group; shuffles below run in every lane
    const int pc = sm.at[fb][j];
    const double v0 = sm.vhead[j], tj = sm.tau[j];
    const int jo = j % G, jk = j / G;
    double s = 0.0;
    double xr[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int i = g + G * k;
      xr[k] = (i > j && i < l) ? sm.rs[i][pc] : 0.0;
      s = fma(xr[k], r[k], s);
    }
    if (g == jo) {
#pragma unroll
      for (int k = 0; k < RPT; ++k)
        if (k == jk) s = fma(v0, r[k], s);
    }
    const double w = tj * gsum<G>(s);
    if (upd) {
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int i = g + G * k;
        if (i > j) r[k] = fma(-xr[k], w, r[k]);
        else if (i == j) r[k] = fma(-v0, w, r[k]);
      }
    }
  }
  if (live_col) {
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int i = g + G * k;
      if (i < l) qtT[(int64_t)c * ldq + i] = r[k];
    }
  }
  if (tid < l) {
    const int pcol = sm.at[fb][tid];
    if (perm_out) perm_out[tid] = pcol;
    perm32[tid] = pcol;
  }
  if (tid == 0 && r_out) *r_out = delta >= 0.0 ? rcount : kend;
  (void)NWP;
}

}  // namespace qreg
