// tsr_svd's two sketches from ONE pass over A (sketch.py:160-163
// `fused_sketch`, used by tsr_svd sketch.py:220-241): y = A psi (m x l) and
// z = A' phi (n x l) for narrow sketches (l <= 16).
//
// Every 128 x 16 tile of A that TMA lands in shared memory feeds both
// products on the FP64 tensor pipe (DMMA.884):
//   * warps 4-7 (y): y[rows] += A_tile psi_tile (KK fragments as
//     gemm::mainloop), accumulated in registers over the 16 k-tiles of a
//     256-column block, then added into the CTA's y rows in shared memory;
//   * warps 0-3 (z): z[tile columns] += A_tile' phi[rows] -- the same
//     swizzled tile read transposed (row = k', column = m') -- warp w owning
//     one 8 x 8 output block (column half w & 1, l half w >> 1) for each of
//     the block's 16 k-tiles, in registers across the CTA's row sub-blocks.
// A CTA owns a contiguous run of 128-row sub-blocks (its y rows complete,
// written once at the end) and walks all 256-column blocks; after each it
// writes its z partial for those columns (slot = CTA), summed over CTAs in
// CTA order by the finalize (deterministic).  Loads: A tile 16 KB + psi'
// tile 2 KB per stage, phi's 128 x 16 rows (16 KB) with the first k-tile of
// every sub-block into a buffer picked by sub-block parity; S-stage ring
// with S - 1 tiles of lookahead across sub-block and column-block edges.
// A is read once: 8 m n bytes per call, against 16 m n for two sweeps.
#pragma once
#include "common.cuh"

namespace dual {

constexpr int BM = 128, BK = 16, KT = 16, CB = BK * KT, S = 3;
constexpr int THREADS = 256;
constexpr int YMAX = 7;                       // row sub-blocks per CTA (y rows in shared memory)
constexpr int A_BYTES = BM * BK * 8;          // 16 KB
constexpr int P_BYTES = 16 * BK * 8;          // psi' tile: 2 KB
constexpr int PHI_BYTES = BM * 16 * 8;        // 16 KB
constexpr int LDY = 16;
constexpr int SMEM = 1024 + S * (A_BYTES + P_BYTES) + 2 * PHI_BYTES + YMAX * BM * LDY * 8 + 16 * 8;

__device__ __forceinline__ int swz(int row, int col) {
  return row * 16 + ((((col >> 1) ^ (row & 7)) << 1) | (col & 1));
}

// y: m x ldy (cols >= l written as 0); zpart: gridDim.x slices of n x 16.
__global__ void __launch_bounds__(THREADS, 1)
    dual_sketch_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapP,
                       const __grid_constant__ CUtensorMap mapF, int64_t m, int64_t n, int msubs_total,
                       double* __restrict__ y, int64_t ldy, double* __restrict__ zpart, int* bad_flag) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* base = smem_raw + pad;
  double* sa = reinterpret_cast<double*>(base);
  double* sp = reinterpret_cast<double*>(base + S * A_BYTES);
  double* sf = reinterpret_cast<double*>(base + S * (A_BYTES + P_BYTES));
  double* sy = reinterpret_cast<double*>(base + S * (A_BYTES + P_BYTES) + 2 * PHI_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S * (A_BYTES + P_BYTES) + 2 * PHI_BYTES + YMAX * BM * LDY * 8);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r8 = lane >> 2, c4 = lane & 3;
  const int G = gridDim.x, c = blockIdx.x;
  const int ms0 = (int)(((long long)c * msubs_total) / G), ms1 = (int)(((long long)(c + 1) * msubs_total) / G);
  const int nms = ms1 - ms0;
  const int ncb = (int)((n + CB - 1) / CB);
  const int total = ncb * nms * KT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    fence_barrier_init();
  }
  for (int e = threadIdx.x; e < nms * BM * LDY; e += THREADS) sy[e] = 0.0;
  __syncthreads();
  // load q = ((cb * nms) + msl) * KT + kt of this CTA's stream into its slot
  auto issue = [&](int q) {
    const int kt = q % KT, msl = (q / KT) % nms, cb = q / (KT * nms);
    const int slot = q % S;
    if (q >= S) mbar_wait(&empty[slot], ((q / S) - 1) & 1);
    const int kcol = (cb * KT + kt) * BK, row0 = (ms0 + msl) * BM;
    mbar_arrive_expect_tx(&full[slot], A_BYTES + P_BYTES + (kt == 0 ? PHI_BYTES : 0));
    tma_load_2d(sa + slot * (BM * BK), &mapA, &full[slot], kcol, row0);
    tma_load_2d(sp + slot * (16 * BK), &mapP, &full[slot], kcol, 0);
    // phi buffer by the parity of the sub-block's position in the stream
    if (kt == 0) tma_load_2d(sf + ((q / KT) & 1) * (BM * 16), &mapF, &full[slot], 0, row0);
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapP);
    tma_prefetch_desc(&mapF);
    for (int q = 0; q < S - 1 && q < total; ++q) issue(q);
  }
  const bool zw = warp < 4;
  // z-warp block: tile columns mh*8 .. +7 (the k' index of A'), l columns nh*8 .. +7
  const int mh = warp & 1, nh = (warp >> 1) & 1;
  // y-warp rows: (warp - 4) * 32 .. +31
  const int yw = warp - 4;
  int offA[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) offA[p] = ((4 * p + c4) ^ r8) << 1;
  const int rowA = (yw * 32 + r8) * 16;
  bool bad = false;  // as_matrix's finiteness check (dense.py:41-50), on the y warps' reads of every A element
  for (int cb = 0; cb < ncb; ++cb) {
    double z[KT][2];
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) z[kt][0] = z[kt][1] = 0.0;
    for (int msl = 0; msl < nms; ++msl) {
      double acc[4][2][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) acc[mi][nj][0] = acc[mi][nj][1] = 0.0;
      const double* fb = sf + ((cb * nms + msl) & 1) * (BM * 16);
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int q = (cb * nms + msl) * KT + kt;
        if (threadIdx.x == 0 && q + S - 1 < total) issue(q + S - 1);
        const int slot = q % S;
        mbar_wait(&full[slot], (q / S) & 1);
        const double* ta = sa + slot * (BM * BK);
        if (zw) {
          // z[kt] (8 x 8 block) += A_tile[:, mh*8 ..]' phi[:, nh*8 ..], K' = 128 rows.
          // k-step s of a 16-row group reads rows s + 4 (lane & 3): two
          // swizzle phases per fragment, 2 wavefronts per 256 B (gemm MM's
          // trick); both operands use the same row order.
#pragma unroll 4
          for (int g = 0; g < BM / 16; ++g)
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
              const int row = g * 16 + s4 + 4 * c4;
              const double a = ta[swz(row, mh * 8 + r8)];
              const double b = fb[swz(row, nh * 8 + r8)];
              dmma884(z[kt][0], z[kt][1], a, b);
            }
        } else {
          const double* tp = sp + slot * (16 * BK);
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            double2 a2[4], b2[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
              a2[mi] = *reinterpret_cast<const double2*>(ta + rowA + mi * 8 * 16 + offA[p]);
              bad |= is_nonfinite(a2[mi].x) | is_nonfinite(a2[mi].y);
            }
#pragma unroll
            for (int nj = 0; nj < 2; ++nj)
              b2[nj] = *reinterpret_cast<const double2*>(tp + (nj * 8 + r8) * 16 + offA[p]);
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int nj = 0; nj < 2; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a2[mi].x, b2[nj].x);
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int nj = 0; nj < 2; ++nj) dmma884(acc[mi][nj][0], acc[mi][nj][1], a2[mi].y, b2[nj].y);
          }
        }
        __syncwarp();
        __threadfence_block();
        if (lane == 0) mbar_arrive(&empty[slot]);
      }
      if (!zw) {  // y rows of this sub-block += this column block's contribution
        double* yb = sy + msl * (BM * LDY);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj)
#pragma unroll
            for (int e = 0; e < 2; ++e) yb[(yw * 32 + mi * 8 + r8) * LDY + nj * 8 + 2 * c4 + e] += acc[mi][nj][e];
      }
    }
    if (zw) {  // this CTA's z partial for the column block
      double* zp = zpart + (int64_t)c * n * 16;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int64_t col = (int64_t)(cb * KT + kt) * BK + mh * 8 + r8;
        if (col < n) {
          zp[col * 16 + nh * 8 + 2 * c4] = z[kt][0];
          zp[col * 16 + nh * 8 + 2 * c4 + 1] = z[kt][1];
        }
      }
    }
  }
  if (bad_flag && !zw && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(bad_flag, 1);
  __syncthreads();
  for (int e = threadIdx.x; e < nms * BM * 16; e += THREADS) {
    const int64_t row = (int64_t)ms0 * BM + e / 16;
    const int col = e % 16;
    if (row < m && col < ldy) y[row * ldy + col] = sy[(e / 16) * LDY + col];
  }
}

}  // namespace dual
