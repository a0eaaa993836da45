// tsr_svd's two sketches from ONE pass over A (sketch.py:160-163
// `fused_sketch`, used by tsr_svd sketch.py:220-241): y = A psi (m x l) and
// z = A' phi (n x l) for narrow sketches (l <= 8).
//
// Every 128 x 16 tile of A that TMA lands in shared memory (128-byte
// swizzle, mbarrier full/empty ring) feeds both products on the FP64 tensor
// pipe (DMMA.884).  One CTA of sixteen warps per SM (<= 128 registers each;
// four warps per scheduler hide a little more of the DMMA / shared-memory
// latency than two: 8-warp versions streamed A at 3.3-3.5 TB/s, this one at
// 3.7-3.8; profiles/r02_dual_sketch.txt has the anatomy):
//   * y: warp w owns rows 8w .. 8w+7 of every tile: one 8-row fragment,
//     K = the tile's 16 columns (the KK fragment reads of gemm::mainloop),
//     accumulated in registers over the KT k-tiles of a column block and then
//     added to the CTA's y rows in shared memory;
//   * z: warp w owns row quarter w & 3 (32 rows) of every fourth k-tile
//     (kt & 3 == w >> 2): z[tile columns] += A_tile' phi over those rows, the
//     swizzled rows read transposed (k' = rows 4t + (lane & 3), one LDS.128
//     per k-step feeding the two 8-column fragments), phi's 32 rows held in
//     registers for the sub-block, accumulators kept in registers across the
//     panel's row sub-blocks.  A window of four tiles keeps all warps busy
//     while the ring's other slots take the next window.
// A CTA walks panels of <= NMS 128-row sub-blocks; per panel it walks the
// column blocks (<= KT k-tiles each) and, inside, the panel's sub-blocks.
// After a column block the four row quarters of each tile are summed in
// quarter order through shared memory and stored to the panel's slot of
// zpart; the panel slots are summed in panel order afterwards
// (aux::splitk_finalize_kernel) -- deterministic.  y rows are complete per
// panel and written once.
//
// A is read once: 8 m n bytes per call against 16 m n for two sweeps.
#pragma once
#include "common.cuh"

#ifndef DUAL_SMAX
#define DUAL_SMAX 6  // ring depth cap (a build knob: the depth sweep of profiles/r02_dual_sketch.txt)
#endif

namespace dual {

constexpr int BM = 128, BK = 16;
constexpr int WARPS = 16, THREADS = WARPS * 32;
constexpr int NMS = 4;                        // row sub-blocks per panel (y rows in shared memory)
constexpr int KT = 8;                         // k-tiles per column block
constexpr int ZW = 8;                         // stored sketch width
constexpr int ZT = KT / 4;                    // k-tiles of a column block a warp owns a row quarter of
constexpr int A_BYTES = BM * BK * 8;          // 16 KB
constexpr int P_BYTES = ZW * BK * 8;          // psi' tile: 1 KB
constexpr int PHI_BYTES = BM * 16 * 8;        // 16 KB
constexpr int SY_BYTES = NMS * BM * ZW * 8;   // 32 KB
constexpr int ZRED_BYTES = 4 * ZT * 2 * 3 * 32 * 16;  // quarters 1..3 of every tile of a column block: 24 KB
constexpr int FIXED = 2 * PHI_BYTES + SY_BYTES + ZRED_BYTES + 256;
constexpr int S_FIT = (225 * 1024 - 1024 - FIXED) / (A_BYTES + P_BYTES);
// measured on the kernel alone (8.6 GB, l = 8): S = 3: 2.91 ms, 4: 2.28, 5: 2.65, 6: 2.31, 7: 2.56 --
// a step takes two tiles, and an even ring keeps each step's slot pair fixed
constexpr int S = S_FIT > DUAL_SMAX ? DUAL_SMAX : S_FIT;
static_assert(S >= 3, "a step issues two tiles while two are being consumed");
constexpr int SMEM = 1024 + S * (A_BYTES + P_BYTES) + FIXED;

// Producer cursor: the next tile of the CTA's stream
// (panel, column block, sub-block, k-tile) and its ring position.
struct Cursor {
  int pi, cb, msl, kt;  // position
  int sbi;              // running (column block, sub-block) count: phi buffer parity
  int slot, round;      // ring slot and how many times the ring wrapped
  int ms0, nms;         // the panel's first sub-block and sub-block count   } cached: the 64-bit
  int kt0, ktn;         // the column block's first k-tile and k-tile count  } divisions run only
                        //                                                   } when pi / cb change
};

// y: m x ldy (columns >= l written as 0); zpart: panels x n x ZW.
__global__ void __launch_bounds__(THREADS, 1)
    dual_sketch_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapP,
                       const __grid_constant__ CUtensorMap mapF, int64_t m, int64_t n, int msubs_total,
                       int panels_total, int panels_per_cta, double* __restrict__ y, int64_t ldy,
                       double* __restrict__ zpart, int* bad_flag, int dbg) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  unsigned char* base = smem_raw + pad;
  double* sa = reinterpret_cast<double*>(base);
  double* sp = reinterpret_cast<double*>(base + S * A_BYTES);
  double* sf = reinterpret_cast<double*>(base + S * (A_BYTES + P_BYTES));
  double* sy = reinterpret_cast<double*>(base + S * (A_BYTES + P_BYTES) + 2 * PHI_BYTES);
  double2* zred = reinterpret_cast<double2*>(base + S * (A_BYTES + P_BYTES) + 2 * PHI_BYTES + SY_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S * (A_BYTES + P_BYTES) + 2 * PHI_BYTES + SY_BYTES +
                                               ZRED_BYTES);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r8 = lane >> 2, c4 = lane & 3;
  const int p_first = blockIdx.x * panels_per_cta;
  const int p_last = min(panels_total, p_first + panels_per_cta);  // exclusive
  // Column blocks: the kt_total k-tiles split evenly into ncb blocks of at
  // most KT (host: kt_total >= KT), so every block has >= KT / 2 k-tiles.
  // With S <= 2 (KT / 2) + 2 two consecutive (column block, sub-block) runs
  // cover the ring's lookahead, which is what lets the ring's empty barriers
  // also guard the two phi buffers: phi for run i + 2 is issued after the
  // empty wait on a tile that lies inside run i + 1 or later -- every warp
  // has read run i's phi into registers by then.
  const int kt_total = (int)((n + BK - 1) / BK);
  const int ncb = (kt_total + KT - 1) / KT;
  static_assert(2 * (KT / 2) >= S - 2, "phi double buffer needs two runs to cover the lookahead");
  auto panel_ms0 = [&](int p) { return (int)(((long long)p * msubs_total) / panels_total); };
  auto kt0_of = [&](int cb) { return (int)(((long long)cb * kt_total) / ncb); };
  // Each CTA starts its walk over the column blocks at a different one
  // (wrapping around): with every CTA on the same few hundred columns at
  // the same time, the rows' power-of-two stride puts all their requests
  // on the same few memory channels.
  const int cb_rot = (int)(((long long)blockIdx.x * ncb) / gridDim.x);
  auto cb_phys = [&](int cb) { return cb + cb_rot >= ncb ? cb + cb_rot - ncb : cb + cb_rot; };
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (p_first >= p_last) return;

  // ---- producer (thread 0, inline): issue the tile at `cur`, advance it
  Cursor cur{p_first, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  cur.ms0 = panel_ms0(p_first);
  cur.nms = panel_ms0(p_first + 1) - cur.ms0;
  cur.kt0 = kt0_of(cb_phys(0));
  cur.ktn = kt0_of(cb_phys(0) + 1) - cur.kt0;
  bool cur_done = false;
  auto issue_next = [&]() {
    if (cur_done) return;
    if (cur.round > 0) mbar_wait(&empty[cur.slot], (cur.round - 1) & 1);
    const int kcol = (cur.kt0 + cur.kt) * BK, row0 = (cur.ms0 + cur.msl) * BM;
    mbar_arrive_expect_tx(&full[cur.slot], A_BYTES + P_BYTES + (cur.kt == 0 ? PHI_BYTES : 0));
    tma_load_2d(sa + cur.slot * (BM * BK), &mapA, &full[cur.slot], kcol, row0);
    tma_load_2d(sp + cur.slot * (ZW * BK), &mapP, &full[cur.slot], kcol, 0);
    if (cur.kt == 0) tma_load_2d(sf + (cur.sbi & 1) * (BM * 16), &mapF, &full[cur.slot], 0, row0);
    if (++cur.slot == S) {
      cur.slot = 0;
      ++cur.round;
    }
    if (++cur.kt == cur.ktn) {
      cur.kt = 0;
      ++cur.sbi;
      if (++cur.msl == cur.nms) {
        cur.msl = 0;
        if (++cur.cb == ncb) {
          cur.cb = 0;
          if (++cur.pi == p_last) {
            cur_done = true;
            return;
          }
          cur.ms0 = panel_ms0(cur.pi);
          cur.nms = panel_ms0(cur.pi + 1) - cur.ms0;
        }
        cur.kt0 = kt0_of(cb_phys(cur.cb));
        cur.ktn = kt0_of(cb_phys(cur.cb) + 1) - cur.kt0;
      }
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapP);
    tma_prefetch_desc(&mapF);
    // S - 2 ahead: a step consumes up to two tiles and refills the two slots
    // the step before released
    for (int i = 0; i < S - 2; ++i) issue_next();
  }

  // ---- consumers
  // rho: DMMA row index r8 -> operand row.  A 128-bit shared load is served
  // per quarter-warp (r8 in {2q, 2q+1} x c4 in 0..3); rows q and q + 4 have
  // swizzle phases that differ in bit 2, so the quarter's eight 16-byte
  // chunks fall in eight different bank groups (rows q, q + 1 would collide
  // pairwise: measured 2x the wavefronts).
  const int rho = (r8 >> 1) + 4 * (r8 & 1);
  int offA[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) offA[p] = ((4 * p + c4) ^ rho) << 1;
  const int rowA = (warp * 8 + rho) * 16;  // y: this lane's A row
  // z: k-step t reads tile rows 32 zq + 4t + c4, the 16-byte chunk holding
  // columns 2 rho, 2 rho + 1 (fragment e = column parity); the swizzle phase
  // (4t + c4) & 7 only depends on t & 1
  const int zq = warp & 3, tw = warp >> 2;
  int offZ[2];
#pragma unroll
  for (int tp = 0; tp < 2; ++tp) offZ[tp] = (32 * zq + c4) * 16 + ((rho ^ (4 * tp + c4)) << 1);  // + 64 t
  constexpr int NZ = 2;   // independent accumulator sets per z fragment (DMMA dependent-issue latency)
  constexpr int YS = 4;   // the same for the y fragment: every DMMA of a tile extends its own chain
  int slot = 0;
  uint32_t phase = 0;
  int sbi = 0;
  // as_matrix's finiteness check (dense.py:41-50): the y reads touch every A
  // element once; bit 31 of (exponent field + 1 ulp of it) is set iff the
  // exponent is all ones -- integer work only, nothing on the FP64 pipe
  uint32_t badbits = 0;
  for (int pi = p_first; pi < p_last; ++pi) {
    const int ms0 = panel_ms0(pi), nms = panel_ms0(pi + 1) - ms0;
    for (int e = threadIdx.x; e < nms * BM * ZW; e += THREADS) sy[e] = 0.0;
    __syncthreads();
    for (int cb = 0; cb < ncb; ++cb) {
      const int kt0 = kt0_of(cb_phys(cb));
      const int ktn = kt0_of(cb_phys(cb) + 1) - kt0;
      double z[ZT][NZ][2][2];
#pragma unroll
      for (int zt = 0; zt < ZT; ++zt)
#pragma unroll
        for (int q = 0; q < NZ; ++q)
#pragma unroll
          for (int e = 0; e < 2; ++e) z[zt][q][e][0] = z[zt][q][e][1] = 0.0;
      for (int msl = 0; msl < nms; ++msl, ++sbi) {
        double acc[YS][2];
#pragma unroll
        for (int ys = 0; ys < YS; ++ys) acc[ys][0] = acc[ys][1] = 0.0;
        double phr[8];  // phi[row 32 zq + 4t + c4][r8] of this sub-block
        // one landed tile: the warp's y rows, and its z row quarter if it owns the tile
        auto tile = [&](const int kt, const double* ta, const double* tp) {  // kt: a constant after unrolling
          // dbg (measurement only, results are wrong): 1 skips the y product, 2 the z product
          if (!(dbg & 1))
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const double2 a2 = *reinterpret_cast<const double2*>(ta + rowA + offA[p]);
            const double2 b2 = *reinterpret_cast<const double2*>(tp + rho * 16 + offA[p]);
            badbits |= (static_cast<uint32_t>(__double2hiint(a2.x)) & 0x7ff00000u) + 0x00100000u;
            badbits |= (static_cast<uint32_t>(__double2hiint(a2.y)) & 0x7ff00000u) + 0x00100000u;
            dmma884(acc[2 * p][0], acc[2 * p][1], a2.x, b2.x);
            dmma884(acc[2 * p + 1][0], acc[2 * p + 1][1], a2.y, b2.y);
          }
          if ((kt & 3) == tw && !(dbg & 2)) {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const double2 av = *reinterpret_cast<const double2*>(ta + t * 64 + offZ[t & 1]);
              dmma884(z[kt / 4][t % NZ][0][0], z[kt / 4][t % NZ][0][1], av.x, phr[t]);
              dmma884(z[kt / 4][t % NZ][1][0], z[kt / 4][t % NZ][1][1], av.y, phr[t]);
            }
          }
        };
        // Two tiles per step (both waited for, then computed in one
        // straight-line block the scheduler can interleave), released together.
#pragma unroll
        for (int kt = 0; kt < KT; kt += 2) {
          if (kt < ktn) {
            const bool two = kt + 1 < ktn;
            if (threadIdx.x == 0) {
              issue_next();
              if (two) issue_next();
            }
            const int s0 = slot, s1 = slot + 1 == S ? 0 : slot + 1;
            const uint32_t ph1 = slot + 1 == S ? phase ^ 1u : phase;
            mbar_wait(&full[s0], phase);
            if (two) mbar_wait(&full[s1], ph1);
            if (kt == 0) {
              const double* fb = sf + (sbi & 1) * (BM * 16);
#pragma unroll
              for (int t = 0; t < 8; ++t) phr[t] = fb[swz128(32 * zq + 4 * t + c4, r8)];
            }
            if (two) {
              tile(kt, sa + s0 * (BM * BK), sp + s0 * (ZW * BK));
              tile(kt + 1, sa + s1 * (BM * BK), sp + s1 * (ZW * BK));
            } else {
              tile(kt, sa + s0 * (BM * BK), sp + s0 * (ZW * BK));
            }
            // every LDS of these stages completes before the slots are released
            __syncwarp();
            __threadfence_block();
            if (lane == 0) {
              mbar_arrive(&empty[s0]);
              if (two) mbar_arrive(&empty[s1]);
            }
            slot += two ? 2 : 1;
            if (slot >= S) {
              slot -= S;
              phase ^= 1u;
            }
          }
        }
        // this sub-block's y rows += the column block's contribution; fragment
        // column 2 c4 + e is sketch column rho(2 c4 + e) = c4 + 4 e
        double* yb = sy + (msl * BM + warp * 8 + rho) * ZW;
#pragma unroll
        for (int e = 0; e < 2; ++e) yb[c4 + 4 * e] += (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
      }
      // The column block is complete over the panel's rows: sum each
      // fragment's accumulator sets; row quarters 1..3 hand theirs to
      // quarter 0's warp through shared memory, which adds them in quarter
      // order (fixed) and stores to the panel's slot.
      if (zq != 0) {
#pragma unroll
        for (int zt = 0; zt < ZT; ++zt)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            zred[((((tw * ZT + zt) * 2 + e) * 3 + (zq - 1)) << 5) + lane] =
                make_double2(z[zt][0][e][0] + z[zt][1][e][0], z[zt][0][e][1] + z[zt][1][e][1]);
      }
      __syncthreads();
      if (zq == 0) {
#pragma unroll
        for (int zt = 0; zt < ZT; ++zt) {
          const int kt = zt * 4 + tw;
          if (kt < ktn) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int64_t col = (int64_t)(kt0 + kt) * BK + 2 * rho + e;
              double v0 = z[zt][0][e][0] + z[zt][1][e][0], v1 = z[zt][0][e][1] + z[zt][1][e][1];
#pragma unroll
              for (int q = 0; q < 3; ++q) {
                const double2 o = zred[((((tw * ZT + zt) * 2 + e) * 3 + q) << 5) + lane];
                v0 += o.x;
                v1 += o.y;
              }
              if (col < n)
                *reinterpret_cast<double2*>(zpart + ((int64_t)pi * n + col) * ZW + 2 * c4) = make_double2(v0, v1);
            }
          }
        }
      }
      __syncthreads();
    }
    // the panel's y rows are complete
    for (int e = threadIdx.x; e < nms * BM * ZW; e += THREADS) {
      const int64_t row = (int64_t)ms0 * BM + e / ZW;
      const int col = e % ZW;
      if (row < m) y[row * ldy + col] = sy[e];
    }
    for (int e = threadIdx.x; e < nms * BM * (16 - ZW); e += THREADS) {
      const int64_t row = (int64_t)ms0 * BM + e / (16 - ZW);
      const int col = ZW + e % (16 - ZW);
      if (row < m && col < ldy) y[row * ldy + col] = 0.0;
    }
    __syncthreads();
  }
  if (bad_flag && __any_sync(0xffffffffu, (badbits >> 31) != 0) && lane == 0) atomicOr(bad_flag, 1);
}

}  // namespace dual
