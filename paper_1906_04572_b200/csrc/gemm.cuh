// FP64 tensor-core (DMMA) GEMMs for the CoR-UTV sketch contractions.
//
// Two operand orientations, both fed by TMA (cp.async.bulk.tensor, 128-byte
// swizzle) through an mbarrier full/empty ring, one producer warp and eight
// consumer warps issuing mma.sync.m8n8k4.f64 (SASS DMMA.884):
//
//   KK ("both K-major"):  C[M x N] = A[M x K] * Bt[N x K]^T
//        A·Ω, A·Q2 (sketch.py:149,158), X·R^-1 (QR), Q1·Q~ (sketch.py:205),
//        U_r·(T_r V')  (rpca.py:129) with fused ALM / residual epilogues.
//   MM ("both M-major"):  C[M x N] = A[K x M]^T * B[K x N]
//        A'·C1 (sketch.py:153), Gram X'X (QR), Q1'·(A Q2) (sketch.py:158).
//
// CTA tile: 128 rows x 16J columns (J = 1..8), warps 4 (M) x 2 (N), each warp
// 32 x 8J.  One stage = 16 k-values: A tile 16 KB + B tile 2J KB.  For KK the
// fragment lanes read k = 4s + (lane&3) (conflict-free on the swizzled
// K-major rows); for MM they read rows k = s + 4*(lane&3) — a k permutation
// (both operands use it, so the contraction is unchanged) that makes the
// M-major swizzled tiles conflict-free as well.
#pragma once
#include "common.cuh"

#ifndef KK_RHO
#define KK_RHO 1  // build knob: 0 restores fragment rows r8 (2-way bank conflicts on every KK LDS.128)
#endif

namespace gemm {

// KK operand rows: a 128-bit shared load is served per quarter-warp
// (fragment rows r8 in {2q, 2q+1} x the four k chunks); consecutive rows
// would put the quarter's eight 16-byte chunks on four bank groups twice
// (ncu: half of all shared-memory wavefronts of the sweeps were conflicts).
// Mapping fragment row r8 to operand row q / q + 4 -- swizzle phases that
// differ in bit 2 -- spreads them over all eight.  The accumulator
// fragment then holds tile row kk_row(r8) and tile columns kk_col(c4, e).
__host__ __device__ constexpr int kk_row(int r8) { return KK_RHO ? (r8 >> 1) + 4 * (r8 & 1) : r8; }
__host__ __device__ constexpr int kk_col(int c4, int e) { return KK_RHO ? c4 + 4 * e : 2 * c4 + e; }

constexpr int BM = 128;
constexpr int BK = 16;
constexpr int NCW = 8;                 // warps (all compute; thread 0 also issues TMA)
constexpr int THREADS = NCW * 32;       // 2 warps per SMSP -> up to 255 registers each
constexpr int SMEM_BUDGET = 200 * 1024;

// WN = warps along N: 2 (CTA 128 x 16J, the default) or 1 (CTA 256 x 8J, for
// narrow N <= 64: an 8-column granularity instead of 16 halves the padding)
__host__ __device__ constexpr int bm_of(int WN) { return 32 * (NCW / WN); }       // CTA rows
__host__ __device__ constexpr int bn_of(int J, int WN) { return 8 * J * WN; }     // CTA columns
__host__ __device__ constexpr int nb16_of(int J, int WN) { return (bn_of(J, WN) + 15) / 16; }
__host__ __device__ constexpr int a_stage_bytes(int WN = 2) { return bm_of(WN) * BK * 8; }
// B slot: room for the 16-column boxes of the MM layout (>= the KK rows)
__host__ __device__ constexpr int b_stage_bytes(int J, int WN = 2) { return nb16_of(J, WN) * 16 * BK * 8; }
__host__ __device__ constexpr int stage_bytes(int J, int WN = 2) { return a_stage_bytes(WN) + b_stage_bytes(J, WN); }
// bytes TMA actually writes per stage (the mbarrier transaction count)
__host__ __device__ constexpr int stage_tx(int J, int WN, bool MM) {
  return a_stage_bytes(WN) + (MM ? b_stage_bytes(J, WN) : bn_of(J, WN) * BK * 8);
}
// MINB = CTAs per SM the launch targets: 2 halves the ring (112 KB each)
// so two CTAs -- twice the independent DMMA accumulator chains per SM
// sub-partition -- share an SM (narrow-N sweeps, whose 12 chains per warp
// leave the DMMA pipe latency-bound at one CTA per SM)
__host__ __device__ constexpr int smem_budget(int MINB) { return MINB == 1 ? SMEM_BUDGET : 112 * 1024; }
__host__ __device__ constexpr int num_stages(int J, int WN = 2, int MINB = 1) {
  return (smem_budget(MINB) - 1024) / stage_bytes(J, WN) > 8 ? 8 : (smem_budget(MINB) - 1024) / stage_bytes(J, WN);
}
__host__ __device__ constexpr int smem_bytes(int J, int WN = 2, int MINB = 1) {
  return 1024 /*align slack*/ + num_stages(J, WN, MINB) * stage_bytes(J, WN) + 2 * 8 * 8 + 64;
}
// low-rank (ALM / residual / store) kernels: K = r is short, so 2 stages; the
// same bytes are reused to stage the 128 x (16J + 2) result tile.
constexpr int LR_STAGES = 2;
__host__ __device__ constexpr int lr_tile_bytes(int J) { return BM * (16 * J + 2) * 8; }
__host__ __device__ constexpr int lr_data_bytes(int J) {
  return LR_STAGES * stage_bytes(J) > lr_tile_bytes(J) ? LR_STAGES * stage_bytes(J) : lr_tile_bytes(J);
}
__host__ __device__ constexpr int lr_smem_bytes(int J) { return 1024 + lr_data_bytes(J) + 2 * 8 * 8 + 64; }

struct Tile {
  int M, N, K;          // problem (this launch)
  int m_tiles, n_tiles;
  int k_tiles;          // total k tiles (ceil(K / 16))
  int k_tiles_per_split;
  int splits;
  int mm3d;             // MM operands as one 3-D box per stage: bit 0 A, bit 1 B;
                        // bit 2: A (the data matrix, read once) loaded evict-first
  int sk;               // > 0: stream-K (persistent grid over the linear (tile, k-tile)
                        // space; sk = partial slots per tile), 0: classic split-K
};

// Stream-K partition: CTA c of G owns units [c U / G, (c + 1) U / G) of the
// U = tiles * k_tiles linear (tile, k-tile) space; sk_cta_of(u) is the CTA
// owning unit u.  A tile's partial slots are numbered by owning CTA in
// order, so the finalize sums them in a fixed order (deterministic).
__host__ __device__ inline int sk_cta_of(long long u, long long U, int G) {
  int c = (int)((u * G) / U);
  while (c + 1 < G && ((long long)(c + 1) * U) / G <= u) ++c;
  while (c > 0 && ((long long)c * U) / G > u) --c;
  return c;
}

// Accumulator for one consumer warp: 4 (M) x J (N) DMMA fragments.
template <int J>
struct Acc {
  double v[4][J][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < J; ++j) v[i][j][0] = v[i][j][1] = 0.0;
  }
};

struct Smem {
  double* a;        // [stages][BM*BK]
  double* b;        // [stages][16J*BK]
  uint64_t* full;   // [stages]
  uint64_t* empty;  // [stages]
};

// Pointer arithmetic on the __shared__ array (never through an integer) so
// the compiler keeps the shared address space and emits LDS.
template <int J, int S, int DATA = S * (a_stage_bytes() + b_stage_bytes(J)), int WN = 2>
__device__ __forceinline__ Smem carve(unsigned char* raw) {
  const uint32_t pad = (1024u - (smem_u32(raw) & 1023u)) & 1023u;
  unsigned char* p = raw + pad;
  Smem s;
  s.a = reinterpret_cast<double*>(p);
  s.b = reinterpret_cast<double*>(p + S * a_stage_bytes(WN));
  s.full = reinterpret_cast<uint64_t*>(p + DATA);
  s.empty = s.full + 8;
  return s;
}

// Issue the TMA loads of k tile `kt` into ring slot `st` (thread 0 only).
template <int J, bool MM, int WN = 2>
__device__ __forceinline__ void issue_stage(const Smem& sm, const CUtensorMap* mapA,
                                            const CUtensorMap* mapB, int m0, int n0, int kt,
                                            int st, int mm3d = 0) {
  constexpr int BMW = bm_of(WN), NB16 = nb16_of(J, WN);
  mbar_arrive_expect_tx(&sm.full[st], stage_tx(J, WN, MM));
  double* sa = sm.a + st * (BMW * BK);
  double* sb = sm.b + st * (NB16 * 16 * BK);
  const bool ef = (mm3d & 4) != 0;
  const uint64_t pol = ef ? policy_evict_first() : 0;
  if (!MM) {
    if (ef) tma_load_2d_hint(sa, mapA, &sm.full[st], kt * BK, m0, pol);
    else tma_load_2d(sa, mapA, &sm.full[st], kt * BK, m0);
    tma_load_2d(sb, mapB, &sm.full[st], kt * BK, n0);
  } else {
    // mm3d bit 0 / bit 1: A / B fetched as one 3-D box {16 cols, rows, column
    // groups} (lands as [group][row][16]); otherwise one 2-D box per 16
    // columns (B columns need not start on a 16-column group)
    if (mm3d & 1) {
      if (ef) tma_load_3d_hint(sa, mapA, &sm.full[st], 0, kt * BK, m0 / 16, pol);
      else tma_load_3d(sa, mapA, &sm.full[st], 0, kt * BK, m0 / 16);
    } else {
#pragma unroll
      for (int bx = 0; bx < BMW / 16; ++bx) {
        if (ef) tma_load_2d_hint(sa + bx * 16 * BK, mapA, &sm.full[st], m0 + 16 * bx, kt * BK, pol);
        else tma_load_2d(sa + bx * 16 * BK, mapA, &sm.full[st], m0 + 16 * bx, kt * BK);
      }
    }
    if (mm3d & 2) {
      tma_load_3d(sb, mapB, &sm.full[st], 0, kt * BK, n0 / 16);
    } else {
#pragma unroll
      for (int bx = 0; bx < NB16; ++bx)
        tma_load_2d(sb + bx * 16 * BK, mapB, &sm.full[st], n0 + 16 * bx, kt * BK);
    }
  }
}

// Pipelined mainloop over k tiles [kt0, kt1).  Thread 0 keeps S-1..S stages
// in flight: at iteration i it refills the slot released at iteration i-1
// (waiting on that slot's `empty` barrier, i.e. on the slowest warp), so the
// wait almost never stalls.  Every warp: wait full -> 4 DMMA k-steps ->
// fence -> arrive empty.  All fragments are computed unconditionally (TMA zero-fills
// out-of-range rows/columns), so the DMMA stream has no predicates.
//
// KK: both operands K-major, 128-B rows, 128-B swizzle.  A lane reads the
//     16-byte chunk holding k = 8p + 2(lane&3) + {0,1}: one LDS.128 feeds
//     k-steps 2p and 2p+1 (the k order inside a stage is permuted
//     identically for A and B).  Physical chunk = (4p + (lane&3)) ^ (row&7):
//     4 wavefronts per 512 B, the minimum.
// MM: both operands M-major (16-column boxes, rows = k); lanes read rows
//     k = s + 4(lane&3): the 4 rows of a fragment fall on two different
//     (k & 7) swizzle phases, 2 wavefronts per 256 B, the minimum.
template <int J, bool MM, bool CHECK, int S = num_stages(J), int WN = 2>
__device__ __forceinline__ void mainloop(const Smem& sm, const CUtensorMap* mapA,
                                         const CUtensorMap* mapB, int m0, int n0, int kt0,
                                         int kt1, Acc<J>& acc, int wm, int wn, int lane, int nvf,
                                         int mvf, bool& bad, int mm3d = 0, int i0 = 0, int np_last = 2) {
  // i0: ring iterations already run by this CTA (stream-K: a second
  // segment continues the ring where the first left it)
  // np_last (KK only): 8-value k groups of the LAST k tile that hold any
  // k < K; 1 skips the group TMA zero-filled (K mod 16 in 1..8)
  (void)nvf;
  (void)mvf;
  const int nkt = kt1 - kt0;
  const bool leader = threadIdx.x == 0;
  if (leader) {
    if (i0 == 0) {
      tma_prefetch_desc(mapA);
      tma_prefetch_desc(mapB);
    }
    for (int i = 0; i < S && i < nkt; ++i) {
      const int g = i0 + i;
      if (g >= S) mbar_wait(&sm.empty[g % S], ((g / S) - 1) & 1);
      issue_stage<J, MM, WN>(sm, mapA, mapB, m0, n0, kt0 + i, g % S, mm3d);
    }
  }
  const int r8 = lane >> 2, c4 = lane & 3;
  // per-lane element offsets (in doubles) inside one stage
  int offA[2], offB[2];      // KK: chunk offsets for the two k pairs
  int rowA = 0, rowB = 0;    // KK: row bases
  int mmB[4];                // MM: per k-step B row offsets
  if (!MM) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      offA[p] = ((4 * p + c4) ^ kk_row(r8)) << 1;
      offB[p] = offA[p];
    }
    rowA = (wm * 32 + kk_row(r8)) * 16;
    rowB = (wn * 8 * J + kk_row(r8)) * 16;
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) mmB[s] = (s + 4 * c4) * 16;
  }
  for (int i = 0; i < nkt; ++i) {
    const int st = (i0 + i) % S;
    const uint32_t ph = ((i0 + i) / S) & 1;
    if (leader && i >= 1 && (i - 1) + S < nkt) {
      const int g = i0 + i - 1;
      const int ps = g % S;
      mbar_wait(&sm.empty[ps], (g / S) & 1);
      issue_stage<J, MM, WN>(sm, mapA, mapB, m0, n0, kt0 + (i - 1) + S, ps, mm3d);
    }
    mbar_wait(&sm.full[st], ph);
    const double* sa = sm.a + st * (bm_of(WN) * BK);
    const double* sb = sm.b + st * (nb16_of(J, WN) * 16 * BK);
    if (!MM) {
      const int np = (i == nkt - 1) ? np_last : 2;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        if (p >= np) break;
        double2 a2[4], b2[J];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          a2[mi] = *reinterpret_cast<const double2*>(sa + rowA + mi * 8 * 16 + offA[p]);
          if (CHECK) bad |= is_nonfinite(a2[mi].x) | is_nonfinite(a2[mi].y);
        }
#pragma unroll
        for (int nj = 0; nj < J; ++nj)
          b2[nj] = *reinterpret_cast<const double2*>(sb + rowB + nj * 8 * 16 + offB[p]);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < J; ++nj) dmma884(acc.v[mi][nj][0], acc.v[mi][nj][1], a2[mi].x, b2[nj].x);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int nj = 0; nj < J; ++nj) dmma884(acc.v[mi][nj][0], acc.v[mi][nj][1], a2[mi].y, b2[nj].y);
      }
    } else {
      // MM: fragment mi = 2q + e of this warp holds output rows
      // wm*32 + 16q + 2*(lane>>2) + e, so one LDS.128 at (row k, columns
      // 2*(lane>>2), +1) of box (wm*2 + q) feeds fragments 2q and 2q + 1.
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int k = s + 4 * c4;
        double2 a2[2];
        double bf[J];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          a2[q] = *reinterpret_cast<const double2*>(sa + (wm * 2 + q) * (16 * BK) + k * 16 + ((r8 ^ (k & 7)) << 1));
          if (CHECK) bad |= is_nonfinite(a2[q].x) | is_nonfinite(a2[q].y);
        }
        // B: fragments 2p and 2p+1 hold columns 16p + 2(lane>>2) + {0, 1}
        // of the warp's slice, so one LDS.128 feeds both; an odd
        // last fragment keeps the plain column order.
#pragma unroll
        for (int pq = 0; pq < J / 2; ++pq) {
          const int col = wn * 8 * J + pq * 16 + 2 * r8;
          const double2 b2 = *reinterpret_cast<const double2*>(
              sb + (col >> 4) * (16 * BK) + mmB[s] + ((((col & 15) >> 1) ^ (k & 7)) << 1));
          bf[2 * pq] = b2.x;
          bf[2 * pq + 1] = b2.y;
        }
        if (J & 1) {
          const int col = wn * 8 * J + (J - 1) * 8 + r8;
          bf[J - 1] = sb[(col >> 4) * (16 * BK) + mmB[s] + (((((col & 15) >> 1) ^ (k & 7)) << 1) | (col & 1))];
        }
#pragma unroll
        for (int nj = 0; nj < J; ++nj) {
          dmma884(acc.v[0][nj][0], acc.v[0][nj][1], a2[0].x, bf[nj]);
          dmma884(acc.v[1][nj][0], acc.v[1][nj][1], a2[0].y, bf[nj]);
          dmma884(acc.v[2][nj][0], acc.v[2][nj][1], a2[1].x, bf[nj]);
          dmma884(acc.v[3][nj][0], acc.v[3][nj][1], a2[1].y, bf[nj]);
        }
      }
    }
    // The fence makes every LDS of this stage complete before the release:
    // the arrive alone can be scheduled ahead of LDS still queued behind the
    // DMMAs, and the refill TMA would overwrite bytes not yet read.
    __syncwarp();
    __threadfence_block();
    if (lane == 0) mbar_arrive(&sm.empty[st]);
  }
}

template <int S>
__device__ __forceinline__ void init_barriers(const Smem& sm) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
}

// -------------------------------------------------------------- plain GEMM
struct StoreParams {
  double* c;       // direct output (splits == 1) or partial workspace
  int64_t ldc;
  int64_t split_stride;  // elements between split partials (0 when direct)
  int* bad_flag;         // nullable: set to 1 if a non-finite A entry was read
};

// Store one warp's accumulator tile (rows m0.., columns ncol0..) to out.
template <int J, bool MM>
__device__ __forceinline__ void store_acc(const Acc<J>& acc, double* out, int64_t ldc, const Tile& t, int m0,
                                          int ncol0, int wm, int lane) {
  const bool vec = ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  const int r8 = lane >> 2, c4 = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int row = MM ? m0 + wm * 32 + 16 * (mi >> 1) + 2 * r8 + (mi & 1) : m0 + wm * 32 + mi * 8 + kk_row(r8);
    if (row >= t.M) continue;
    double* rowp = out + (int64_t)row * ldc;
#pragma unroll
    for (int nj = 0; nj < J; ++nj) {
      if (MM && nj < (J & ~1)) {
        // paired fragments (see mainloop): element e of fragment 2p+h sits
        // at column 16p + 4(lane&3) + 2e + h
        if (nj & 1) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = ncol0 + (nj >> 1) * 16 + 4 * c4 + 2 * e;
          if (vec && col + 1 < t.N) {
            *reinterpret_cast<double2*>(rowp + col) = make_double2(acc.v[mi][nj][e], acc.v[mi][nj + 1][e]);
          } else {
            if (col < t.N) rowp[col] = acc.v[mi][nj][e];
            if (col + 1 < t.N) rowp[col + 1] = acc.v[mi][nj + 1][e];
          }
        }
      } else {
        // (MM with an odd last fragment keeps the plain column order)
        const int c0 = ncol0 + nj * 8 + (MM ? 2 * c4 : kk_col(c4, 0));
        const int c1 = ncol0 + nj * 8 + (MM ? 2 * c4 + 1 : kk_col(c4, 1));
        if (c0 < t.N) rowp[c0] = acc.v[mi][nj][0];
        if (c1 < t.N) rowp[c1] = acc.v[mi][nj][1];
      }
    }
  }
}

template <int J, bool MM, bool CHECK, int WN = 2, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB)
    gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                Tile t, StoreParams sp) {
  extern __shared__ unsigned char smem_raw[];
  constexpr int S = num_stages(J, WN, MINB);
  Smem sm = carve<J, S, S * stage_bytes(J, WN), WN>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int WMW = NCW / WN;  // warps along M
  const int wm = warp % WMW, wn = warp / WMW;
  init_barriers<S>(sm);
  if (t.sk > 0) {
    // stream-K: this CTA's contiguous run of (tile, k-tile) units, one
    // segment per tile it touches, the TMA ring continuing across segments
    const int G = gridDim.x, c = blockIdx.x;
    const long long U = (long long)t.m_tiles * t.n_tiles * t.k_tiles;
    long long u = ((long long)c * U) / G;
    const long long u1 = ((long long)(c + 1) * U) / G;
    int i0 = 0;
    while (u < u1) {
      const int tile = (int)(u / t.k_tiles);
      const int kt0 = (int)(u % t.k_tiles);
      const int kt1 = (int)min((long long)t.k_tiles, kt0 + (u1 - u));
      const int nt = tile % t.n_tiles;
      const int m0 = (tile / t.n_tiles) * bm_of(WN);
      const int n0 = nt * bn_of(J, WN);
      const int ncol0 = n0 + wn * 8 * J;
      const int nvf = max(0, min(J, (t.N - ncol0 + 7) / 8));
      const int mvf = max(0, min(4, (t.M - (m0 + wm * 32) + 7) / 8));
      const int cfirst = sk_cta_of((long long)tile * t.k_tiles, U, G);
      Acc<J> acc;
      acc.zero();
      bool bad = false;
      mainloop<J, MM, CHECK, S, WN>(sm, &mapA, &mapB, m0, n0, kt0, kt1, acc, wm, wn, lane, nvf, mvf, bad, t.mm3d, i0);
      if (CHECK && sp.bad_flag) {
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(sp.bad_flag, 1);
      }
      store_acc<J, MM>(acc, sp.c + (int64_t)(c - cfirst) * sp.split_stride, sp.ldc, t, m0, ncol0, wm, lane);
      if (kt1 == t.k_tiles) {
        // the tile's last segment: zero its unused slots so a finalize of
        // t.sk slices sums exactly the segments
        Acc<J> z;
        z.zero();
        for (int sl = c - cfirst + 1; sl < t.sk; ++sl)
          store_acc<J, MM>(z, sp.c + (int64_t)sl * sp.split_stride, sp.ldc, t, m0, ncol0, wm, lane);
      }
      i0 += kt1 - kt0;
      u += kt1 - kt0;
    }
    return;
  }
  const int bid = blockIdx.x;
  const int nt = bid % t.n_tiles;
  const int rest = bid / t.n_tiles;
  const int m0 = (rest % t.m_tiles) * bm_of(WN);
  const int split = rest / t.m_tiles;
  const int n0 = nt * bn_of(J, WN);
  const int kt0 = split * t.k_tiles_per_split;
  const int kt1 = min(t.k_tiles, kt0 + t.k_tiles_per_split);
  const int ncol0 = n0 + wn * 8 * J;
  const int nvf = max(0, min(J, (t.N - ncol0 + 7) / 8));
  const int mvf = max(0, min(4, (t.M - (m0 + wm * 32) + 7) / 8));
  Acc<J> acc;
  acc.zero();
  bool bad = false;
  mainloop<J, MM, CHECK, S, WN>(sm, &mapA, &mapB, m0, n0, kt0, kt1, acc, wm, wn, lane, nvf, mvf, bad, t.mm3d);
  if (CHECK && sp.bad_flag) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(sp.bad_flag, 1);
  }
  store_acc<J, MM>(acc, sp.c + (int64_t)split * sp.split_stride, sp.ldc, t, m0, ncol0, wm, lane);
}

// ------------------------------------------------ low-rank product epilogues
// C = U_r * Wt^T (K = r) is never stored as a whole; the epilogue consumes
// each 128 x 16J tile in registers.
enum LrMode { LR_STORE = 0, LR_ALM = 1, LR_RESID = 2 };

// a / b, correctly rounded (bitwise the IEEE quotient), for a divisor that is
// the same for every element: rb = RN(1 / b) comes from the host.  q0 = a rb
// is within 1.5 ulp; one residual correction makes it faithful, and by
// Markstein's theorem (rb the correctly rounded reciprocal, q faithful, the
// residual a - b q exact in an FMA) the second correction rounds to RN(a / b).
// 5 FP64 operations instead of the ~14-instruction division sequence.  Outside
// the exponent range where the residuals are exact (|a| in [2^-800, 2^800];
// includes a = 0, whose sign the corrections would lose) or when the host
// passes rb = 0 (b outside [2^-200, 2^200]) the plain division runs.
CU_DEV double div_const(double a, double b, double rb) {
  const uint32_t e = (static_cast<uint32_t>(__double2hiint(a)) >> 20) & 0x7ffu;
  if (rb != 0.0 && e - 223u <= 1600u) {
    const double q0 = a * rb;
    const double r0 = fma(-b, q0, a);
    const double q1 = fma(r0, rb, q0);
    const double r1 = fma(-b, q1, a);
    return fma(r1, rb, q1);
  }
  return a / b;
}

struct LrParams {
  int64_t ld;            // leading dimension of all n x n operands
  const double* m_mat;   // ALM: M ; RESID: A
  double* s;             // ALM: S out
  double* y;             // ALM: Y in/out
  double* g_next;        // ALM: next G out ; STORE: L out
  double mu, lam_over_mu, mu_next;
  double inv_mu, inv_mu_next;  // RN(1 / mu), RN(1 / mu_next) for div_const; 0: use the plain division
  int np_last;           // mainloop: k groups of the last k tile (1 when r mod 16 is in 1..8)
  double* part_sum;      // per-CTA partial sum of squares
  long long* part_cnt;   // per-CTA partial nnz
  int vec;               // 16-byte (double2) accesses allowed: ld even and every
                         // n x n operand 16-byte aligned (checked on the host)
};

// MINB: CTAs per SM (launch bound).  3 (with J = 2, 128 x 32 tiles and
// 4 row slots in flight per warp) keeps three CTAs' mainloops and
// streaming epilogues interleaved on each SM for the rank-r ALM update.
template <int J, int MODE, int MINB = 2>
__global__ void __launch_bounds__(THREADS, MINB)
    lowrank_kernel(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapW,
                   Tile t, LrParams p) {
  extern __shared__ unsigned char smem_raw[];
  __shared__ double red_sum[NCW];
  __shared__ long long red_cnt[NCW];
  Smem sm = carve<J, LR_STAGES, lr_data_bytes(J)>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bid = blockIdx.x;
  const int nt = bid % t.n_tiles;
  const int m0 = (bid / t.n_tiles) * BM;
  const int n0 = nt * 16 * J;
  init_barriers<LR_STAGES>(sm);
  const int wm = warp & 3, wn = warp >> 2;
  const int ncol0 = n0 + wn * 8 * J;
  const int nvf = max(0, min(J, (t.N - ncol0 + 7) / 8));
  const int mvf = max(0, min(4, (t.M - (m0 + wm * 32) + 7) / 8));
  if (MODE != LR_STORE) {
    // pull this tile's M (and Y) rows into L2 while the mainloop runs, so
    // the streaming epilogue finds them there (128-byte lines, no registers)
    const int tn = 16 * J;
    const int lines_per_row = (tn * 8 + 127) / 128;
    for (int e = threadIdx.x; e < BM * lines_per_row; e += THREADS) {
      const int row = e / lines_per_row, ln = e % lines_per_row;
      if (m0 + row >= t.M || n0 + ln * 16 >= t.N) continue;
      const int64_t off = (int64_t)(m0 + row) * p.ld + n0 + ln * 16;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p.m_mat + off));
      if (MODE == LR_ALM) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.y + off));
    }
  }
  Acc<J> acc;
  acc.zero();
  bool bad = false;
  mainloop<J, false, false, LR_STAGES>(sm, &mapU, &mapW, m0, n0, 0, t.k_tiles, acc, wm, wn, lane, nvf, mvf, bad, 0, 0,
                                       p.np_last);

  // Stage the 128 x 16J tile of L in shared memory (the pipeline buffers are
  // free now), then stream it row by row: each warp owns rows, lanes cover
  // 2 consecutive columns (double2), so every global access of M, Y, S, G is
  // a fully used 512-byte warp transaction; 4 rows in flight per warp.
  __syncthreads();
  constexpr int TN = 16 * J;        // tile columns
  constexpr int LDT = TN + 2;       // padded row (doubles), keeps double2 alignment
  double* tileL = sm.a;             // 128 x LDT doubles (<= 130 KB)
  const int r8 = lane >> 2, c4 = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int row = wm * 32 + mi * 8 + kk_row(r8);
#pragma unroll
    for (int nj = 0; nj < J; ++nj) {
      const int col = wn * 8 * J + nj * 8;
      tileL[row * LDT + col + kk_col(c4, 0)] = acc.v[mi][nj][0];
      tileL[row * LDT + col + kk_col(c4, 1)] = acc.v[mi][nj][1];
    }
  }
  __syncthreads();
  double ssum = 0.0;
  long long cnt = 0;
  const int ncols = min(TN, t.N - n0);
  const bool vec = p.vec != 0;
  // Warp w owns rows [16 w, 16 w + 16) of the tile.  LPR lanes cover one
  // row (2 columns each, double2), RPI = 32 / LPR rows per warp
  // instruction; RB instruction slots have all their M / Y loads issued
  // before any store (Y is read and written, so loads of later rows could
  // not otherwise move above earlier stores): RB x 2 x 512 B per warp in
  // flight.
  constexpr int LPR = (TN / 2 <= 16) ? TN / 2 : 32;
  constexpr int RPI = 32 / LPR;
  constexpr int RPW = BM / NCW;
  constexpr int SLOTS = RPW / RPI;
  constexpr int RB = MINB >= 3 ? 4 : 8;
  const int lrow = lane / LPR;
  const int c = 2 * (lane % LPR);
  const bool pair = vec && (c + 1 < ncols);
  for (int s0 = 0; s0 < SLOTS; s0 += RB) {
    double2 mv[RB], yv[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int row = warp * RPW + (s0 + q) * RPI + lrow;
      const int grow = m0 + row;
      mv[q] = make_double2(0.0, 0.0);
      yv[q] = make_double2(0.0, 0.0);
      if (MODE != LR_STORE && s0 + q < SLOTS && grow < t.M && c < ncols) {
        const int64_t idx = (int64_t)grow * p.ld + n0 + c;
        if (pair) {
          mv[q] = __ldcs(reinterpret_cast<const double2*>(p.m_mat + idx));
          if (MODE == LR_ALM) yv[q] = __ldcs(reinterpret_cast<const double2*>(p.y + idx));
        } else {
          mv[q].x = p.m_mat[idx];
          if (c + 1 < ncols) mv[q].y = p.m_mat[idx + 1];
          if (MODE == LR_ALM) {
            yv[q].x = p.y[idx];
            if (c + 1 < ncols) yv[q].y = p.y[idx + 1];
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int row = warp * RPW + (s0 + q) * RPI + lrow;
      const int grow = m0 + row;
      if (s0 + q >= SLOTS || grow >= t.M || c >= ncols) continue;
      const int64_t idx = (int64_t)grow * p.ld + n0 + c;
      const double2 l2 = *reinterpret_cast<const double2*>(tileL + row * LDT + c);
      const double lv[2] = {l2.x, l2.y};
      const double mvv[2] = {mv[q].x, mv[q].y}, yvv[2] = {yv[q].x, yv[q].y};
      double sv[2], yn[2], gv[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (e == 1 && c + 1 >= ncols) continue;
        const double l = lv[e];
        if (MODE == LR_RESID) {
          const double d = mvv[e] - l;
          ssum = fma(d, d, ssum);
        } else if (MODE == LR_ALM) {
          // rpca.py:211-214, operation order mirrored from the numpy source
          const double mm = mvv[e], yy = yvv[e];
          const double g = (mm - l) + div_const(yy, p.mu, p.inv_mu);
          const double ag = fabs(g) - p.lam_over_mu;
          const double sg = (g > 0.0) ? 1.0 : ((g < 0.0) ? -1.0 : g);
          sv[e] = sg * fmax(ag, 0.0);
          const double z = (mm - l) - sv[e];
          yn[e] = yy + p.mu * z;
          gv[e] = (mm - sv[e]) + div_const(yn[e], p.mu_next, p.inv_mu_next);
          ssum = fma(z, z, ssum);
          cnt += (fabs(sv[e]) > 1e-12) ? 1 : 0;
        }
      }
      if (MODE == LR_STORE) {
        if (pair) *reinterpret_cast<double2*>(p.g_next + idx) = make_double2(lv[0], lv[1]);
        else {
          p.g_next[idx] = lv[0];
          if (c + 1 < ncols) p.g_next[idx + 1] = lv[1];
        }
      } else if (MODE == LR_ALM) {
        if (pair) {
          // streaming (evict-first) stores: none of S, Y, G is re-read from L2
          __stcs(reinterpret_cast<double2*>(p.s + idx), make_double2(sv[0], sv[1]));
          __stcs(reinterpret_cast<double2*>(p.y + idx), make_double2(yn[0], yn[1]));
          __stcs(reinterpret_cast<double2*>(p.g_next + idx), make_double2(gv[0], gv[1]));
        } else {
          p.s[idx] = sv[0]; p.y[idx] = yn[0]; p.g_next[idx] = gv[0];
          if (c + 1 < ncols) { p.s[idx + 1] = sv[1]; p.y[idx + 1] = yn[1]; p.g_next[idx + 1] = gv[1]; }
        }
      }
    }
  }
  if (MODE != LR_STORE) {
    ssum = warp_sum(ssum);
    cnt = warp_sum(cnt);
    if (lane == 0) {
      red_sum[warp] = ssum;
      red_cnt[warp] = cnt;
    }
    __syncthreads();
    if (warp == 0 && lane == 0) {
      double s2 = 0.0;
      long long c2 = 0;
      for (int w = 0; w < NCW; ++w) {
        s2 += red_sum[w];
        c2 += red_cnt[w];
      }
      p.part_sum[bid] = s2;
      if (p.part_cnt) p.part_cnt[bid] = c2;
    }
  }
}

}  // namespace gemm
