// Device generator for the reference's Gaussian test matrix:
//   np.random.Generator(np.random.PCG64(seed)).standard_normal((rows, cols))
// (sketch.py:63-68), bit-identical.
//
// PCG64 (128-bit LCG, XSL-RR output) from the host-expanded (state, inc);
// the 256-layer ziggurat of numpy's random_standard_normal with tables in
// ziggurat_tables.cuh (tools/derive_ziggurat.py).  The stream is
// sequential (a sample consumes 1 draw 99.3% of the time, more on the wedge
// and tail paths), so generation is three data-parallel passes:
//   1. eval:    every raw position p is evaluated as if a sample started there
//               (state by LCG jump-ahead): value, draws consumed c(p), tail flag;
//   2. resolve: a position starts a sample iff no earlier sample's extra draws
//               cover it -- a 16-state automaton whose transition maps are
//               composed by a parallel exclusive scan;
//   3. scatter: sample index = number of starts before p (exclusive scan);
//               write row-major (and optionally transposed) output.
// Arithmetic that feeds decisions or values uses explicitly rounded
// intrinsics (no FMA contraction, as in numpy's scalar C).  Tail-path samples
// (value = r + (-log1p(-u)/r)) are finished on the host with the same libm
// log1p numpy calls, so every value is bit-identical.
#pragma once
#include <stdint.h>

#include "common.cuh"
#include "ziggurat_tables.cuh"

namespace rng {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | (u128)lo;
}

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return mk128(0x2360ed051fc65da4ull, 0x4385df649fccf645ull);
}

// state after `delta` more steps (Brown's algorithm for LCG jump-ahead)
__host__ __device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

struct Pcg {
  u128 s, inc;
  __device__ __forceinline__ uint64_t next() {
    s = s * pcg_mult() + inc;
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const uint64_t x = hi ^ lo;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  __device__ __forceinline__ double next_double() {
    return (double)(next() >> 11) * (1.0 / 9007199254740992.0);
  }
};

struct Eval {
  double val;   // sample value, or the accepted tail uniform u1 (tail != 0)
  uint32_t cnt; // draws consumed
  uint32_t tail;  // 0, or 1 + sign bit for a tail-path sample
};

// numpy random_standard_normal starting at the draw `r0` (already taken
// from g).  Matches distributions.c: fast path, wedge test, tail loop.
__device__ __forceinline__ Eval sample_from(uint64_t r0, Pcg g) {
  uint32_t cnt = 1;
  uint64_t r = r0;
  for (;;) {
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, zig::wi[idx]);
    if (sign) x = -x;
    if (rabs < zig::ki[idx]) return Eval{x, cnt, 0};
    if (idx == 0) {
      for (;;) {
        const double u1 = g.next_double();
        const double u2 = g.next_double();
        cnt += 2;
        const double xx = __dmul_rn(-zig::kInvR, log1p(-u1));
        const double yy = -log1p(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) return Eval{u1, cnt, 1u + (uint32_t)((rabs >> 8) & 1)};
      }
    } else {
      const double u = g.next_double();
      cnt += 1;
      const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(zig::fi[idx - 1], -zig::fi[idx]), u), zig::fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return Eval{x, cnt, 0};
    }
    r = g.next();
    cnt += 1;
  }
}

constexpr int RUN = 16;  // consecutive raw positions per thread

// pass 1: evaluate every position p in [0, P)
__global__ void eval_kernel(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t P,
                            double* __restrict__ val, uint8_t* __restrict__ cnt,
                            uint8_t* __restrict__ tail) {
  const u128 s0 = mk128(s_hi, s_lo), inc = mk128(i_hi, i_lo);
  const int64_t nruns = (P + RUN - 1) / RUN;
  for (int64_t run = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; run < nruns;
       run += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = run * RUN;
    Pcg g{pcg_advance(s0, inc, (uint64_t)p0), inc};
    for (int t = 0; t < RUN && p0 + t < P; ++t) {
      const uint64_t r = g.next();
      const Eval e = sample_from(r, g);
      val[p0 + t] = e.val;
      cnt[p0 + t] = (uint8_t)min(e.cnt, 255u);
      tail[p0 + t] = (uint8_t)e.tail;
    }
  }
}

// pass 2: which raw positions start a sample.  Reading the positions in
// order is a finite-state automaton over "draws still to skip" (0..15): at
// state 0 the position starts a sample and the state becomes cnt - 1, else
// the state decrements.  Each position's transition is a 16-entry map packed
// in nibbles; the exclusive scan of map compositions gives every position's
// entry state (nibble 0 of the prefix map) in parallel.
constexpr uint64_t kIdentityMap = 0xFEDCBA9876543210ull;

struct CountToMap {
  __host__ __device__ __forceinline__ uint64_t operator()(const uint8_t& c) const {
    // entry 0 -> c - 1, entry s > 0 -> s - 1
    const uint64_t down = kIdentityMap << 4;  // nibble s holds s - 1 (s >= 1)
    return (down & ~0xFull) | (uint64_t)((c - 1) & 0xF);
  }
};

struct ComposeMaps {  // apply a, then b
  __host__ __device__ __forceinline__ uint64_t operator()(const uint64_t& a, const uint64_t& b) const {
    uint64_t out = 0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const uint64_t as = (a >> (4 * s)) & 0xF;
      out |= ((b >> (4 * as)) & 0xF) << (4 * s);
    }
    return out;
  }
};

// starts[p] = 1 iff the automaton enters p in state 0; flags counts > 16
__global__ void starts_from_maps_kernel(const uint64_t* __restrict__ prefix, const uint8_t* __restrict__ cnt,
                                        int64_t* __restrict__ starts, int64_t P, int* too_long) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    starts[p] = ((prefix[p] & 0xF) == 0) ? 1 : 0;
    if (cnt[p] > 16) atomicOr(too_long, 1);
  }
}

// pass 3: sample index of each start; write out (rows x cols, ld) and, if
// outT != nullptr, its transpose (cols x rows, ldT).  Tail samples append
// (index, u1, sign) to `tails` for the host to finish.
__global__ void scatter_kernel(const double* __restrict__ val, const int64_t* __restrict__ starts,
                               const uint8_t* __restrict__ tail, const int64_t* __restrict__ rank,
                               int64_t P, int64_t N, int64_t cols, double* __restrict__ out, int64_t ld,
                               double* __restrict__ outT, int64_t ldT, int64_t* tail_idx,
                               double* tail_u, int* tail_sign, unsigned long long* n_tail,
                               int tail_cap) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!starts[p]) continue;
    const int64_t k = rank[p];
    if (k >= N) continue;
    const int64_t i = k / cols, j = k % cols;
    double v = val[p];
    if (tail[p]) {
      const unsigned long long slot = atomicAdd(n_tail, 1ull);
      if ((int)slot < tail_cap) {
        tail_idx[slot] = k;
        tail_u[slot] = v;
        tail_sign[slot] = (int)tail[p] - 1;
      }
      v = 0.0;  // patched by the host
    }
    out[i * ld + j] = v;
    if (outT) outT[j * ldT + i] = v;
  }
}

// host patch: scatter finished tail values (n small)
__global__ void patch_kernel(const int64_t* __restrict__ idx, const double* __restrict__ v, int n,
                             int64_t cols, double* __restrict__ out, int64_t ld, double* __restrict__ outT,
                             int64_t ldT) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t k = idx[t], i = k / cols, j = k % cols;
  out[i * ld + j] = v[t];
  if (outT) outT[j * ldT + i] = v[t];
}

}  // namespace rng
