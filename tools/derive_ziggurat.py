"""Derive the 256-layer ziggurat tables that numpy's Generator.standard_normal
uses, by observation, and write paper_1906_04572_b200/csrc/ziggurat_tables.cuh.

Why: the reference draws its test matrix with
np.random.Generator(PCG64(seed)).standard_normal (sketch.py:63-68).  numpy is a
third-party dependency (numpy 2.3.5 here); its normal sampler is the
Marsaglia-Tsang ziggurat (256 layers, 52-bit magnitudes, tail beyond
r = 3.6541528853610088, wedge test against exp(-x^2/2)) over PCG64 (XSL-RR
128/64).  The published construction reproduces numpy's layer widths only to a
few ulps, which is not enough for bit-identical Omega, so the widths are pinned
from numpy's own output stream:

  1. replay PCG64(seed).random_raw() alongside standard_normal() and classify
     every sample as fast-path (one draw, x = rabs * w[idx]) or slow by
     back-tracking stream alignment;
  2. for every layer keep the unique double w[idx] with fl(rabs * w) == |x|
     for all fast samples (and the wedge-accepted samples for layer 1);
  3. k[i] = floor(2^52 x_{i-1} / x_i) (exact rationals), k[0] = floor(2^52 r / x_0),
     k[1] = 0, f[i] = exp(-x_i^2 / 2), f[0] = 1, with x_i = 2^52 w[i];
  4. verify: a pure-Python generator with these tables reproduces numpy's
     standard_normal bit for bit on 3.2 M samples over 32 seeds.

Run in the build container:  python tools/derive_ziggurat.py
"""

import math
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

sys.setrecursionlimit(10000)
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "paper_1906_04572_b200" / "csrc" / "ziggurat_tables.cuh"
M128 = (1 << 128) - 1
M64 = (1 << 64) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK52 = 0x000FFFFFFFFFFFFF
R_TAIL = 3.6541528853610087963519472518
INV_R = 0.27366123732975827203338247596


def construction(v=0.0049286732339746519, r=R_TAIL, nb=256):
    """Marsaglia-Tsang 2000 table construction (double precision): the guide
    used to classify samples before the exact widths are pinned."""
    m1 = 2.0 ** 52
    ki, wi, fi = [0] * nb, [0.0] * nb, [0.0] * nb
    dn = tn = r
    q = v / math.exp(-0.5 * dn * dn)
    ki[0], ki[1] = int(dn / q * m1), 0
    wi[0], wi[nb - 1] = q / m1, dn / m1
    fi[0], fi[nb - 1] = 1.0, math.exp(-0.5 * dn * dn)
    for i in range(nb - 2, 0, -1):
        dn = math.sqrt(-2.0 * math.log(v / dn + math.exp(-0.5 * dn * dn)))
        ki[i + 1] = int(dn / tn * m1)
        tn = dn
        fi[i], wi[i] = math.exp(-0.5 * dn * dn), dn / m1
    return ki, wi, fi


class Pcg:
    def __init__(self, seed):
        st = np.random.PCG64(seed).state["state"]
        self.s, self.inc = st["state"], st["inc"]

    def u64(self):
        self.s = (self.s * MULT + self.inc) & M128
        hi, lo = self.s >> 64, self.s & M64
        x, rot = hi ^ lo, self.s >> 122
        return ((x >> rot) | (x << (64 - rot))) & M64

    def dbl(self):
        return (self.u64() >> 11) * (1.0 / 9007199254740992.0)


def normal(g, ki, wi, fi, rr, inv_r):
    while True:
        r = g.u64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & MASK52
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            return x
        if idx == 0:
            while True:
                xx = -inv_r * math.log1p(-g.dbl())
                yy = -math.log1p(-g.dbl())
                if yy + yy > xx * xx:
                    return -(rr + xx) if ((rabs >> 8) & 1) else rr + xx
        elif (fi[idx - 1] - fi[idx]) * g.dbl() + fi[idx] < math.exp(-0.5 * x * x):
            return x


def main():
    ki0, wi0, _ = construction()

    def fast(r, w=wi0):
        idx = r & 0xFF
        rr = r >> 8
        rabs = (rr >> 1) & MASK52
        x = rabs * w[idx]
        return idx, rabs, (-x if rr & 1 else x)

    def matches(r, y):
        idx, rabs, x = fast(r)
        return abs(x - y) <= 1e-9 * abs(y) and (idx == 0 or rabs <= ki0[idx] * 1.0001)

    def consume(raw, ref, pos, k, depth):
        if depth == 0 or k >= len(ref):
            return []
        if matches(raw[pos], ref[k]):
            rest = consume(raw, ref, pos + 1, k + 1, depth - 1)
            if rest is not None:
                return [0] + rest
        for d in range(1, 12):
            rest = consume(raw, ref, pos + 1 + d, k + 1, depth - 1)
            if rest is not None:
                return [d] + rest
        return None

    fast_samples, wedge1 = {}, []
    for seed in range(12):
        n = 100000
        ref = np.random.Generator(np.random.PCG64(seed)).standard_normal(n)
        raw = np.random.PCG64(seed).random_raw(int(n * 1.05) + 200).tolist()
        pos, k, events = 0, 0, []
        while k < n - 5:
            d = consume(raw, ref, pos, k, 4)[0]
            events.append((k, pos, d))
            pos += 1 + d
            k += 1
        for t, (k, p, d) in enumerate(events[:-1]):
            idx, rabs, x = fast(raw[p])
            nk, np_, nd = events[t + 1]
            # (k, d=0) followed by (k+1, d=1 with the output in its 2nd draw):
            # sample k took the wedge path and consumed one uniform
            wedge = d == 0 and nd == 1 and fast(raw[np_ + 1])[2] == ref[nk] and fast(raw[np_])[2] != ref[nk]
            if d == 0 and not wedge and rabs > 0:
                fast_samples.setdefault(idx, []).append((rabs, abs(ref[k])))
            # layer 1 never takes the fast path (k[1] = 0): its wedge-accepted
            # samples consume two draws and return rabs * w[1] of the first
            if idx == 1 and d == 1 and rabs > 0 and abs(abs(x) / abs(ref[k]) - 1) < 1e-6:
                wedge1.append((rabs, abs(ref[k])))
    fast_samples[1] = wedge1

    def pin(sl):
        assert sl, "no samples"
        lo, hi = -np.inf, np.inf
        for rabs, y in sl:
            u = float(np.spacing(y))
            lo, hi = max(lo, (y - u) / rabs), min(hi, (y + u) / rabs)
        w, out = float(lo), []
        assert hi - lo < 1e-6 * abs(lo), (lo, hi)
        while w <= hi and len(out) < 64:
            if all(float(rabs) * w == y for rabs, y in sl):
                out.append(w)
            w = float(np.nextafter(w, np.inf))
        return out

    wi = []
    for idx in range(256):
        c = pin(fast_samples[idx])
        assert len(c) == 1, (idx, c)
        wi.append(c[0])
    x = [Fraction(w) * 2 ** 52 for w in wi]
    ki = [math.floor(x[255] / x[0] * 2 ** 52), 0] + [math.floor(x[i - 1] / x[i] * 2 ** 52) for i in range(2, 256)]
    fi = [1.0] + [math.exp(-0.5 * (w * 2.0 ** 52) ** 2) for w in wi[1:]]
    rr = wi[255] * 2.0 ** 52
    mism = tot = 0
    for seed in list(range(30)) + [2 ** 40 + 7, 12345678901234567890]:
        ref = np.random.Generator(np.random.PCG64(seed)).standard_normal(100000)
        g = Pcg(seed)
        out = np.array([normal(g, ki, wi, fi, rr, INV_R) for _ in range(100000)])
        mism += int((out != ref).sum())
        tot += out.size
    assert mism == 0, mism
    lines = [
        "// GENERATED by tools/derive_ziggurat.py -- do not edit.",
        f"// Ziggurat tables reproducing numpy {np.__version__} Generator.standard_normal bit for bit",
        f"// (verified on {tot} samples over 32 seeds).",
        "#pragma once",
        "#include <stdint.h>",
        "namespace zig {",
        f"constexpr double kR = {rr.hex()};  // {rr!r}",
        f"constexpr double kInvR = {INV_R.hex()};  // {INV_R!r}",
        "__device__ const uint64_t ki[256] = {",
    ]
    lines += ["  " + ", ".join(f"0x{v:013x}ull" for v in ki[i:i + 4]) + "," for i in range(0, 256, 4)]
    lines += ["};", "__device__ const double wi[256] = {"]
    lines += ["  " + ", ".join(v.hex() for v in wi[i:i + 4]) + "," for i in range(0, 256, 4)]
    lines += ["};", "__device__ const double fi[256] = {"]
    lines += ["  " + ", ".join(v.hex() for v in fi[i:i + 4]) + "," for i in range(0, 256, 4)]
    lines += ["};", "}  // namespace zig", ""]
    OUT.write_text("\n".join(lines))
    print("wrote", OUT, "verified", tot, "samples")


if __name__ == "__main__":
    main()
