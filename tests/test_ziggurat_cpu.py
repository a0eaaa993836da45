"""The generated ziggurat tables (csrc/ziggurat_tables.cuh, written by
tools/derive_ziggurat.py) drive a pure-Python mirror of the device sampler
that must reproduce numpy's Generator.standard_normal bit for bit."""

import math
import re
from pathlib import Path

import numpy as np
import pytest

HDR = Path(__file__).resolve().parents[1] / "paper_1906_04572_b200" / "csrc" / "ziggurat_tables.cuh"
M128, M64, MULT = (1 << 128) - 1, (1 << 64) - 1, 0x2360ED051FC65DA44385DF649FCCF645


def tables():
    src = HDR.read_text()

    def arr(name):
        body = src.split(name + "[256] = {")[1].split("};")[0]
        toks = [t.strip() for t in body.replace("\n", " ").split(",") if t.strip()]
        return [int(t[:-3], 16) if t.endswith("ull") else float.fromhex(t) for t in toks]

    kr = float.fromhex(re.search(r"kR = (\S+);", src).group(1))
    kinv = float.fromhex(re.search(r"kInvR = (\S+);", src).group(1))
    return arr("ki"), arr("wi"), arr("fi"), kr, kinv


def stream(seed, n):
    ki, wi, fi, kr, kinv = tables()
    st = np.random.PCG64(seed).state["state"]
    s, inc = st["state"], st["inc"]
    out = []

    def u64():
        nonlocal s
        s = (s * MULT + inc) & M128
        x, rot = (s >> 64) ^ (s & M64), s >> 122
        return ((x >> rot) | (x << (64 - rot))) & M64

    def dbl():
        return (u64() >> 11) * (1.0 / 9007199254740992.0)

    while len(out) < n:
        r = u64()
        while True:
            idx = r & 0xFF
            rr = r >> 8
            rabs = (rr >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * wi[idx]
            x = -x if rr & 1 else x
            if rabs < ki[idx]:
                out.append(x)
                break
            if idx == 0:
                while True:
                    xx = -kinv * math.log1p(-dbl())
                    yy = -math.log1p(-dbl())
                    if yy + yy > xx * xx:
                        out.append(-(kr + xx) if (rabs >> 8) & 1 else kr + xx)
                        break
                break
            if (fi[idx - 1] - fi[idx]) * dbl() + fi[idx] < math.exp(-0.5 * x * x):
                out.append(x)
                break
            r = u64()
    return np.array(out)


@pytest.mark.parametrize("seed", [0, 1, 12345, 2**64 - 3])
def test_tables_reproduce_numpy(seed):
    assert np.array_equal(stream(seed, 60000), np.random.Generator(np.random.PCG64(seed)).standard_normal(60000))
