"""Stress the low-rank STORE kernel: count wrong elements vs torch over repeats.
usage: python tools/store_dbg.py [libpath]"""
import sys; sys.path.insert(0, '.')
import torch
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import _lib
if len(sys.argv) > 1:
    _lib._lib = _lib.load_library(sys.argv[1])
torch.cuda.set_device(0)
tot = 0
for (rows, cols, ell, r) in ((4096, 4096, 600, 600), (10000, 10000, 51, 50), (4096, 4096, 51, 50), (8192, 8192, 130, 100)):
    g = torch.Generator(device="cuda"); g.manual_seed(rows + cols + ell)
    u = torch.randn((rows, ell), generator=g, dtype=torch.float64, device="cuda")
    t = torch.triu(torch.randn((ell, ell), generator=g, dtype=torch.float64, device="cuda"))
    v = torch.randn((cols, ell), generator=g, dtype=torch.float64, device="cuda")
    ref = u[:, :r] @ (t[:r, :] @ v.T)
    bad = []
    for rep in range(10):
        out = P.rpca._lowrank_device(u, t, v, r)
        bad.append(int(((out - ref).abs() > 1e-9 * ref.abs().max()).sum()))
    tot += sum(bad)
    print((rows, cols, ell, r), "bad per rep", bad, flush=True)
print("TOTAL_BAD", tot)
