"""One C4-size decompose at a large sample size (the ALM's ell = 600 step)."""
import sys
import time
sys.path.insert(0, '.')
import torch
import os
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import _lib
if os.environ.get("CORUTV_LIB"):
    _lib._lib = _lib.load_library(os.environ["CORUTV_LIB"])
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
n = 10000
ell = int(sys.argv[1]) if len(sys.argv) > 1 else 600
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device=dev)
g.manual_seed(777)
x = torch.randn((n, 50), generator=g, dtype=torch.float64, device=dev) / 100.0
mat = x @ x.T + 0.01 * torch.randn((n, n), generator=g, dtype=torch.float64, device=dev)
cfg = P.SketchConfig(ell=ell, q_power=1, seed=3)
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f, r = P.sketch.corutv_truncated(mat, cfg, 1e-3)
    torch.cuda.synchronize()
    print(f"ell {ell}: {1e3 * (time.perf_counter() - t0):.2f} ms r={r}", flush=True)
