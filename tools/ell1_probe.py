"""One ALM-sized decomposition at ell = 1 (C4's 20 low-rank iterations):
10000^2, q = 1, seeded Omega, truncated at delta (corutv_truncated).
Timed with CUDA events; run under ncu for the launch list."""
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_1906_04572_b200 as P
from paper_1906_04572_b200.sketch import corutv_truncated

torch.cuda.set_device(0)
n = 10000
ell = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
A = torch.randn(n, n, dtype=torch.float64, device='cuda')
cfg = P.SketchConfig(ell=ell, q_power=1, seed=3)
for _ in range(3):
    corutv_truncated(A, cfg, 1e3)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    corutv_truncated(A, cfg, 1e3)
torch.cuda.synchronize()
print(f"ell {ell}: {(time.perf_counter() - t0) / reps * 1e3:.3f} ms per truncated decomposition")
