"""C4 alm_corutv with a numpy input and numpy outputs (the reference user's
call), wall time split."""
import math
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
n, k = 10000, 50
g = torch.Generator(device=dev)
g.manual_seed(777)
x = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
y = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
mat = x @ y.T
pos = torch.randperm(n * n, generator=g, device=dev)[:n * n // 20]
mat.view(-1)[pos] += (torch.rand((n * n // 20,), generator=g, dtype=torch.float64, device=dev) * 1000.0) - 500.0
host = mat.cpu().numpy()
snorm = P.spectral_norm(mat)
cfg = P.AlmConfig(lam=1 / math.sqrt(n), tol=1e-7, ell=2 * k, q_power=1, seed=0, mu0=1.25 / snorm)
for _ in range(3):
    t0 = time.perf_counter()
    sol = P.alm_corutv(host, cfg)
    print(f"alm_corutv(numpy) e2e {1e3 * (time.perf_counter() - t0):.1f} ms, {sol.iterations} iterations, "
          f"outputs {type(sol.l).__name__}", flush=True)
