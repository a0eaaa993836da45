"""GPU busy time vs wall time of one C4 ALM solve (torch.profiler / CUPTI
records every kernel, ours included)."""
import math
import sys
import time
sys.path.insert(0, '.')
import torch
from torch.profiler import ProfilerActivity, profile
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
n, k = 10000, 50
g = torch.Generator(device=dev)
g.manual_seed(777)
x = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
y = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
mat = x @ y.T
nnz = n * n // 20
pos = torch.randperm(n * n, generator=g, device=dev)[:nnz]
vals = (torch.rand((nnz,), generator=g, dtype=torch.float64, device=dev) * 1000.0) - 500.0
mat.view(-1)[pos] += vals
snorm = P.spectral_norm(mat)
cfg = P.AlmConfig(lam=1 / math.sqrt(n), tol=1e-7, ell=2 * k, q_power=1, seed=0, mu0=1.25 / snorm)
P.alm_corutv(mat, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    sol = P.alm_corutv(mat, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
busy = sum(e.device_time_total for e in ev if e.device_time_total) / 1e3
print(f"wall {wall * 1e3:.1f} ms, kernels+copies {busy:.1f} ms over {len(ev)} events, iterations {sol.iterations}")
agg = {}
for e in ev:
    key = e.name[:60]
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += e.device_time_total / 1e3
for kname, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{t:9.3f} ms {c:6d}  {kname}")
