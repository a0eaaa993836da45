"""C4-size spectral norm only (for an ncu launch list)."""
import sys
import time
sys.path.insert(0, '.')
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
nnz = n * n // 20
pos = torch.randperm(n * n, generator=g, device=dev)[:nnz]
vals = (torch.rand((nnz,), generator=g, dtype=torch.float64, device=dev) * 1000.0) - 500.0
mat.view(-1)[pos] += vals
torch.cuda.synchronize()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for _ in range(reps):
    t0 = time.perf_counter()
    s, it = P.dense.spectral_norm_iters(mat)
    torch.cuda.synchronize()
    print(f"{1e3 * (time.perf_counter() - t0):.1f} ms {it} iters {s!r}", flush=True)
