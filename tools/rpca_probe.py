"""Per-iteration breakdown of the C4 ALM solve (decompose vs fused update)
and the spectral-norm cost, with syncs around each phase."""
import ctypes
import math
import sys
import time
sys.path.insert(0, '.')
import torch
import bench
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import rpca, _lib
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
for rep in range(2):
    t0 = time.perf_counter()
    snorm, sit = P.dense.spectral_norm_iters(mat)
    torch.cuda.synchronize()
    print(f"spectral_norm: {1e3 * (time.perf_counter() - t0):.1f} ms, {sit} iters", flush=True)
cfg = P.AlmConfig(lam=1 / math.sqrt(n), tol=1e-7, ell=2 * k, q_power=1, seed=0, mu0=1.25 / snorm)
P.alm_corutv(mat, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
sol = P.alm_corutv(mat, cfg)
torch.cuda.synchronize()
print(f"alm total {1e3 * (time.perf_counter() - t0):.1f} ms, {sol.iterations} iters", flush=True)
rec = []
orig_trunc = rpca.corutv_truncated
def trunc(*a, **kw):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = orig_trunc(*a, **kw)
    torch.cuda.synchronize(); rec.append(("decomp", a[1].ell, r[1], 1e3 * (time.perf_counter() - t)))
    return r
rpca.corutv_truncated = trunc
orig_call = _lib.Handle.call
def call(self, name, *a):
    if name != "corutv_alm_update":
        return orig_call(self, name, *a)
    torch.cuda.synchronize(); t = time.perf_counter()
    r = orig_call(self, name, *a)
    torch.cuda.synchronize(); rec.append(("update", 0, 0, 1e3 * (time.perf_counter() - t)))
    return r
_lib.Handle.call = call
t0 = time.perf_counter()
sol = P.alm_corutv(mat, cfg)
torch.cuda.synchronize()
print(f"instrumented total {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
for i in range(0, len(rec), 2):
    d, u = rec[i], rec[i + 1]
    print(f"iter {i // 2:2d} ell {d[1]:4d} r {d[2]:4d}: decompose {d[3]:7.3f} ms  update {u[3]:6.3f} ms")
