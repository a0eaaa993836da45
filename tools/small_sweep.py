"""corutv on an n x n Gaussian-plus-low-rank matrix for a given ell (ncu per-kernel timing of
the one-CTA kernels at that ell)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1906_04572_b200 as P
ell = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
torch.cuda.set_device(0)
g = torch.Generator(device='cuda'); g.manual_seed(1)
a = torch.randn(n, 64, generator=g, dtype=torch.float64, device='cuda') @ torch.randn(64, n, generator=g, dtype=torch.float64, device='cuda')
a += 1e-3 * torch.randn(n, n, generator=g, dtype=torch.float64, device='cuda')
cfg = P.SketchConfig(ell=ell, q_power=1)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); P.corutv(a, cfg); torch.cuda.synchronize()
    print(ell, "%.3f ms" % ((time.perf_counter() - t0) * 1e3))
