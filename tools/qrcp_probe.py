"""Time the QRCP of an ell x ell core alone via corutv on a small matrix
(ncu launch list target) -- prints the decomposition wall time."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
ell = int(sys.argv[1])
g = torch.Generator(device="cuda"); g.manual_seed(1)
a = torch.randn((4 * ell, 2 * ell), generator=g, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    P.corutv(a, P.SketchConfig(ell=ell, q_power=0, seed=2))
    torch.cuda.synchronize()
print(f"ell {ell}: {1e3 * (time.perf_counter() - t0):.3f} ms")
