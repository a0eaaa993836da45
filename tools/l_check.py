"""C4: is the returned L consistent with the solve?  Checks the reference's own
identity |M - L - S|_F / |M|_F == residuals[-1] (pkg/tests/test_rpca.py:146-157)
and the STORE-mode low-rank product against torch at C4 size."""
import json, math, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import rpca as R
torch.cuda.set_device(0); dev = torch.device("cuda", 0)
n, k = 10000, 50
g = torch.Generator(device=dev); g.manual_seed(777)
x = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
y = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
mat = x @ y.T
nnz = n * n // 20
pos = torch.randperm(n * n, generator=g, device=dev)[:nnz]
vals = (torch.rand((nnz,), generator=g, dtype=torch.float64, device=dev) * 1000.0) - 500.0
mat.view(-1)[pos] += vals
snorm = P.spectral_norm(mat)
cfg = P.AlmConfig(lam=1 / math.sqrt(n), tol=1e-7, ell=2 * k, q_power=1, seed=0, mu0=1.25 / snorm)
cap = {}
orig = R._lowrank_device
def spy(u, t, v, r):
    out = orig(u, t, v, r)
    ref = u[:, :r] @ (t[:r, :] @ v.T)
    cap["store_vs_torch"] = float((out - ref).norm() / ref.norm())
    return out
R._lowrank_device = spy
sol = P.alm_corutv(mat, cfg)
ident = float((mat - sol.l - sol.s).norm() / mat.norm())
out = {"identity_rel_err": abs(ident - sol.residuals[-1]) / sol.residuals[-1], "zeta_last": sol.residuals[-1],
       "recomputed": ident, **cap, "L_norm": float(sol.l.norm()), "L_vs_plant": float((sol.l - x @ y.T).norm() / (x @ y.T).norm())}
print(json.dumps(out))
