"""Diagnose C4 iteration 0: |diag T| of corutv(M, ell=100, q=1, seed=0) on the
device (seeded Omega and explicit numpy Omega) vs the CPU oracle, and the rank
count against delta = 1/mu0."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import oracle as O
import paper_1906_04572_b200 as P
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
m_host = mat.cpu().numpy()
snorm, _ = P.dense.spectral_norm_iters(mat)
delta = snorm / 1.25
cfg = P.SketchConfig(ell=100, q_power=1, seed=0)
f1 = P.corutv(mat, cfg)
om = P.gaussian_matrix(n, 100, 0)
f2 = P.corutv(mat, cfg, omega=om)
t0 = time.perf_counter()
ref = O.corutv(m_host, 100, 1, omega=om)
t_cpu = time.perf_counter() - t0
d1 = f1.t.diagonal().abs().cpu().numpy(); d2 = f2.t.diagonal().abs().cpu().numpy(); dr = np.abs(np.diag(ref["t"]))
out = {"snorm": snorm, "delta": delta, "count_dev_seeded": int((d1 > delta).sum()),
       "count_dev_explicit": int((d2 > delta).sum()), "count_oracle": int((dr > delta).sum()),
       "diag_rel_diff_dev_vs_oracle": float(np.abs(d2 - dr).max() / dr[0]),
       "diag_seeded_vs_explicit_equal": bool(np.array_equal(d1, d2)),
       "diag_over_delta_first": (dr[:5] / delta).tolist(), "diag_over_delta_around_cut": (np.sort(dr / delta)[::-1][55:75]).tolist(),
       "perm_equal_first20": bool(np.array_equal(f2.perm.cpu().numpy()[:20], ref["perm"][:20])),
       "cpu_oracle_s": t_cpu}
print(json.dumps(out, indent=1))
