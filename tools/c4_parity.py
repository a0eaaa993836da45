"""Full-size RPCA parity (BASELINE configs[3], C4, n = 10000) against the CPU
oracle, run on the GPU box (the oracle needs ~5 min of 16-core OpenBLAS).

Same M for both (synthesised on the device, copied to the host); the oracle
computes its own mu0 = 1.25/|M|_2 (dense.py:405-442 block power iteration),
and the device ALM is run with that mu0 so the two loops are comparable; the
device spectral norm is compared separately.  Writes gpurun_out/c4_parity.json.
"""
import json
import math
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import oracle as O
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
m_host = mat.cpu().numpy()
out = {}
t0 = time.perf_counter()
snorm_dev, it_dev = P.dense.spectral_norm_iters(mat)
out["spectral_norm_device"] = snorm_dev
out["spectral_norm_device_iters"] = it_dev
out["spectral_norm_device_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
snorm_ref, it_ref = O.spectral_norm(m_host)
out["spectral_norm_oracle"] = snorm_ref
out["spectral_norm_oracle_iters"] = it_ref
out["spectral_norm_oracle_s"] = time.perf_counter() - t0
out["spectral_norm_rel_diff"] = abs(snorm_dev - snorm_ref) / snorm_ref
mu0 = 1.25 / snorm_ref
cfg = dict(lam=1 / math.sqrt(n), tol=1e-7, q_power=1, seed=0, mu0=mu0)
torch.cuda.synchronize()
t0 = time.perf_counter()
sol = P.alm_corutv(mat, P.AlmConfig(ell=2 * k, **cfg))
torch.cuda.synchronize()
out["device_alm_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
ref = O.alm_corutv(m_host, ell=2 * k, **cfg)
out["oracle_alm_s"] = time.perf_counter() - t0
l_dev, s_dev = sol.l.cpu().numpy(), sol.s.cpu().numpy()
out.update({
    "iterations": [sol.iterations, ref["iterations"]],
    "ell_history": [sol.ell_history, ref["ell_history"]],
    "rank_history": [sol.rank_history, ref["rank_history"]],
    "nnz_history_equal": sol.nnz_history == ref["nnz_history"],
    "rank_of_l": [sol.rank_of_l, ref["rank_of_l"]],
    "nnz_of_s": [sol.nnz_of_s, ref["nnz_of_s"]],
    "final_residual": [sol.residuals[-1], ref["residuals"][-1]],
    "residuals_max_rel_diff": float(np.max(np.abs(np.array(sol.residuals) - np.array(ref["residuals"][:len(sol.residuals)])) / np.array(ref["residuals"][:len(sol.residuals)]))) if sol.iterations == ref["iterations"] else None,
    "L_rel_diff": float(np.linalg.norm(l_dev - ref["l"]) / np.linalg.norm(ref["l"])),
    "S_rel_diff": float(np.linalg.norm(s_dev - ref["s"]) / np.linalg.norm(ref["s"])),
    "cpu_cores": __import__("os").cpu_count(),
})
print(json.dumps(out))
json.dump(out, open("gpurun_out/c4_parity.json", "w"), indent=1)
