"""tsr_svd at the C3 shape (device-resident A) for narrow ell: per-call time
and the leading singular values (A/B of the one-pass dual sketch against two
sweeps: CORUTV_DUAL_OFF=1)."""
import sys
import time
sys.path.insert(0, '.')
import torch
import bench
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
m, n = 131072, 32768
a = bench.gen_rows_device(torch, "c3", 0, m, torch.device("cuda", 0))
for ell in (8, 16):
    cfg = P.SketchConfig(ell=ell, seed=3)
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = P.tsr_svd(a, cfg)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    s = f.sigma
    s = s.cpu().numpy() if hasattr(s, "cpu") else s
    print(f"ell={ell} tsr_svd", " ".join(f"{t:.2f}" for t in ts), "ms  sigma[:3]", [float(x) for x in s[:3]], flush=True)
