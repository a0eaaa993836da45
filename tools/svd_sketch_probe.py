"""sor_svd / tsr_svd at the C3 shape (device-resident A), per-call wall time."""
import sys
import time
sys.path.insert(0, '.')
import torch
import bench
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
m, n = 131072, 32768
a = bench.gen_rows_device(torch, "c3", 0, m, torch.device("cuda", 0))
for name, fn, cfg in (("corutv", P.corutv, P.SketchConfig(ell=110, q_power=2)),
                      ("sor_svd", P.sor_svd, P.SketchConfig(ell=110, q_power=2)),
                      ("tsr_svd", P.tsr_svd, P.SketchConfig(ell=110)),
                      ("corutv", P.corutv, P.SketchConfig(ell=110, q_power=2))):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(a, cfg)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(name, " ".join(f"{t:.1f}" for t in ts), "ms", flush=True)
