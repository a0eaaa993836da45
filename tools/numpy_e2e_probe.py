"""corutv on a pageable numpy array at the C3 shape (what a reference user
passes), vs the pinned-tensor path."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
m, n = 131072, 32768
a = bench.gen_rows_device(torch, "c3", 0, m, torch.device("cuda", 0))
host = np.empty((m, n), dtype=np.float64)
host[:] = a.cpu().numpy() if False else 0.0
t0 = time.perf_counter()
torch.from_numpy(host).copy_(a)
print(f"D2H into pageable numpy: {time.perf_counter() - t0:.2f} s", flush=True)
del a
torch.cuda.empty_cache()
cfg = P.SketchConfig(ell=110, q_power=2, seed=0)
for _ in range(3):
    t0 = time.perf_counter()
    P.corutv(host, cfg)
    torch.cuda.synchronize()
    print(f"corutv(numpy pageable): {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
