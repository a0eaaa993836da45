"""ncu target: tsr_svd (one-pass dual sketch) on a device-resident
65536 x 16384 matrix, ell = 8 then 16, two calls each."""
import sys
sys.path.insert(0, '.')
import torch
import bench
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
m, n = 65536, 16384
a = bench.gen_rows_device(torch, "c3", 0, m, torch.device("cuda", 0))[:, :n].contiguous()
for ell in (8, 16):
    for _ in range(2):
        f = P.tsr_svd(a, P.SketchConfig(ell=ell, seed=3))
torch.cuda.synchronize()
print("ok", float(f.sigma[0]))
