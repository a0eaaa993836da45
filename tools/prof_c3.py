"""One C3-size A sweep of each GEMM orientation (131072 x 32768, ell = 110) for
ncu --set full: launch 1 = K1 (A X, KK), launch 3 = K2 (A' C1, MM)."""
import sys
sys.path.insert(0, '.')
import torch
import bench
from paper_1906_04572_b200 import _lib
torch.cuda.set_device(0)
m, n, ell = 131072, 32768, 110
A = bench.gen_rows_device(torch, "c3", 0, m, torch.device("cuda", 0))
X = torch.randn(n, ell, dtype=torch.float64, device='cuda')
# C1 as the decompose lays it out: ld = round_up(ell, 16) (3-D TMA boxes)
Yp = torch.randn(m, 112, dtype=torch.float64, device='cuda')
Y = Yp[:, :ell]
C1 = torch.empty(m, ell, dtype=torch.float64, device='cuda')
C2 = torch.empty(n, ell, dtype=torch.float64, device='cuda')
torch.cuda.synchronize()
h = _lib.handle(0)
h.call("corutv_gemm", 0, m, ell, n, A.data_ptr(), n, X.data_ptr(), ell, C1.data_ptr(), ell)
h.call("corutv_gemm", 1, n, ell, m, A.data_ptr(), n, Y.data_ptr(), 112, C2.data_ptr(), ell)
torch.cuda.synchronize()
print("ok")
