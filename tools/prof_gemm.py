"""Run the sketch GEMMs (K1: A X, K2: A' C1) at a C3 row-block shape for ncu."""
import sys
sys.path.insert(0, '.')
import torch
from paper_1906_04572_b200 import _lib
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
n, ell = 32768, 110
torch.cuda.set_device(0)
h = _lib.handle(0)
A = torch.randn(m, n, dtype=torch.float64, device='cuda')
X = torch.randn(n, ell, dtype=torch.float64, device='cuda')
Y = torch.randn(m, ell, dtype=torch.float64, device='cuda')
C1 = torch.empty(m, ell, dtype=torch.float64, device='cuda')
C2 = torch.empty(n, ell, dtype=torch.float64, device='cuda')
for _ in range(2):
    h.call("corutv_gemm", 0, m, ell, n, A.data_ptr(), n, X.data_ptr(), ell, C1.data_ptr(), ell)
    h.call("corutv_gemm", 1, n, ell, m, A.data_ptr(), n, Y.data_ptr(), ell, C2.data_ptr(), ell)
torch.cuda.synchronize()
print("ok")
