"""C4-size fused ALM update alone (ncu target): 10000^2, ell = 51, r = 50."""
import ctypes
import sys
sys.path.insert(0, '.')
import os
from pathlib import Path
import torch
from paper_1906_04572_b200 import _lib
if os.environ.get("CORUTV_LIB"):  # A/B a variant build of the library
    _lib.LIB_PATH = Path(os.environ["CORUTV_LIB"]).resolve()
torch.cuda.set_device(0)
n, ell = 10000, 51
r = int(os.environ.get("ALM_R", "50"))
M = torch.randn(n, n, dtype=torch.float64, device='cuda')
S = torch.zeros_like(M)
Y = torch.zeros_like(M)
G = torch.empty_like(M)
u = torch.randn(n, ell, dtype=torch.float64, device='cuda')
t = torch.triu(torch.randn(ell, ell, dtype=torch.float64, device='cuda'))
v = torch.randn(n, ell, dtype=torch.float64, device='cuda')
h = _lib.handle(0)
z, c = ctypes.c_double(), ctypes.c_int64()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    h.call("corutv_alm_update", M.data_ptr(), S.data_ptr(), Y.data_ptr(), G.data_ptr(), n, n, u.data_ptr(),
           t.data_ptr(), v.data_ptr(), ell, r, 1e-3, 0.5, 1.5e-3, ctypes.byref(z), ctypes.byref(c))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    h.call("corutv_alm_update", M.data_ptr(), S.data_ptr(), Y.data_ptr(), G.data_ptr(), n, n, u.data_ptr(),
           t.data_ptr(), v.data_ptr(), ell, r, 1e-3, 0.5, 1.5e-3, ctypes.byref(z), ctypes.byref(c))
e1.record()
torch.cuda.synchronize()
print(f"alm_update {e0.elapsed_time(e1) / 10:.3f} ms")
