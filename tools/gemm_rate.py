"""Time corutv_gemm (KK: A X, MM: A' Y) at a C3 row-block shape and the
low-rank STORE kernel with CUDA events.  usage: gemm_rate.py [libpath]"""
import sys
sys.path.insert(0, '.')
import torch
from paper_1906_04572_b200 import _lib
import paper_1906_04572_b200 as P
if len(sys.argv) > 1:
    _lib._lib = _lib.load_library(sys.argv[1])
torch.cuda.set_device(0)
h = _lib.handle(0)
m, n, ell = 65536, 32768, 110
A = torch.randn(m, n, dtype=torch.float64, device='cuda')
X = torch.randn(n, ell, dtype=torch.float64, device='cuda')
Yp = torch.randn(m, 112, dtype=torch.float64, device='cuda')  # decompose layout, ld 112
Y = Yp[:, :ell]
C1 = torch.empty(m, ell, dtype=torch.float64, device='cuda')
C2 = torch.empty(n, ell, dtype=torch.float64, device='cuda')
def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
kk = timeit(lambda: h.call("corutv_gemm", 0, m, ell, n, A.data_ptr(), n, X.data_ptr(), ell, C1.data_ptr(), ell))
mm = timeit(lambda: h.call("corutv_gemm", 1, n, ell, m, A.data_ptr(), n, Y.data_ptr(), 112, C2.data_ptr(), ell))
mm2 = timeit(lambda: h.call("corutv_gemm", 1, n, ell, m, A.data_ptr(), n, Yp.contiguous()[:, :ell].contiguous().data_ptr(), ell, C2.data_ptr(), ell))
fl = 2.0 * m * n * ell
print(f"KK {kk:.3f} ms {fl / kk / 1e9:.2f} TF   MM(3-D boxes) {mm:.3f} ms {fl / mm / 1e9:.2f} TF   "
      f"MM(ld 110, 2-D boxes) {mm2:.3f} ms {fl / mm2 / 1e9:.2f} TF")
del A
u = torch.randn(10000, 100, dtype=torch.float64, device='cuda')
t = torch.triu(torch.randn(100, 100, dtype=torch.float64, device='cuda'))
v = torch.randn(10000, 100, dtype=torch.float64, device='cuda')
lr = timeit(lambda: P.rpca._lowrank_device(u, t, v, 60))
print(f"lowrank STORE 10000^2 r=60: {lr:.3f} ms  ({10000 * 10000 * 8 / lr / 1e6:.0f} GB/s write)")
