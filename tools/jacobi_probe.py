"""Device one-sided Jacobi SVD timing (cold and warm-started), n x n."""
import sys
import time
sys.path.insert(0, '.')
import os
from pathlib import Path
import torch
import paper_1906_04572_b200 as P
if os.environ.get("CORUTV_LIB"):  # A/B a variant build of the library
    P._lib.LIB_PATH = Path(os.environ["CORUTV_LIB"]).resolve()

torch.cuda.set_device(0)
for n in [int(x) for x in sys.argv[1:]] or [400, 1000]:
    g = torch.Generator(device='cuda').manual_seed(n)
    a = torch.randn(n, n, dtype=torch.float64, device='cuda', generator=g)
    P.jacobi_svd(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = P.jacobi_svd(a)
    torch.cuda.synchronize()
    cold = time.perf_counter() - t0
    b = a + 1e-4 * torch.randn(n, n, dtype=torch.float64, device='cuda', generator=g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.jacobi_svd(b, v_init=f.v)
    torch.cuda.synchronize()
    warm = time.perf_counter() - t0
    t0 = time.perf_counter()
    P.singular_values(a)
    torch.cuda.synchronize()
    sv = time.perf_counter() - t0
    print(f"n {n}: svd cold {cold*1e3:.1f} ms, warm {warm*1e3:.1f} ms, singular_values {sv*1e3:.1f} ms", flush=True)
