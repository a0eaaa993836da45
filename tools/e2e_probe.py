"""Where does the end-to-end (host input) C3 step spend its time?"""
import os
import sys
import time
sys.path.insert(0, '.')
import torch
import bench
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
m, n, ell = 131072, 32768, 110
a = bench.gen_rows_device(torch, "c3", 0, m, dev)
ah = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
ah.copy_(a)
cfg = P.SketchConfig(ell=ell, q_power=2, seed=0)
def wall(fn, reps=2):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
print(f"H2D one copy 34.4 GB: {wall(lambda: a.copy_(ah, non_blocking=True)):.1f} ms", flush=True)
print(f"device corutv: {wall(lambda: P.corutv(a, cfg)):.1f} ms", flush=True)
del a
torch.cuda.empty_cache()
for cb in (None, str(4 << 30), str(256 << 20)):
    if cb is None:
        os.environ.pop("CORUTV_HOST_CHUNK_BYTES", None)
    else:
        os.environ["CORUTV_HOST_CHUNK_BYTES"] = cb
    print(f"host corutv chunk={cb}: {wall(lambda: P.corutv(ah, cfg)):.1f} ms", flush=True)
os.environ.pop("CORUTV_HOST_CHUNK_BYTES", None)
# split: time to the end of the decompose vs output copies
import ctypes
from paper_1906_04572_b200 import _lib, sketch
ad = torch.empty((m, n), dtype=torch.float64, device=dev)
u = torch.empty((m, ell), dtype=torch.float64, device=dev)
t = torch.empty((ell, ell), dtype=torch.float64, device=dev)
v = torch.empty((n, ell), dtype=torch.float64, device=dev)
perm = torch.empty((ell,), dtype=torch.int64, device=dev)
h = _lib.handle(0)
passes = ctypes.c_int64(0)
def raw():
    h.call("corutv_decompose_host", ah.data_ptr(), m, n, n, ad.data_ptr(), n, ell, 2, 0, None,
           sketch.pcg_state(0), u.data_ptr(), t.data_ptr(), v.data_ptr(), perm.data_ptr(), ctypes.byref(passes))
print(f"raw corutv_decompose_host (no output D2H): {wall(raw):.1f} ms", flush=True)
print(f"outputs D2H (pageable .cpu()): {wall(lambda: (u.cpu(), t.cpu(), v.cpu(), perm.cpu())):.1f} ms", flush=True)
