"""C3 device-resident corutv: explicit vs seeded Omega, wall vs CUDA events,
and the per-class profile split."""
import ctypes
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import _lib, sketch
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
m, n, ell = 131072, 32768, 110
a = bench.gen_rows_device(torch, "c3", 0, m, dev)
cfg = P.SketchConfig(ell=ell, q_power=2, seed=0)
om = sketch.gaussian_matrix_device(n, ell, 0)
h = _lib.handle(0)
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, e0.elapsed_time(e1) / reps
for name, fn in (("explicit omega", lambda: P.corutv(a, cfg, omega=om)), ("seeded", lambda: P.corutv(a, cfg)),
                 ("explicit omega", lambda: P.corutv(a, cfg, omega=om))):
    w, e = timed(fn)
    print(f"{name}: wall {w:.1f} ms, events {e:.1f} ms", flush=True)
out = (ctypes.c_double * 12)()
launches = ctypes.c_int64(0)
for name, o in (("explicit", om), ("seeded", None)):
    h.bind_stream()
    h.lib.corutv_profile_begin(h.ptr)
    P.corutv(a, cfg, omega=o)
    torch.cuda.synchronize()
    h.lib.corutv_profile_end(h.ptr, out, ctypes.byref(launches))
    print(name, "profile classes (ms, flops...)", [round(x, 3) for x in out], launches.value, flush=True)
