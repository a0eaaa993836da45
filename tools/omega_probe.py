"""Time the device Gaussian test matrix and a C3 decompose with explicit vs
seeded Omega."""
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import sketch
torch.cuda.set_device(0)
def wall(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
for rows, cols in ((1000, 15), (10000, 1), (10000, 100), (32768, 110), (32768, 272), (1 << 20, 64)):
    ms = wall(lambda: sketch.gaussian_matrix_device(rows, cols, 7))
    print(f"gaussian {rows}x{cols}: {ms:.3f} ms ({rows * cols / ms / 1e6:.1f} M samples/ms)", flush=True)
