"""Debug: the 'repeated' spectrum case of test_spectral_norm_block_power_spectra."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import oracle as O
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
kind = sys.argv[1] if len(sys.argv) > 1 else "repeated"
rng = np.random.Generator(np.random.PCG64(len(kind)))
m, n = 300, 200
qu, _ = np.linalg.qr(rng.standard_normal((m, n)))
qv, _ = np.linalg.qr(rng.standard_normal((n, n)))
sig = {"repeated": np.r_[np.full(5, 3.0), np.linspace(1.0, 0.1, n - 5)],
       "graded": 10.0 ** -np.linspace(0, 12, n)}[kind]
a = (qu * sig) @ qv.T
val, it = P.dense.spectral_norm_iters(a)
oval, oit = O.spectral_norm(a)
print("device", val, it, "oracle", oval, oit, flush=True)
