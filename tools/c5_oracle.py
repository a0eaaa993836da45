"""Record the CPU oracle's CoR-UTV of BASELINE configs[4] (C5: 262144 x
32768, U512 diag(0.99^i) V512' + 1e-6 G with orthonormal U512 / V512, ell =
272, q = 2, seeded Omega) as tests/golden/c5_oracle.json, the way
tools/c4_parity.py records C4.  Runs on the GPU box (the device generates A,
bench.gen_rows_device; the oracle -- numpy restatement of sketch.py:166-208
-- runs on a host copy, ~72 GB of host memory, ~150 s on 16 cores).

    python tools/c5_oracle.py   ->  gpurun_out/c5_oracle.json
"""
import ctypes
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import oracle as O
from paper_1906_04572_b200 import _device as D
from paper_1906_04572_b200 import _lib

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
m, n, ell, q, k, noise, desc = bench.WORKLOADS["c5"]
a = bench.gen_rows_device(torch, "c5", 0, m, dev)
torch.cuda.synchronize()
a_host = a.cpu().numpy()
t0 = time.perf_counter()
with bench.all_blas_threads():
    ref = O.corutv(a_host, ell, q, seed=0)
t_oracle = time.perf_counter() - t0
del a_host


def err_of(u, t, v):
    e = ctypes.c_double(0.0)
    _lib.handle(0).call("corutv_lowrank_error", D.ptr(a), m, n, a.stride(0), D.ptr(u), D.ptr(t), D.ptr(v), ell,
                        ctypes.byref(e))
    return e.value


ut = torch.from_numpy(np.ascontiguousarray(ref["u"])).to(dev)
tt = torch.from_numpy(np.ascontiguousarray(ref["t"])).to(dev)
vt = torch.from_numpy(np.ascontiguousarray(ref["v"])).to(dev)
a2 = float((a * a).sum())
out = {
    "made_by": "tools/c5_oracle.py on a B200 box: the CPU oracle (oracle.corutv, numpy restatement of "
               "sketch.py:166-208) on the device-generated C5 matrix (bench.gen_rows_device 'c5', seed 1234): "
               + desc + "; Omega = gaussian_matrix(32768, 272, seed 0)",
    "shape": [m, n], "ell": ell, "q": q,
    "diag_t_abs": np.abs(np.diag(ref["t"])).tolist(),
    "perm": [int(x) for x in ref["perm"]],
    "err": err_of(ut, tt, vt),
    "a_fro2": a2,
    "passes": ref["passes"],
    "u_col0_sample": ref["u"][::4096, 0].tolist(),
    "v_col0_sample": ref["v"][::512, 0].tolist(),
    "oracle_s": t_oracle,
    "cores": bench.host_cores(),
}
json.dump(out, open("gpurun_out/c5_oracle.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if not isinstance(v, list)}, indent=1))
