"""Full-size C3 / C5 parity (BASELINE configs[2]: 131072 x 32768, ell 110,
q 2; configs[4]: 262144 x 32768, ell 272, q 2) against the CPU oracle, on the
GPU box (oracle: numpy restatement of sketch.py:166-208 on 16 cores; ~36 /
~72 GB of host memory).  usage: full_parity.py [c3|c5] [exact-d|approx-d]

Same A for both (bench.gen_rows_device, copied to the host) and the same
seeded Omega (the device draws numpy's PCG64 stream bit-identically).
Compares |diag T|, the QRCP permutation, U / V (leading columns, up to
sign) and the reconstruction error |A - U T V'|_F (both evaluated on the
device by the fused residual kernel).  Writes gpurun_out/c3_parity.json.
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
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import _device as D
from paper_1906_04572_b200 import _lib

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
variant = sys.argv[2] if len(sys.argv) > 2 else "exact-d"
m, n, ell, q, k, noise, _ = bench.WORKLOADS[wl]
a = bench.gen_rows_device(torch, wl, 0, m, dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
f = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, seed=0, variant=variant))
torch.cuda.synchronize()
out = {"workload": wl, "variant": variant, "device_s": time.perf_counter() - t0}
a_host = a.cpu().numpy()
t0 = time.perf_counter()
ref = O.corutv(a_host, ell, q, seed=0, variant=variant)
out["oracle_s"] = time.perf_counter() - t0
del a_host


def err_of(u, t, v):
    e = ctypes.c_double(0.0)
    _lib.handle(0).call("corutv_lowrank_error", D.ptr(a), m, n, a.stride(0), D.ptr(u), D.ptr(t), D.ptr(v), ell,
                        ctypes.byref(e))
    return e.value


ut = torch.from_numpy(np.ascontiguousarray(ref["u"])).to(dev)
tt = torch.from_numpy(np.ascontiguousarray(ref["t"])).to(dev)
vt = torch.from_numpy(np.ascontiguousarray(ref["v"])).to(dev)
e_dev, e_ref = err_of(f.u, f.t, f.v), err_of(ut, tt, vt)
d_dev = f.t.diagonal().abs().cpu().numpy()
d_ref = np.abs(np.diag(ref["t"]))
perm_dev = np.asarray(f.perm.cpu())
u_dev, v_dev = f.u[:, :k].cpu().numpy(), f.v[:, :k].cpu().numpy()
s_u = np.sign(np.sum(u_dev * ref["u"][:, :k], axis=0))
s_v = np.sign(np.sum(v_dev * ref["v"][:, :k], axis=0))
out.update({
    "shape": [m, n], "ell": ell, "q": q,
    "err_device": e_dev, "err_oracle": e_ref, "err_rel_diff": abs(e_dev - e_ref) / e_ref,
    "diagT_lead_max_rel_diff": float(np.max(np.abs(d_dev[:k] - d_ref[:k])) / d_ref[0]),
    "diagT_all_max_rel_diff": float(np.max(np.abs(d_dev - d_ref)) / d_ref[0]),
    "perm_lead_equal": bool(np.array_equal(perm_dev[:k], ref["perm"][:k])),
    "perm_all_equal": bool(np.array_equal(perm_dev, ref["perm"])),
    "u_lead_max_abs_diff": float(np.max(np.abs(u_dev * s_u - ref["u"][:, :k]))),
    "v_lead_max_abs_diff": float(np.max(np.abs(v_dev * s_v - ref["v"][:, :k]))),
    "passes_oracle": ref["passes"],
})
print(json.dumps(out, indent=1))
tag = "" if variant == "exact-d" else "_approx"
json.dump(out, open(f"gpurun_out/{wl}{tag}_parity.json", "w"), indent=1)
