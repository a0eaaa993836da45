"""Randomised stress of the secondary paths: sor_svd / tsr_svd (device and
host inputs), corutv_truncated + the fused ALM update, CRUTVMAT streaming,
small ALM solves -- against the oracle / torch.  usage: stress2.py [seconds]"""
import os
import sys
import tempfile
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import oracle as O
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import matio

torch.cuda.set_device(0)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.Generator(np.random.PCG64(77))
t_end = time.time() + budget
stats = {}
tmpdir = tempfile.mkdtemp()


def bad(kind, msg):
    stats[kind + "_bad"] = stats.get(kind + "_bad", 0) + 1
    print(f"BAD {kind}: {msg}"[:400], flush=True)


while time.time() < t_end:
    kind = ["svd", "alm_update", "file", "alm"][int(rng.integers(0, 4))]
    stats[kind] = stats.get(kind, 0) + 1
    try:
        if kind == "svd":
            m = int(rng.integers(2, 1500)); n = int(rng.integers(2, m + 1)); k = int(rng.integers(1, min(m, n) + 1))
            ell = int(rng.integers(1, min(k, 120) + 1))  # ell <= rank: determined factors
            a = rng.standard_normal((m, k)) @ rng.standard_normal((k, n))
            seed = int(rng.integers(0, 1 << 30))
            if rng.random() < 0.5:
                cfg = P.SketchConfig(ell=ell, q_power=int(rng.integers(0, 3)), seed=seed)
                f = P.sor_svd(a if rng.random() < 0.5 else torch.from_numpy(a).cuda(), cfg)
                o = O.sor_svd(a, ell, cfg.q_power, seed)
            else:
                cfg = P.SketchConfig(ell=ell, seed=seed)
                f = P.tsr_svd(a if rng.random() < 0.5 else torch.from_numpy(a).cuda(), cfg)
                o = O.tsr_svd(a, ell, seed)
            s = f.sigma.cpu().numpy() if hasattr(f.sigma, "cpu") else f.sigma
            if not np.all(np.isfinite(s)) or np.abs(s - o["sigma"]).max() > 1e-8 * o["sigma"][0]:
                bad(kind, f"m={m} n={n} k={k} ell={ell} sigma diff {np.abs(s - o['sigma']).max():.3e} / {o['sigma'][0]:.3e}")
        elif kind == "alm_update":
            rows = int(rng.integers(1, 3000)); cols = int(rng.integers(1, 3000))
            ell = int(rng.integers(1, min(rows, cols, 80) + 1)); r = int(rng.integers(0, ell + 1))
            dev = torch.device("cuda", 0)
            g = torch.Generator(device=dev); g.manual_seed(int(rng.integers(0, 1 << 30)))
            u = torch.randn((rows, ell), generator=g, dtype=torch.float64, device=dev)
            t = torch.triu(torch.randn((ell, ell), generator=g, dtype=torch.float64, device=dev))
            v = torch.randn((cols, ell), generator=g, dtype=torch.float64, device=dev)
            out = P.rpca._lowrank_device(u, t, v, r)
            ref = u[:, :r] @ (t[:r, :] @ v.T) if r > 0 else torch.zeros((rows, cols), dtype=torch.float64, device=dev)
            err = float((out - ref).abs().max())
            if not err <= 1e-12 * max(1.0, float(ref.abs().max())):
                bad(kind, f"rows={rows} cols={cols} ell={ell} r={r} max err {err:.3e}")
        elif kind == "file":
            m = int(rng.integers(2, 2000)); n = int(rng.integers(1, min(m, 400) + 1))
            a = rng.standard_normal((m, n))
            ell = int(rng.integers(1, min(m, n) + 1))
            p = os.path.join(tmpdir, "a.bin")
            matio.write_matrix_bin(p, a)
            os.environ["CORUTV_HOST_CHUNK_BYTES"] = str(int(rng.integers(1 << 12, 1 << 22)))
            cfg = P.SketchConfig(ell=ell, q_power=int(rng.integers(0, 3)), seed=int(rng.integers(0, 1 << 30)))
            f = matio.corutv_file(p, cfg)
            gdev = P.corutv(torch.from_numpy(a).cuda(), cfg)
            os.environ.pop("CORUTV_HOST_CHUNK_BYTES", None)
            if not (np.array_equal(f.t, gdev.t.cpu().numpy()) and np.array_equal(f.u, gdev.u.cpu().numpy())):
                bad(kind, f"m={m} n={n} ell={ell}: streamed != device")
        else:
            n = int(rng.integers(40, 160)); k = max(1, round(0.05 * n)); s = round(0.05 * n * n)
            m_, _, _ = O.gen_rpca_instance(n, k, s, seed=int(rng.integers(0, 1 << 20)))
            sol = P.alm_corutv(m_, P.AlmConfig(ell=2 * k, q_power=1, seed=3))
            if not (np.all(np.isfinite(sol.l)) and sol.residuals[-1] < 1e-5):
                bad(kind, f"n={n}: residual {sol.residuals[-1]:.3e}")
            iden = np.linalg.norm(m_ - sol.l - sol.s) / np.linalg.norm(m_)
            if abs(iden - sol.residuals[-1]) > 1e-9:
                bad(kind, f"n={n}: |M-L-S|/|M| {iden:.3e} vs zeta {sol.residuals[-1]:.3e}")
    except Exception as exc:  # noqa: BLE001
        bad(kind, f"exception {exc!r}")
print("stress2:", stats)
