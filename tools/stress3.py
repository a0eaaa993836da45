"""Randomised stress of the InexactALM pieces: Jacobi SVD (one-CTA and grid
paths, cold and warm-started, zero columns, tall / wide), svt, small
inexact_alm solves -- against the oracle.  usage: stress3.py [seconds]"""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import oracle as O
import paper_1906_04572_b200 as P

torch.cuda.set_device(0)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.Generator(np.random.PCG64(303))
t_end = time.time() + budget
stats = {}


def note(kind, ok, msg=""):
    s = stats.setdefault(kind, [0, 0])
    s[0] += 1
    if not ok:
        s[1] += 1
        print("BAD", kind, msg, flush=True)


while time.time() < t_end:
    kind = rng.choice(["svd", "svd_warm", "svt", "ialm"], p=[0.35, 0.25, 0.25, 0.15])
    try:
        if kind in ("svd", "svd_warm"):
            m = int(rng.integers(1, 700))
            n = int(rng.integers(1, 700))
            a = rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-3, 3)
            if rng.random() < 0.2 and n > 3:
                a[:, rng.choice(n, size=min(n, int(rng.integers(1, 4))), replace=False)] = 0.0
            k = min(m, n)
            v0 = None
            if kind == "svd_warm":
                at = a if m >= n else a.T
                v0 = O.jacobi_svd(at + 1e-3 * np.abs(at).max() * rng.standard_normal(at.shape))[2]
            f = P.jacobi_svd(a, v_init=v0)
            s = O.jacobi_svd(a, v0)[1]
            s0 = max(s[0], 1e-300)
            ok = np.abs(f.sigma - s).max() <= 1e-11 * s0
            ok &= np.abs(f.u.T @ f.u - np.eye(k)).max() <= 1e-10
            ok &= np.abs((f.u * f.sigma) @ f.v.T - a).max() <= 1e-10 * s0
            note(kind, bool(ok), f"{m}x{n} warm={v0 is not None}")
        elif kind == "svt":
            m = int(rng.integers(1, 300))
            n = int(rng.integers(1, 300))
            b = rng.standard_normal((m, n))
            s = O.jacobi_svd(b)[1]
            delta = float(rng.uniform(0, s[0] * 1.1))
            mat, r = P.svt(b, delta)
            want, rw = O.svt(b, delta)
            # r is a count against delta: a gap of ~1e-12 s0 can flip it
            near = np.min(np.abs(s - delta)) <= 1e-10 * s[0]
            ok = (r == rw or near) and (r != rw or np.abs(mat - want).max() <= 1e-9 * max(s[0], 1.0))
            note(kind, bool(ok), f"{m}x{n} delta={delta} r={r}/{rw}")
        else:
            n = int(rng.integers(20, 160))
            k = max(1, round(0.05 * n))
            s_ = round(0.05 * n * n)
            mm, _, _ = O.gen_rpca_instance(n, k, s_, seed=int(rng.integers(0, 1000)))
            sol = P.inexact_alm(mm, P.AlmConfig(ell=2 * k))
            ref = O.inexact_alm(mm, ell=2 * k)
            ok = (sol.iterations == ref["iterations"] and sol.rank_history == ref["rank_history"]
                  and sol.nnz_history == ref["nnz_history"])
            note(kind, bool(ok), f"n={n} it={sol.iterations}/{ref['iterations']}")
    except Exception as e:  # noqa: BLE001
        note(kind, False, f"{type(e).__name__}: {e}")
print({k: f"{v[0]} cases, {v[1]} bad" for k, v in stats.items()}, flush=True)
