"""Randomised stress of the device path against the CPU oracle: random
shapes, ranks, ell, q, variants, input residency; prints any disagreement.
usage: python tools/stress.py [seconds]"""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import oracle as O
import paper_1906_04572_b200 as P

torch.cuda.set_device(0)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.Generator(np.random.PCG64(2026))
t_end = time.time() + budget
n_cases = n_bad = 0
while time.time() < t_end:
    m = int(rng.integers(1, 2500))
    n = int(rng.integers(1, m + 1))
    k = int(rng.integers(1, min(m, n) + 1))
    ell = int(rng.integers(1, min(m, n, 200) + 1))
    q = int(rng.integers(0, 3))
    variant = P.VARIANT_EXACT if rng.random() < 0.7 else P.VARIANT_APPROX
    noise = float(10.0 ** rng.uniform(-12, -1))
    seed = int(rng.integers(0, 2 ** 32))
    a = rng.standard_normal((m, k)) @ rng.standard_normal((k, n)) + noise * rng.standard_normal((m, n))
    where = rng.integers(0, 3)  # numpy (streamed host path), device tensor, pinned host tensor
    x = a if where == 0 else (torch.from_numpy(a).cuda() if where == 1 else torch.from_numpy(a).pin_memory())
    cfg = P.SketchConfig(ell=ell, q_power=q, seed=seed, variant=variant)
    n_cases += 1
    try:
        f = P.corutv(x, cfg)
        u, t, v = (np.asarray(z.cpu()) if hasattr(z, "cpu") else z for z in (f.u, f.t, f.v))
        ref = O.corutv(a, ell, q, seed=seed, variant=variant)
        na = np.linalg.norm(a)
        err = np.linalg.norm(a - u @ (t @ v.T))
        eref = O.corutv_lowrank_error(a, ref)
        ok = abs(err - eref) <= 1e-8 * na + 1e-6 * eref
        ok &= bool(np.all(np.isfinite(u)) and np.all(np.isfinite(t)) and np.all(np.isfinite(v)))
        ok &= np.abs(u.T @ u - np.eye(ell)).max() < 1e-8 or k < ell  # rank-deficient cores may lose columns
        if not ok:
            n_bad += 1
            print(f"MISMATCH m={m} n={n} k={k} ell={ell} q={q} {variant} noise={noise:.1e} where={where} "
                  f"err={err:.6e} ref={eref:.6e} |A|={na:.3e}", flush=True)
    except Exception as exc:  # noqa: BLE001
        n_bad += 1
        print(f"ERROR m={m} n={n} k={k} ell={ell} q={q} {variant} where={where}: {exc!r}"[:300], flush=True)
print(f"stress: {n_cases} cases, {n_bad} bad")
