"""InexactALM baseline (rpca.py:258-273) on the device vs the oracle.

    python tools/ialm_probe.py [n ...]      (default 400 1000)

Instance: gen_rpca_instance(n, k = n/20, s = n^2/20, seed 0), AlmConfig(ell=2k)
(test_rpca.py:160-180, test_acceptance.py:209-218).  The oracle leg runs for
n <= 400 only (the reference's own desk-scale cap is 60 s per solve).
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1906_04572_b200 as P  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [400, 1000]:
    k, s = max(1, round(0.05 * n)), round(0.05 * n * n)
    m, l_true, s_true = O.gen_rpca_instance(n, k, s, seed=0)
    md = torch.from_numpy(m).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = P.inexact_alm(md, P.AlmConfig(ell=2 * k))
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    sol = P.inexact_alm(md, P.AlmConfig(ell=2 * k))
    torch.cuda.synchronize()
    dev_s2 = time.perf_counter() - t0
    out = dict(n=n, k=k, s=s, iterations=sol.iterations, rank_of_l=sol.rank_of_l, nnz_of_s=sol.nnz_of_s,
               device_s_first=round(dev_s, 4), device_s=round(dev_s2, 4),
               l_err=float(torch.linalg.norm(sol.l.cpu() - torch.from_numpy(l_true)) / np.linalg.norm(l_true)))
    if n <= 400:
        t0 = time.perf_counter()
        ref = O.inexact_alm(m, ell=2 * k)
        out["oracle_s"] = round(time.perf_counter() - t0, 3)
        out["histories_equal"] = (ref["rank_history"] == sol.rank_history and ref["nnz_history"] == sol.nnz_history
                                  and ref["iterations"] == sol.iterations)
    print(json.dumps(out), flush=True)
