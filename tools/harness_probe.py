"""Device harness wall time at the reference's default experiment configs
(bench.ExperimentConfig defaults: n = 400, k = 20, 20 trials).

    python tools/harness_probe.py            -> one JSON line per experiment
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1906_04572_b200 import harness as H  # noqa: E402

torch.cuda.set_device(0)
H.run_sv_compare(H.ExperimentConfig("sv-compare", n=64, k=4, trials=8))  # warm handles / pool
for threads in ("1", "8"):
    os.environ["CORUTV_THREADS"] = threads
    for exp, fn in (("sv-compare", H.run_sv_compare), ("lowrank-error", H.run_lowrank_error),
                    ("rpca-recovery", H.run_rpca_recovery)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rows = fn(H.ExperimentConfig(exp))
        torch.cuda.synchronize()
        print(json.dumps({"experiment": exp, "threads": int(threads), "seconds": round(time.perf_counter() - t0, 3),
                          "rows": len(rows)}), flush=True)
