"""Time the REFERENCE harness (bench.run_sv_compare / run_lowrank_error /
run_rpca_recovery at their default configs) on this container's CPU.
Build-container only (imports /root/reference); output -> profiles/."""
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
from corutv import bench  # noqa: E402

out = {"cpu_threads_env": os.environ.get("CORUTV_THREADS", "1"), "cores": os.cpu_count()}
for exp, fn in (("sv-compare", bench.run_sv_compare), ("lowrank-error", bench.run_lowrank_error),
                ("rpca-recovery", bench.run_rpca_recovery)):
    t0 = time.perf_counter()
    rows = fn(bench.ExperimentConfig(experiment=exp))
    out[exp] = {"seconds": round(time.perf_counter() - t0, 2), "rows": len(rows)}
    print(json.dumps(out), flush=True)
