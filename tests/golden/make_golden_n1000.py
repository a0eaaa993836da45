"""Golden rows of the reference harness at n = 1000 (the cores past the old
640 limit: the "qrcp" method factors the whole 1000 x 1000 matrix and
"utv-approx" runs corutv with ell = n = 1000; bench.py:150-153).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_n1000.py

Writes tests/golden/golden_n1000.npz from the REFERENCE package itself
(read-only import of /root/reference/pkg/src).  The GPU box only reads the
committed .npz.
"""

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from corutv import bench as rbench  # noqa: E402

t0 = time.time()
cfg = rbench.ExperimentConfig(experiment="sv-compare", n=1000, k=20, trials=2, q_power=1,
                              methods=("qrcp", "utv-approx"))
rows = rbench.run_sv_compare(cfg)
cols = list(zip(*rows))
out = {
    "what": np.array("bench.run_sv_compare(ExperimentConfig('sv-compare', n=1000, k=20, trials=2, q_power=1, "
                     "methods=('qrcp', 'utv-approx')))"),
    "c0": np.array(cols[0]), "method": np.array(cols[1]), "c2": np.array(cols[2]),
    "c3": np.array(cols[3]), "c4": np.array(cols[4]),
}
here = Path(__file__).resolve().parent
np.savez_compressed(here / "golden_n1000.npz", **out)
print("wrote", len(rows), "rows in", round(time.time() - t0, 1), "s")
