"""The reference package's OWN tests, run against the device through
``install()`` (SURVEY §8(c) last paragraph; VERDICT r01 "next" #8).

pkg/tests/test_sketch.py, test_rpca.py, test_dense.py and the fast
(``not slow``) tier of test_acceptance.py run unmodified from
``baseline/_ref/ref_tests`` (tools/stage_reference.sh) under
tests/ref_suite/corutv_ref_plugin.py, which rebinds the reference's ``corutv``,
``alm_corutv``, ``sor_svd``, ``tsr_svd``, ``inexact_alm`` and ``svt`` to this
package before the test modules import them.

The bar is the reference's own outcome, not "all green": the reference's
recorded run (pkg/test_output.txt:566-567) fails two statistical acceptance
checks on its own numpy path (test_c3_lowrank_error_optimality[3-400]:
mean e_k/optimal 1.0245 > 1.02; test_c6_desk_scale_inexact_alm: exact on
18/20 seeds -- a slow-tier test, not run here).  The fast tier of the pure
reference, run here on numpy, fails only the first.  The device computes the
same numbers, so it may fail only those and must pass everything else.
Exceptions: install() makes the device path's ConvergenceError a subclass of
the reference's, so test_rpca.py's ``pytest.raises(ConvergenceError)`` holds."""

from __future__ import annotations

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = ROOT / "baseline" / "_ref" / "ref_tests"

# the reference's own failures on its numpy path (pkg/test_output.txt:566-567)
REFERENCE_OWN_FAILURES = {
    "test_acceptance.py::test_c3_lowrank_error_optimality[3-400]",
    "test_acceptance.py::test_c6_desk_scale_inexact_alm",
}


def _outcomes(xml_path: Path) -> dict[str, str]:
    out = {}
    for case in ET.parse(xml_path).getroot().iter("testcase"):
        mod = case.get("classname", "").split(".")[-1] + ".py"
        name = f"{mod}::{case.get('name')}"
        state = "passed"
        for child in case:
            if child.tag in ("failure", "error"):
                state = "failed"
            elif child.tag == "skipped":
                state = "skipped"
        out[name] = state
    return out


def test_reference_suite_through_install(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not (REF_TESTS / "test_sketch.py").exists() or not (ROOT / "baseline" / "_ref" / "corutv").exists():
        pytest.skip("baseline/_ref not staged (tools/stage_reference.sh)")
    xml = tmp_path / "ref_suite.xml"
    calls = tmp_path / "calls.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT / "tests" / "ref_suite"), str(ROOT)]), CORUTV_REF_SUITE_CALLS=str(calls))
    files = ["test_sketch.py", "test_rpca.py", "test_dense.py", "test_acceptance.py"]
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "corutv_ref_plugin", "-m", "not slow",
         "-p", "no:cacheprovider", f"--junitxml={xml}", *files],
        cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1500)
    tail = (proc.stdout + proc.stderr)[-4000:]
    assert xml.exists(), tail
    res = _outcomes(xml)
    failed = {k for k, v in res.items() if v == "failed"}
    n_pass = sum(v == "passed" for v in res.values())
    counts = json.loads(calls.read_text()) if calls.exists() else {}
    print(f"reference suite on the device: {n_pass} passed, failed={sorted(failed)}, calls={counts}")
    assert counts.get("corutv.sketch.corutv", 0) > 0, (counts, tail)
    assert counts.get("corutv.rpca.alm_corutv", 0) > 0, (counts, tail)
    assert failed <= REFERENCE_OWN_FAILURES, tail
    assert n_pass >= 60, (n_pass, tail)
