"""pytest plugin: run the reference package's OWN test files with its hot
path rebound to the device by ``paper_1906_04572_b200.install()`` (SURVEY
§8(c), last paragraph: the reference's tests are the acceptance suite of the
drop-in).

    python -m pytest -p corutv_ref_plugin baseline/_ref/ref_tests/test_sketch.py ...

``baseline/_ref`` holds the unmodified reference (pip install --target, see
tools/stage_reference.sh) and ``baseline/_ref/ref_tests`` an unmodified copy
of its ``pkg/tests``; both are git-ignored and travel to the GPU box with the
snapshot.  install() runs in ``pytest_configure``, i.e. before the test
modules are imported, so their ``from corutv.sketch import corutv`` binds the
device function -- exactly what a maintainer's one-line ``install()`` in the
reference's ``__init__`` would do.  Every rebound name is wrapped in a call
counter; the session FAILS if the device path was never called (a suite that
silently ran on numpy proves nothing).
"""

from __future__ import annotations

import functools
import importlib
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF = ROOT / "baseline" / "_ref"

CALLS: dict[str, int] = {}


def _counted(name, fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*args, **kwargs)

    return wrapper


def pytest_configure(config):
    for p in (str(ROOT), str(REF)):
        if p not in sys.path:
            sys.path.insert(0, p)
    ref = importlib.import_module("corutv")
    if not str(getattr(ref, "__file__", "")).startswith(str(REF)):
        raise RuntimeError(f"corutv resolved to {ref.__file__}, not the baseline/_ref install")
    import paper_1906_04572_b200 as P

    done = P.install(ref)
    for full in done:
        if not full.replace(".", "").replace("_", "").isalnum():
            continue  # e.g. the exception base-class adoption note
        modname, name = full.rsplit(".", 1)
        mod = sys.modules[modname]
        setattr(mod, name, _counted(full, getattr(mod, name)))
    config._corutv_rebound = done


def pytest_report_header(config):
    return "corutv install(): rebound " + ", ".join(getattr(config, "_corutv_rebound", []))


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("CORUTV_REF_SUITE_CALLS")
    if out:
        Path(out).write_text(json.dumps(CALLS, sort_keys=True))
    if exitstatus == 0 and session.testscollected and not CALLS:
        session.exitstatus = 1


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line("device calls through install(): " + json.dumps(CALLS, sort_keys=True))
