"""Host-side API logic (no GPU): configs, validation messages, flop model,
ALM schedule helpers, telemetry, and the rebinding into the reference
package namespace."""

import types

import numpy as np
import pytest

import oracle as O
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import rpca as R
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_sketch_config_validation():
    # pkg/tests/test_sketch.py:90-101
    with pytest.raises(ValueError):
        P.SketchConfig(ell=0, seed=1)
    with pytest.raises(ValueError):
        P.SketchConfig(ell=5, q_power=-1)
    with pytest.raises(ValueError):
        P.SketchConfig(ell=5, variant="other")
    with pytest.raises(ValueError, match="exceeds"):
        P.SketchConfig(ell=35).validated_for(40, 30)
    assert P.SketchConfig(ell=30).validated_for(40, 30).ell == 30


def test_alm_config_validation():
    # pkg/tests/test_rpca.py:125-136
    with pytest.raises(ValueError):
        P.AlmConfig(tol=0.0)
    with pytest.raises(ValueError):
        P.AlmConfig(rho=1.0)
    with pytest.raises(ValueError):
        P.AlmConfig(mu0=2.0, mu_bar=1.0)
    with pytest.raises(ValueError):
        P.AlmConfig(max_iter=0)


def test_alm_requires_ell():
    with pytest.raises(ValueError, match="ell"):
        P.alm_corutv(np.ones((10, 10)), P.AlmConfig())


@pytest.mark.parametrize("m,n,ell,q,variant", [
    (1000, 1000, 15, 0, "exact-d"), (4000, 3000, 50, 1, "exact-d"), (4000, 3000, 50, 2, "exact-d"),
    (131072, 32768, 110, 2, "exact-d"), (262144, 32768, 272, 2, "exact-d"), (3000, 2500, 25, 3, "approx-d"),
])
def test_flop_estimate_matches_oracle(m, n, ell, q, variant):
    assert P.flop_estimate(m, n, ell, q, variant) == O.flop_estimate(m, n, ell, q, variant)


def test_flop_estimate_known_values():
    # C1 9.1629e7, C2 6.0658e9 / 8.4658e9, C3 6.6230e12, C5 3.2812e13
    assert abs(P.flop_estimate(1000, 1000, 15, 0) - 9.1629e7) < 1e4
    assert abs(P.flop_estimate(4000, 3000, 50, 1) - 6.0658e9) < 1e6
    assert abs(P.flop_estimate(131072, 32768, 110, 2) - 6.6230e12) < 1e9


@pytest.mark.parametrize("cap,rank,limit,grow,want", [
    (100, 0, 10000, 500, 1), (100, 100, 10000, 500, 600), (600, 1, 10000, 500, 2),
    (5, 5, 6, 1, 6), (1, 0, 10, 1, 1),
])
def test_next_cap(cap, rank, limit, grow, want):
    assert R._next_cap(cap, rank, limit, grow) == want == O.next_cap(cap, rank, limit, grow)


def test_numerical_rank():
    sig = np.array([1.0, 1e-3, 1e-13, 0.0])
    assert R._numerical_rank(sig, (10, 10)) == O.numerical_rank(sig, (10, 10)) == 2
    assert R._numerical_rank(np.zeros(0), (3, 3)) == 0


def test_telemetry_csv(tmp_path):
    sol = P.RpcaSolution(l=None, s=None, iterations=2, residuals=[0.5, 1e-9], rank_of_l=1,
                         nnz_of_s=3, rank_history=[1, 1], nnz_history=[3, 3],
                         mu_history=[0.1, 0.15], ell_history=[2, 2])
    p = tmp_path / "t.csv"
    P.write_telemetry_csv(sol, p)
    lines = p.read_text().strip().split("\n")
    assert lines[0] == "iter,zeta,rank_l,nnz_s,mu"
    assert lines[2] == "2,1e-09,1,3,0.15"


def test_install_rebinds_reference_names():
    pkg = types.ModuleType("fakecorutv")
    pkg.__path__ = []
    import sys

    mods = {}
    for sub in ("sketch", "rpca", "bench"):
        m = types.ModuleType(f"fakecorutv.{sub}")
        m.corutv = object()
        if sub != "sketch":
            m.alm_corutv = object()
        mods[sub] = m
        sys.modules[f"fakecorutv.{sub}"] = m
    sys.modules["fakecorutv"] = pkg
    try:
        done = P.install(pkg)
        assert mods["sketch"].corutv is P.corutv
        assert mods["rpca"].corutv is P.corutv and mods["rpca"].alm_corutv is P.alm_corutv
        assert mods["bench"].corutv is P.corutv
        assert pkg.corutv is P.corutv and pkg.alm_corutv is P.alm_corutv
        assert "fakecorutv.rpca.alm_corutv" in done
    finally:
        for k in list(sys.modules):
            if k.startswith("fakecorutv"):
                del sys.modules[k]


def test_install_rebinds_the_real_reference_package():
    """install() against the unmodified reference in baseline/_ref (pip
    --target, tools/stage_reference.sh): every hot-path name the reference's
    own modules and tests import resolves to the device implementation."""
    import subprocess
    import sys

    ref = ROOT / "baseline" / "_ref"
    if not (ref / "corutv" / "__init__.py").exists():
        pytest.skip("baseline/_ref not staged (tools/stage_reference.sh)")
    code = (
        "import sys; sys.path[:0] = [%r, %r]\n"
        "import corutv, corutv.sketch, corutv.rpca, corutv.bench\n"
        "assert corutv.__file__.startswith(%r), corutv.__file__\n"
        "import paper_1906_04572_b200 as P\n"
        "done = P.install(corutv)\n"
        "assert corutv.sketch.corutv is P.corutv and corutv.rpca.corutv is P.corutv\n"
        "assert corutv.bench.corutv is P.corutv and corutv.bench.alm_corutv is P.alm_corutv\n"
        "assert corutv.rpca.alm_corutv is P.alm_corutv and corutv.rpca.inexact_alm is P.inexact_alm\n"
        "assert corutv.sketch.sor_svd is P.sor_svd and corutv.sketch.tsr_svd is P.tsr_svd\n"
        "from corutv.sketch import corutv as c; assert c is P.corutv\n"
        "import corutv.errors as E\n"
        "assert issubclass(P.ConvergenceError, E.ConvergenceError) and issubclass(P.CorutvError, E.CorutvError)\n"
        "import paper_1906_04572_b200.errors as OE; assert issubclass(P.ConvergenceError, OE.ConvergenceError)\n"
        "try:\n    raise P.ConvergenceError('cap', residual=1.0, history=[1, 2])\n"
        "except E.ConvergenceError as e:\n    assert e.history == [1, 2] and e.residual == 1.0\n"
        "P.install(corutv)\n"
        "print(len(done))\n" % (str(ROOT), str(ref), str(ref)))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert int(out.stdout.strip()) >= 10


def test_gaussian_matrix_is_the_reference_stream(golden):
    assert np.array_equal(P.gaussian_matrix(30, 7, 12345), golden["omega"]["val"])
    with pytest.raises(ValueError):
        P.gaussian_matrix(0, 3, 1)


def test_pass_counter():
    c = P.PassCounter()
    c.add()
    c.add(4)
    assert c.passes == 5


def test_install_rebinds_the_next_rows():
    # sor_svd / tsr_svd / inexact_alm / svt are rebound where the reference
    # package defines them (sketch.py:220-262, rpca.py:135-158, 258-273)
    import sys

    pkg = types.ModuleType("fakecorutv2")
    pkg.__path__ = []
    pkg.inexact_alm = pkg.svt = pkg.sor_svd = object()
    mods = {}
    for sub in ("sketch", "rpca", "bench"):
        m = types.ModuleType(f"fakecorutv2.{sub}")
        m.corutv = object()
        if sub == "sketch":
            m.sor_svd = m.tsr_svd = object()
        else:
            m.alm_corutv = m.inexact_alm = object()
        if sub == "rpca":
            m.svt = object()
        mods[sub] = m
        sys.modules[f"fakecorutv2.{sub}"] = m
    sys.modules["fakecorutv2"] = pkg
    try:
        done = P.install(pkg)
        assert mods["sketch"].sor_svd is P.sor_svd and mods["sketch"].tsr_svd is P.tsr_svd
        assert mods["rpca"].inexact_alm is P.inexact_alm and mods["rpca"].svt is P.svt
        assert mods["bench"].inexact_alm is P.inexact_alm
        assert pkg.inexact_alm is P.inexact_alm and pkg.svt is P.svt and pkg.sor_svd is P.sor_svd
        assert not hasattr(pkg, "tsr_svd")
        assert "fakecorutv2.rpca.inexact_alm" in done
    finally:
        for k in list(sys.modules):
            if k.startswith("fakecorutv2"):
                del sys.modules[k]
