"""The device experiment harness (harness.py; bench.py:165-306)
against the reference harness's own rows (tests/golden: n = 80, k = 6,
three trials, every method; rpca-recovery at n = 60, 80).

Tolerances: estimates and errors of well-conditioned methods to 1e-8
relative; trial standard deviations (differences of nearly equal numbers)
to 1e-8 of the row's scale.  tsr-svd's low-rank errors at ell = k are
dominated by its ill-conditioned core pseudoinverse (the reference's own
trials spread 0.4 .. 150): compared at 1e-3 relative.  Integer columns
(indices, ranks, nnz, iterations, flop estimates) exactly.
"""

import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1906_04572_b200")
from paper_1906_04572_b200 import harness as H  # noqa: E402
from paper_1906_04572_b200 import synth as S  # noqa: E402

ALL = ("svd", "qrcp", "utv-approx", "corutv", "tsr-svd", "sor-svd")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def test_noisy_generator_matches_reference(golden):
    a, _ = S.gen_noisy_lowrank(S.NoisyLowRankSpec(n=80, k=6, seed=0, noise_coeff=0.1))
    assert np.abs(a - golden["synth_noisy"]["a"]).max() <= 1e-13


def _check_rows(rows, g, loose=()):
    assert [r[0] for r in rows] == [int(x) for x in g["c0"]]
    assert [r[1] for r in rows] == [str(x) for x in g["method"]]
    for r, c2, c3, c4, meth in zip(rows, g["c2"], g["c3"], g["c4"], g["method"]):
        rtol = 1e-3 if str(meth) in loose else 1e-8
        scale = max(abs(c2), abs(c4), 1e-300)
        assert abs(r[2] - c2) <= rtol * abs(c2) + 1e-12 * scale, (r, c2)
        assert abs(r[3] - c3) <= rtol * scale + 1e-12, (r, c3)
        assert abs(r[4] - c4) <= rtol * scale + 1e-12, (r, c4)


def test_sv_compare_matches_reference(golden):
    rows = H.run_sv_compare(H.ExperimentConfig("sv-compare", n=80, k=6, trials=3, q_power=1, methods=ALL))
    _check_rows(rows, golden["harness_sv_compare"])


def test_lowrank_error_matches_reference(golden):
    rows = H.run_lowrank_error(H.ExperimentConfig("lowrank-error", n=80, k=6, trials=3, q_power=1, methods=ALL))
    _check_rows(rows, golden["harness_lowrank_error"], loose=("tsr-svd",))


def test_rpca_recovery_matches_reference(golden):
    g = golden["harness_rpca_recovery"]
    rows = H.run_rpca_recovery(H.ExperimentConfig("rpca-recovery", sizes=(60, 80)))
    assert [r[:5] for r in rows] == [
        (int(n), str(s), int(r), int(z), int(i))
        for n, s, r, z, i in zip(g["n"], g["solver"], g["rank_l"], g["nnz_s"], g["iters"])]
    assert [r[6] for r in rows] == [int(x) for x in g["flops"]]
    assert np.allclose([r[5] for r in rows], g["zeta"], rtol=1e-6, atol=0)


def test_reports_are_byte_identical_and_schedule_independent(tmp_path, monkeypatch):
    # bench.py:11-12: byte-identical re-runs; here also across worker counts
    outs = []
    for threads in ("8", "8", "1", "3"):
        monkeypatch.setenv("CORUTV_THREADS", threads)
        p = tmp_path / f"sv{len(outs)}.csv"
        H.run_sv_compare(H.ExperimentConfig("sv-compare", n=120, k=8, trials=6, q_power=1,
                                            methods=("corutv", "tsr-svd", "sor-svd", "utv-approx"),
                                            out_path=str(p)))
        outs.append(p.read_bytes())
    assert all(o == outs[0] for o in outs)


def test_default_sv_compare_runs_fast():
    # the reference harness's default configuration (n = 400, 20 trials)
    t0 = time.perf_counter()
    rows = H.run_sv_compare(H.ExperimentConfig("sv-compare"))
    dt = time.perf_counter() - t0
    assert len(rows) == 5 * 40
    assert dt < 30.0
