"""Host-side pieces of the device harness (harness.py / synth.py): config
validation, CSV bytes, and the seeded generators against the reference's
golden outputs (bench.py:82-150, synth.py:77-134)."""

import numpy as np
import pytest

import oracle as O
from paper_1906_04572_b200 import harness as H
from paper_1906_04572_b200 import synth as S


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError, match="experiment"):
        H.ExperimentConfig(experiment="nope")
    with pytest.raises(ValueError, match="trials"):
        H.ExperimentConfig(experiment="sv-compare", trials=0)
    with pytest.raises(ValueError, match="unknown method"):
        H.ExperimentConfig(experiment="sv-compare", methods=("svd", "lu"))
    with pytest.raises(ValueError, match="unknown solver"):
        H.ExperimentConfig(experiment="rpca-recovery", solvers=("admm",))
    with pytest.raises(ValueError, match="outside"):
        H.ExperimentConfig(experiment="lowrank-error", k=5, n=20, ell_sweep=(4,))
    c = H.ExperimentConfig(experiment="lowrank-error", k=20)
    assert c.resolved_ell() == 40 and c.resolved_sweep() == (20, 30, 40, 60)


def test_write_csv_bytes(tmp_path):
    p = tmp_path / "r.csv"
    H.write_csv(p, H.RPCA_HEADER, [(60, "alm-corutv", 3, 180, 13, 5.475297263e-06, 62474400)])
    assert p.read_bytes() == b"n,solver,rank_l,nnz_s,iters,zeta,flops_est\n60,alm-corutv,3,180,13,5.475297263e-06,62474400\n"


def test_threads_env_is_validated(monkeypatch):
    monkeypatch.setenv("CORUTV_THREADS", "x")
    with pytest.raises(ValueError, match="CORUTV_THREADS"):
        H._max_workers()
    monkeypatch.setenv("CORUTV_THREADS", "0")
    assert H._max_workers() == 1


def test_noiseless_generator_matches_reference(golden):
    # LAPACK Householder (np.linalg.qr) follows dense.py:104-115's reflector
    # convention, so the planted factors agree to rounding
    a, sig = S.gen_noisy_lowrank(S.NoisyLowRankSpec(n=50, k=4, seed=3, noise_coeff=0.0))
    ref = golden["synth_noisy"]["a_noiseless"]
    assert np.abs(a - ref).max() <= 1e-14
    assert sig[3] > 0 and not sig[4:].any()


def test_rpca_generator_matches_oracle():
    m, l0, s0 = S.gen_rpca_instance(S.RpcaInstanceSpec(n=40, k=2, s=80, seed=4))
    mo, lo, so = O.gen_rpca_instance(40, 2, 80, seed=4)
    assert np.array_equal(m, mo) and np.array_equal(s0, so)


def test_spec_validation():
    with pytest.raises(ValueError):
        S.NoisyLowRankSpec(n=10, k=10)
    with pytest.raises(ValueError):
        S.RpcaInstanceSpec(n=10, k=2, s=101)


def test_solver_flops_matches_oracle():
    class Sol:
        rank_history = [3, 5, 5]
        ell_history = [6, 4, 6]

    want = O.solver_flops(60, 1, Sol.rank_history, Sol.ell_history)
    assert H.solver_flops("alm-corutv", 60, 1, Sol) == want
    assert H.solver_flops("inexact-alm", 60, 1, Sol) == sum(
        H.svd_flop_estimate(60, 60) + 2 * 60 * 60 * r + 8 * 60 * 60 for r in Sol.rank_history)
