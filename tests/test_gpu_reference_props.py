"""Property tests of the reference suite (pkg/tests/test_rpca.py:77-99,
test_sketch.py:82-132), restated against the device path: thresholding
(C_delta) rules, power iterations, the optimal-error bound, variant
agreement.  Inputs are built here with their own seeds; the properties are
the reference tests' assertions."""

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1906_04572_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _rank_k(seed, m, n, k):
    g = np.random.Generator(np.random.PCG64(seed))
    return g.standard_normal((m, k)) @ g.standard_normal((k, n))


def test_threshold_counting_rule():
    """rpca.py:107-119, |diag T| > delta counted (test_rpca.py:77-83)."""
    g = np.random.Generator(np.random.PCG64(1))
    u = np.linalg.qr(g.standard_normal((40, 4)))[0]
    v = np.linalg.qr(g.standard_normal((30, 4)))[0]
    b = (u * np.array([5.0, 3.0, 0.1, 0.05])) @ v.T
    mat, r = P.corutv_threshold(b, 1.0, P.SketchConfig(ell=8, q_power=2, seed=3))
    assert r == 2
    # the kept part is the rank-2 head of b
    head = (u[:, :2] * np.array([5.0, 3.0])) @ v[:, :2].T
    assert np.linalg.norm(mat - head) <= 1e-6 * np.linalg.norm(head)


def test_threshold_full_truncation():
    b = np.random.Generator(np.random.PCG64(2)).standard_normal((20, 15))
    mat, r = P.corutv_threshold(b, 10.0 * np.linalg.norm(b, 2), P.SketchConfig(ell=5, seed=1))
    assert r == 0 and np.all(mat == 0.0)


def test_threshold_exact_rank_input():
    b = _rank_k(3, 80, 60, 5)
    sig = np.linalg.svd(b, compute_uv=False)
    mat, r = P.corutv_threshold(b, 0.5 * sig[4], P.SketchConfig(ell=10, q_power=1, seed=2))
    assert r == 5
    assert np.linalg.norm(mat - b) <= 1e-8 * np.linalg.norm(b)


def test_lowrank_error_vanishes_on_exact_rank():
    a = _rank_k(31, 100, 90, 7)
    assert P.corutv_lowrank_error(a, P.SketchConfig(ell=14, seed=2)) <= 1e-9 * np.linalg.norm(a)


@pytest.mark.parametrize("seed", range(5))
def test_power_iterations_do_not_hurt(seed):
    a = O.gen_noisy_lowrank(150, 10, seed=40 + seed)[0]
    e0 = P.corutv_lowrank_error(a, P.SketchConfig(ell=20, q_power=0, seed=seed))
    e2 = P.corutv_lowrank_error(a, P.SketchConfig(ell=20, q_power=2, seed=seed))
    assert e2 <= e0


@pytest.mark.parametrize("seed", range(3))
def test_lowrank_error_respects_optimal_bound(seed):
    a = O.gen_noisy_lowrank(120, 8, seed=60 + seed)[0]
    ell = 16
    err = P.corutv_lowrank_error(a, P.SketchConfig(ell=ell, q_power=2, seed=seed))
    sig = np.linalg.svd(a, compute_uv=False)
    optimal = np.sqrt((sig[ell:] ** 2).sum())
    assert err >= optimal - 1e-9
    assert err <= 1.5 * optimal  # q = 2 is near-optimal (paper's bound)


def test_variants_agree_on_lowrank_input():
    a = _rank_k(29, 150, 120, 6)
    e = P.SketchConfig(ell=12, q_power=0, seed=4, variant=P.VARIANT_EXACT)
    p = P.SketchConfig(ell=12, q_power=0, seed=4, variant=P.VARIANT_APPROX)
    err = np.linalg.norm(P.corutv(a, e).lowrank() - P.corutv(a, p).lowrank())
    assert err <= 1e-6 * np.linalg.norm(a)


def test_tsr_and_sor_recover_exact_rank():
    a = _rank_k(37, 150, 130, 6)
    for fn in (P.tsr_svd, P.sor_svd):
        f = fn(a, P.SketchConfig(ell=12, q_power=1, seed=5))
        assert np.linalg.norm((f.u * f.sigma) @ f.v.T - a) <= 1e-8 * np.linalg.norm(a)
