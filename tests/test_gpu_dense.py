"""Device Jacobi SVD / singular values against the reference's own dense
tests (pkg/tests/test_dense.py:132-198), same inputs and bars."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1906_04572_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _gauss(rng, m, n):
    return rng.standard_normal((m, n))


def test_svd_diagonal():
    f = P.jacobi_svd(np.diag([2.0, 1.0]))
    assert np.abs(f.sigma - [2.0, 1.0]).max() < 1e-14


def test_svd_zeros():
    f = P.jacobi_svd(np.zeros((4, 3)))
    assert np.all(f.sigma == 0.0)
    assert np.abs(f.u.T @ f.u - np.eye(3)).max() < 1e-14
    assert np.abs(f.v.T @ f.v - np.eye(3)).max() < 1e-14


@pytest.mark.parametrize("shape", [(40, 25), (25, 25), (10, 30), (7, 1), (500, 300), (260, 700)])
def test_svd_matches_lapack_values(shape):
    # test_dense.py:144-155, plus two grid-path shapes
    rng = np.random.Generator(np.random.PCG64(sum(shape) * 7919))
    a = rng.standard_normal(shape)
    f = P.jacobi_svd(a)
    want = np.linalg.svd(a, compute_uv=False)
    assert np.abs(f.sigma - want).max() < 1e-11 * want[0]
    k = min(shape)
    assert np.linalg.norm((f.u * f.sigma) @ f.v.T - a) < 1e-9 * np.linalg.norm(a)
    assert np.abs(f.u.T @ f.u - np.eye(k)).max() < 1e-10
    assert np.abs(f.v.T @ f.v - np.eye(k)).max() < 1e-10
    assert np.all(np.diff(f.sigma) <= 0) and np.all(f.sigma >= 0)


@pytest.mark.parametrize("shape", [(30, 20), (400, 300)])
def test_svd_values_only_matches_full(rng, shape):
    a = _gauss(rng, *shape)
    assert np.array_equal(P.singular_values(a), P.jacobi_svd(a).sigma)


def test_svd_graded_spectrum_absolute_accuracy():
    rng = np.random.Generator(np.random.PCG64(5))
    q1 = np.linalg.qr(rng.standard_normal((80, 80)))[0]
    q2 = np.linalg.qr(rng.standard_normal((80, 80)))[0]
    planted = np.linspace(1.0, 1e-9, 80)
    a = (q1 * planted) @ q2.T
    assert np.abs(P.singular_values(a) - planted).max() < 1e-12


def test_svd_warm_start_agrees(rng):
    a = _gauss(rng, 30, 30)
    cold = P.jacobi_svd(a)
    warm = P.jacobi_svd(a + 1e-6 * _gauss(rng, 30, 30), v_init=cold.v)
    assert np.abs(warm.sigma - cold.sigma).max() < 1e-4
    warm_same = P.jacobi_svd(a, v_init=cold.v)
    assert np.abs(warm_same.sigma - cold.sigma).max() < 1e-11


def test_svd_optimality_identity(rng):
    a = _gauss(rng, 30, 20)
    f = P.jacobi_svd(a)
    for k in range(21):
        trunc = (f.u[:, :k] * f.sigma[:k]) @ f.v[:, :k].T
        err = np.linalg.norm(a - trunc)
        want = np.sqrt((f.sigma[k:] ** 2).sum())
        assert abs(err - want) < 1e-9 * max(want, 1.0)


@pytest.mark.parametrize("n", [12, 300])
def test_svd_sweep_cap_raises(n):
    rng = np.random.Generator(np.random.PCG64(6))
    a = rng.standard_normal((n, n))
    with pytest.raises(P.ConvergenceError, match="residual"):
        P.jacobi_svd(a, max_sweeps=1)
