"""InexactALM baseline on the device (rpca.py:135-158, 258-273):
warm-started one-sided Jacobi SVD (dense.py:313-376), singular value
thresholding, and the ALM loop, against the reference's golden vectors
and the oracle.

Tolerances: the device sweeps recompute nothing the reference caches, but
they round differently (FMA dot products, DMMA for the warm-start GEMMs),
so floats are compared at 1e-12 (spectra) / 1e-10 (vectors, thresholded
matrices, relative to the input's scale) and the ALM's integer histories
(rank, nnz, cap, iteration count) exactly.
"""

import time

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


def _sign_close(x, y, tol):
    s = np.sign(np.sum(x * y, axis=0))
    s[s == 0] = 1.0
    return np.abs(x * s - y).max() <= tol


@pytest.mark.parametrize("name", ["svdwarm_sq", "svdwarm_tall", "svdwarm_wide"])
def test_warm_jacobi_svd_golden(golden, name):
    c = golden[name]
    f = P.jacobi_svd(c["a"], v_init=c["v_init"])
    s0 = c["sigma"][0]
    assert np.abs(f.sigma - c["sigma"]).max() <= 1e-13 * s0
    # warm start: same factors as the reference, signs included
    assert np.abs(f.u - c["u"]).max() <= 1e-10
    assert np.abs(f.v - c["v"]).max() <= 1e-10


def test_warm_jacobi_rejects_wrong_v_init(golden):
    c = golden["svdwarm_wide"]
    with pytest.raises(ValueError, match="v_init must be 13x13"):
        P.jacobi_svd(c["a"], v_init=np.eye(29))


@pytest.mark.parametrize("shape", [(300, 300), (333, 257), (190, 411)])
def test_grid_jacobi_matches_oracle(shape):
    # cores above one CTA's shared memory run on the cooperative grid kernel
    g = np.random.Generator(np.random.PCG64(sum(shape)))
    a = g.standard_normal(shape)
    f = P.jacobi_svd(a)
    u, s, v = O.jacobi_svd(a)
    assert np.abs(f.sigma - s).max() <= 1e-12 * s[0]
    # gaps of a Gaussian matrix's spectrum are >= ~1e-3 s0: vectors to 1e-9
    assert _sign_close(f.u, u, 1e-9) and _sign_close(f.v, v, 1e-9)
    k = min(shape)
    assert np.abs(f.u.T @ f.u - np.eye(k)).max() <= 1e-12
    assert np.abs((f.u * f.sigma) @ f.v.T - a).max() <= 1e-11 * s[0]


def test_grid_jacobi_zero_columns_completion():
    # exact zero columns never rotate: zero singular values, completed by
    # unit-vector Gram-Schmidt (dense.py:285-310) in the grid kernel.  Square
    # input: for m > n the reference completes inside its QR-preconditioned
    # space (dense.py:319-323, 350-351), so only the span would compare
    g = np.random.Generator(np.random.PCG64(5))
    a = g.standard_normal((240, 240))
    a[:, [3, 77, 200]] = 0.0
    f = P.jacobi_svd(a)
    u, s, v = O.jacobi_svd(a)
    assert np.array_equal(f.sigma[-3:], np.zeros(3))
    assert np.abs(f.sigma - s).max() <= 1e-12 * s[0]
    assert np.abs(f.u.T @ f.u - np.eye(240)).max() <= 1e-12
    assert np.abs(f.u[:, -3:] - u[:, -3:]).max() <= 1e-10


def test_grid_jacobi_warm_start_takes_fewer_sweeps():
    g = np.random.Generator(np.random.PCG64(9))
    a = g.standard_normal((400, 400))
    v0 = P.jacobi_svd(a + 1e-6 * g.standard_normal((400, 400))).v
    f = P.jacobi_svd(a, v_init=v0)
    u, s, v = O.jacobi_svd(a, v0)
    assert np.abs(f.sigma - s).max() <= 1e-12 * s[0]
    assert np.abs(f.v - v).max() <= 1e-9 and np.abs(f.u - u).max() <= 1e-9


@pytest.mark.parametrize("name", ["svt_diag", "svt_zero", "svt_nuc", "svt_wide", "svt_rank"])
def test_svt_golden(golden, name):
    c = golden[name]
    mat, r = P.svt(c["b"], float(c["delta"]))
    assert r == int(c["r"])
    assert np.abs(mat - c["mat"]).max() <= 1e-10 * max(1.0, np.abs(c["b"]).max())


def test_svt_device_in_device_out():
    b = torch.randn(50, 50, dtype=torch.float64, device="cuda")
    mat, r = P.svt(b, 1.0)
    assert mat.is_cuda and 0 < r <= 50
    want, rw = O.svt(b.cpu().numpy(), 1.0)
    assert r == rw and np.abs(mat.cpu().numpy() - want).max() <= 1e-10


def test_svt_rejects_negative_delta():
    with pytest.raises(ValueError, match="delta"):
        P.svt(np.eye(3), -1.0)


@pytest.mark.parametrize("n", [60, 100])
def test_inexact_alm_golden(golden, n):
    c = golden[f"ialm_n{n}"]
    sol = P.inexact_alm(c["m"], P.AlmConfig(ell=int(c["ell_history"][0])))
    assert sol.iterations == int(c["iterations"])
    assert sol.rank_history == [int(x) for x in c["rank_history"]]
    assert sol.nnz_history == [int(x) for x in c["nnz_history"]]
    assert sol.ell_history == [int(x) for x in c["ell_history"]]
    assert sol.rank_of_l == int(c["rank_of_l"]) and sol.nnz_of_s == int(c["nnz_of_s"])
    assert np.allclose(sol.residuals, c["residuals"], rtol=1e-7, atol=0)
    assert np.allclose(sol.mu_history, c["mu_history"], rtol=1e-12, atol=0)
    scale = np.abs(c["m"]).max()
    assert np.abs(sol.l - c["l"]).max() <= 1e-9 * scale
    assert np.abs(sol.s - c["s"]).max() <= 1e-9 * scale


def test_inexact_alm_max_iter_history(golden):
    c = golden["ialm_maxiter"]
    with pytest.raises(P.ConvergenceError) as exc:
        P.inexact_alm(c["m"], P.AlmConfig(max_iter=2))
    assert np.allclose(exc.value.history, c["history"], rtol=1e-9, atol=0)


def test_inexact_alm_zero_matrix():
    sol = P.inexact_alm(np.zeros((30, 30)), P.AlmConfig())
    assert sol.iterations == 1 and not sol.l.any() and not sol.s.any()


def test_inexact_alm_wide_input_fails_like_the_reference():
    # the warm start handed to the second SVD is the wide matrix's n x m
    # right factor; dense.py:316-318 rejects it (the reference does the same)
    g = np.random.Generator(np.random.PCG64(3))
    m = g.standard_normal((30, 50))
    with pytest.raises(ValueError, match="v_init must be 30x30"):
        O.inexact_alm(m, ell=10)
    with pytest.raises(ValueError, match="v_init must be 30x30"):
        P.inexact_alm(m, P.AlmConfig(ell=10))


def test_inexact_alm_desk_scale_golden(golden):
    # test_rpca.py:160-180 instance (n = 400: grid Jacobi path)
    c = golden["ialm_n400"]
    k = 20
    m, l_true, s_true = O.gen_rpca_instance(400, k, 8000, seed=0)
    assert m.sum() == float(c["m_sum"])
    t0 = time.perf_counter()
    sol = P.inexact_alm(m, P.AlmConfig(ell=2 * k))
    dt = time.perf_counter() - t0
    assert sol.iterations == int(c["iterations"])
    assert sol.rank_history == [int(x) for x in c["rank_history"]]
    assert sol.nnz_history == [int(x) for x in c["nnz_history"]]
    assert sol.ell_history == [int(x) for x in c["ell_history"]]
    assert sol.rank_of_l == k and sol.nnz_of_s == 8000
    assert np.array_equal(np.flatnonzero(np.abs(sol.s) > 1e-12), c["s_support"])
    assert np.abs(sol.l[::37, ::41] - c["l_sample"]).max() <= 1e-8 * np.abs(m).max()
    assert np.linalg.norm(sol.l - l_true) <= 1e-4 * np.linalg.norm(l_true)
    assert dt < 60.0  # the reference's own desk-scale budget (test_acceptance.py:262-270)


@pytest.mark.parametrize("n", [40, 300])
def test_jacobi_svd_sweep_cap_and_tolerance(n):
    # dense.py:357-376 arguments: max_sweeps exceeded -> ConvergenceError
    # (one-CTA path for n = 40, grid path for n = 300); a looser tol stops
    # earlier with the spectrum still right to ~tol
    g = np.random.Generator(np.random.PCG64(n))
    a = g.standard_normal((n, n))
    with pytest.raises(P.ConvergenceError, match="did not converge"):
        P.jacobi_svd(a, max_sweeps=1)
    f = P.jacobi_svd(a, tol=1e-8)
    s = O.jacobi_svd(a)[1]
    assert np.abs(f.sigma - s).max() <= 1e-6 * s[0]
