"""sor_svd / tsr_svd (sketch.py:220-262) and the device Jacobi SVD
(dense.py:357-376) against the reference's golden vectors and the oracle.

Singular vectors are compared up to column sign and only where they are
determined: distinct singular values above the planted rank (the trailing
ones of an exactly rank-k input are rounding noise in every implementation).
"""

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


@pytest.mark.parametrize("name", ["svd_tall", "svd_wide", "svd_square", "svd_zero_cols"])
def test_jacobi_svd_golden(golden, name):
    c = golden[name]
    f = P.dense.jacobi_svd(c["a"])
    s0 = c["sigma"][0]
    assert np.abs(f.sigma - c["sigma"]).max() <= 1e-13 * s0
    k = int((c["sigma"] > 1e-12 * s0).sum())
    assert _sign_close(f.u[:, :k], c["u"][:, :k], 1e-12)
    assert _sign_close(f.v[:, :k], c["v"][:, :k], 1e-12)
    # completion of zero singular values: same deterministic vectors
    assert np.abs(f.u - c["u"] * np.sign(np.sum(f.u * c["u"], axis=0))).max() <= 1e-12
    assert np.abs(f.u.T @ f.u - np.eye(f.u.shape[1])).max() <= 1e-13
    assert np.abs((f.u * f.sigma) @ f.v.T - c["a"]).max() <= 1e-13 * s0


RANK = {"sor_q1": 7, "sor_q0_approx": 5, "sor_c2small": 40, "tsr_tall": 6, "tsr_wide": 5, "tsr_noisy": 6}
ARGS = {"sor_q1": (1, 8), "sor_q0_approx": (0, 3), "sor_c2small": (2, 77), "tsr_tall": (0, 4),
        "tsr_wide": (0, 6), "tsr_noisy": (0, 1)}


@pytest.mark.parametrize("name", sorted(RANK))
def test_svd_sketches_golden(golden, name):
    c = golden[name]
    q, seed = ARGS[name]
    ell = c["sigma"].size
    variant = P.VARIANT_APPROX if "approx" in name else P.VARIANT_EXACT
    cfg = P.SketchConfig(ell=ell, q_power=q, seed=seed, variant=variant)
    cnt = P.PassCounter()
    f = (P.sor_svd if name.startswith("sor") else P.tsr_svd)(c["a"], cfg, cnt)
    assert cnt.passes == int(c["passes"])
    assert isinstance(f.u, np.ndarray) and f.u.shape == c["u"].shape and f.v.shape == c["v"].shape
    k, s0 = RANK[name], c["sigma"][0]
    assert np.abs(f.sigma[:k] - c["sigma"][:k]).max() <= 1e-9 * s0
    assert bool(np.all(np.diff(f.sigma) <= 0.0)) and bool(np.all(f.sigma >= 0.0))
    # the rank-k part of u diag(sigma) v' is determined
    lk = (f.u[:, :k] * f.sigma[:k]) @ f.v[:, :k].T
    rk = (c["u"][:, :k] * c["sigma"][:k]) @ c["v"][:, :k].T
    assert np.abs(lk - rk).max() <= 1e-8 * s0
    if name != "sor_c2small":   # sigma_1..40 = 1 are repeated: vectors not unique
        assert _sign_close(f.u[:, :k], c["u"][:, :k], 1e-8)
        assert _sign_close(f.v[:, :k], c["v"][:, :k], 1e-8)
    assert np.abs(f.u.T @ f.u - np.eye(ell)).max() <= 1e-10
    assert np.abs(f.v.T @ f.v - np.eye(ell)).max() <= 1e-10


def test_sor_svd_matches_corutv_core_spectrum():
    rng = np.random.Generator(np.random.PCG64(5))
    m, n, ell = 3000, 2000, 60
    a = rng.standard_normal((m, 40)) @ rng.standard_normal((40, n)) + 1e-3 * rng.standard_normal((m, n))
    A = torch.from_numpy(a).cuda()
    cfg = P.SketchConfig(ell=ell, q_power=1, seed=3)
    f = P.sor_svd(A, cfg)
    g = P.corutv(A, cfg)
    assert f.u.is_cuda and f.sigma.is_cuda
    sv_t = P.singular_values(g.t)
    sv_t = sv_t.cpu().numpy() if hasattr(sv_t, "cpu") else sv_t
    s = f.sigma.cpu().numpy()
    assert np.abs(s - sv_t).max() <= 1e-11 * s[0]
    # same rank-ell approximant as corutv (both are P1 A P2)
    la = (f.u * f.sigma) @ f.v.T
    lb = g.u @ (g.t @ g.v.T)
    assert (la - lb).abs().max().item() <= 1e-10 * s[0]


def test_tsr_svd_matches_oracle_midsize():
    rng = np.random.Generator(np.random.PCG64(9))
    m, n, ell, k = 1500, 2200, 30, 12
    a = (rng.standard_normal((m, k)) * np.logspace(0, -2, k)) @ rng.standard_normal((k, n))
    a += 1e-6 * rng.standard_normal((m, n))
    f = P.tsr_svd(a, P.SketchConfig(ell=ell, seed=11))
    o = O.tsr_svd(a, ell, 11)
    assert np.abs(f.sigma[:k] - o["sigma"][:k]).max() <= 1e-9 * o["sigma"][0]
    assert _sign_close(f.u[:, :k], o["u"][:, :k], 1e-7)
    assert _sign_close(f.v[:, :k], o["v"][:, :k], 1e-7)


def test_svd_sketch_validation():
    rng = np.random.Generator(np.random.PCG64(2))
    with pytest.raises(ValueError, match="rows >= cols"):
        P.sor_svd(rng.standard_normal((20, 30)), P.SketchConfig(ell=5))
    with pytest.raises(ValueError, match="exceeds"):
        P.tsr_svd(rng.standard_normal((20, 30)), P.SketchConfig(ell=25))
    a = rng.standard_normal((40, 30))
    a[3, 4] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        P.tsr_svd(a, P.SketchConfig(ell=5))


@pytest.mark.parametrize("chunk_bytes", [None, 300000])
def test_svd_sketches_host_streamed_are_bitwise_device(monkeypatch, chunk_bytes):
    """Host inputs stream through corutv_{sor,tsr}_svd_host (tsr: both
    products consume each row chunk) -- bit-identical to the device calls."""
    if chunk_bytes is not None:
        monkeypatch.setenv("CORUTV_HOST_CHUNK_BYTES", str(chunk_bytes))
    rng = np.random.Generator(np.random.PCG64(17))
    a = rng.standard_normal((2500, 12)) @ rng.standard_normal((12, 430)) + 1e-4 * rng.standard_normal((2500, 430))
    ad = torch.from_numpy(a).cuda()
    for fn, cfg in ((P.sor_svd, P.SketchConfig(ell=20, q_power=1, seed=3)),
                    (P.sor_svd, P.SketchConfig(ell=20, q_power=0, seed=3, variant=P.VARIANT_APPROX)),
                    (P.tsr_svd, P.SketchConfig(ell=20, seed=3))):
        cnt = P.PassCounter()
        fh = fn(a, cfg, cnt)
        fd = fn(ad, cfg)
        assert isinstance(fh.u, np.ndarray)
        assert cnt.passes == (1 if fn is P.tsr_svd else 2 * (cfg.q_power + 1) + (cfg.variant == P.VARIANT_EXACT))
        for x, y in ((fh.u, fd.u), (fh.sigma, fd.sigma), (fh.v, fd.v)):
            assert np.array_equal(x, y.cpu().numpy())
