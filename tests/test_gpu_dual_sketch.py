"""The one-pass dual sketch behind tsr_svd (sketch.py:160-163 `fused_sketch`,
used by tsr_svd sketch.py:220-241): y = A psi and z = A' phi from a single
sweep over a device-resident A (csrc/dual_sketch.cuh, l <= 8).

The library switches to it for matrices with many 128-row sub-blocks; the
tests lower that threshold (CORUTV_DUAL_MIN_SUBS) so mid-size shapes with
ragged edges run through it, and compare with the two-sweep path
(CORUTV_DUAL_OFF=1) and with the CPU oracle on identical psi / phi."""

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1906_04572_b200")
from paper_1906_04572_b200 import _lib  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _matrix(m, n, k, seed, noise=1e-5):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.randn((m, k), generator=g, dtype=torch.float64, device="cuda")
    y = torch.randn((n, k), generator=g, dtype=torch.float64, device="cuda")
    sig = torch.logspace(0, -2, k, dtype=torch.float64, device="cuda")
    a = (x * sig) @ y.T
    a += noise * torch.randn((m, n), generator=g, dtype=torch.float64, device="cuda")
    return a


def _sign_close(x, y, tol):
    s = torch.sign((x * y).sum(dim=0))
    s[s == 0] = 1.0
    return float((x * s - y).abs().max()) <= tol


def _a_sweeps(fn):
    """Run fn() and return (result, launches that swept the data matrix): the
    library's measurement hooks count them (class 1 of corutv_profile_end)."""
    import ctypes

    h = _lib.handle(0)
    h.call("corutv_profile_begin")
    out = fn()
    o12 = (ctypes.c_double * 12)()
    n = ctypes.c_int64(0)
    h.call("corutv_profile_end", o12, ctypes.byref(n))
    return out, int(o12[4])


# (m, n, ell, k): ragged row sub-blocks and k-tiles, tall and wide,
# > 4 x 148 sub-blocks (two panels per CTA), the narrowest n (one column block)
SHAPES = [(3000, 700, 8, 5), (5000, 300, 6, 4), (2049, 257, 5, 3), (1300, 4100, 7, 6), (1024, 256, 8, 5),
          (80000, 512, 7, 4), (77000, 130, 3, 2), (4000, 128, 1, 1)]


@pytest.mark.parametrize("m,n,ell,k", SHAPES)
def test_dual_sketch_matches_two_sweeps(monkeypatch, m, n, ell, k):
    a = _matrix(m, n, k, m + n + ell)
    cfg = P.SketchConfig(ell=ell, seed=21)
    monkeypatch.setenv("CORUTV_DUAL_OFF", "1")
    two, sweeps2 = _a_sweeps(lambda: P.tsr_svd(a, cfg))
    monkeypatch.setenv("CORUTV_DUAL_OFF", "0")
    monkeypatch.setenv("CORUTV_DUAL_MIN_SUBS", "2")
    cnt = P.PassCounter()
    one, sweeps1 = _a_sweeps(lambda: P.tsr_svd(a, cfg, cnt))
    assert cnt.passes == 1
    assert (sweeps1, sweeps2) == (1, 2)  # A swept once by the dual kernel, twice by the two GEMMs
    s1, s2 = one.sigma, two.sigma
    assert float((s1[:k] - s2[:k]).abs().max()) <= 1e-12 * float(s2[0])
    assert _sign_close(one.u[:, :k], two.u[:, :k], 1e-9)
    assert _sign_close(one.v[:, :k], two.v[:, :k], 1e-9)
    la = (one.u * one.sigma) @ one.v.T
    lb = (two.u * two.sigma) @ two.v.T
    assert float((la - lb).norm()) <= 1e-9 * float(lb.norm())
    # the sketches differ only in summation order, so a second run is bitwise
    again = P.tsr_svd(a, cfg)
    assert torch.equal(again.sigma, one.sigma) and torch.equal(again.u, one.u) and torch.equal(again.v, one.v)


def test_dual_sketch_matches_oracle(monkeypatch):
    monkeypatch.setenv("CORUTV_DUAL_MIN_SUBS", "2")
    m, n, ell, k = 2600, 900, 8, 5
    a = _matrix(m, n, k, 5, noise=1e-7)
    rng = np.random.Generator(np.random.PCG64(3))
    psi = rng.standard_normal((n, ell))
    phi = rng.standard_normal((m, ell))
    f = P.tsr_svd(a, P.SketchConfig(ell=ell), psi=psi, phi=phi)
    o = O.tsr_svd(a.cpu().numpy(), ell, psi=psi, phi=phi)
    sig = f.sigma.cpu().numpy()
    assert np.abs(sig[:k] - o["sigma"][:k]).max() <= 1e-9 * o["sigma"][0]
    for x, y in ((f.u, o["u"]), (f.v, o["v"])):
        assert _sign_close(x[:, :k], torch.from_numpy(np.ascontiguousarray(y[:, :k])).cuda(), 1e-7)


def test_wider_sketches_keep_two_sweeps(monkeypatch):
    monkeypatch.setenv("CORUTV_DUAL_MIN_SUBS", "2")
    a = _matrix(3000, 500, 5, 2)
    _, sweeps = _a_sweeps(lambda: P.tsr_svd(a, P.SketchConfig(ell=9, seed=1)))
    assert sweeps == 2


def test_dual_sketch_reports_nonfinite(monkeypatch):
    monkeypatch.setenv("CORUTV_DUAL_MIN_SUBS", "2")
    a = _matrix(1500, 400, 4, 8)
    for pos in ((0, 0), (1499, 399), (777, 123)):
        b = a.clone()
        b[pos] = float("nan") if pos[0] else float("inf")
        with pytest.raises(ValueError, match="non-finite"):
            P.tsr_svd(b, P.SketchConfig(ell=6, seed=1))


def test_dual_sketch_unaligned_view(monkeypatch):
    """A column-offset view (8-byte aligned only) goes through the padded copy."""
    monkeypatch.setenv("CORUTV_DUAL_MIN_SUBS", "2")
    big = _matrix(2000, 401, 4, 12)
    a = big[:, 1:]
    cfg = P.SketchConfig(ell=8, seed=2)
    one = P.tsr_svd(a, cfg)
    monkeypatch.setenv("CORUTV_DUAL_OFF", "1")
    two = P.tsr_svd(a.contiguous(), cfg)
    assert float((one.sigma[:4] - two.sigma[:4]).abs().max()) <= 1e-12 * float(two.sigma[0])


def test_dual_sketch_strided_aligned_view(monkeypatch):
    """Columns [0, 400) of a 402-column matrix: 16-byte aligned rows with an
    even leading dimension go to TMA as they are (no padded copy)."""
    monkeypatch.setenv("CORUTV_DUAL_MIN_SUBS", "2")
    big = _matrix(2300, 402, 4, 14)
    a = big[:, :400]
    cfg = P.SketchConfig(ell=5, seed=6)
    one, sweeps = _a_sweeps(lambda: P.tsr_svd(a, cfg))
    assert sweeps == 1
    monkeypatch.setenv("CORUTV_DUAL_OFF", "1")
    two = P.tsr_svd(a.contiguous(), cfg)
    assert float((one.sigma[:4] - two.sigma[:4]).abs().max()) <= 1e-12 * float(two.sigma[0])
    assert _sign_close(one.v[:, :4], two.v[:, :4], 1e-9)
