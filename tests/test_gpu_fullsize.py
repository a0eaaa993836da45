"""BASELINE.json's full sizes on the device (C3: 131072 x 32768, ell 110,
q 2 -- 34.4 GB; C5: 262144 x 32768, ell 272, q 2 -- 68.7 GB), checked
through size-independent properties the oracle cannot reach at this scale:

* exact-d identity |A|_F^2 = |A - U T V'|_F^2 + |T|_F^2 (U T V' = P1 A P2);
* U, V orthonormal; T upper triangular with non-increasing |diag| (QRCP);
* the spectral gap of the planted rank shows in |diag T|;
* the reconstruction error sits at the planted noise / tail level;
* pass count 2(q+1)+1 (sketch.py:169-203); bitwise replay.
"""

import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

P = pytest.importorskip("paper_1906_04572_b200")
import bench  # noqa: E402  (the workload generators)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    yield
    torch.cuda.empty_cache()


def _check_factors(a, f, ell, k):
    dev = a.device
    u, t, v = f.u, f.t, f.v
    eye = torch.eye(ell, dtype=torch.float64, device=dev)
    assert (u.T @ u - eye).abs().max().item() < 1e-12
    assert (v.T @ v - eye).abs().max().item() < 1e-12
    assert torch.equal(t, torch.triu(t))
    d = t.diagonal().abs()
    assert bool((d[1:] <= d[:-1] * (1 + 1e-12)).all())
    a2 = float(P.dense.frobenius_norm(a)) ** 2
    err = P.corutv_lowrank_error(a, P.SketchConfig(ell=ell, q_power=2, seed=0))
    t2 = float((t ** 2).sum())
    assert abs(a2 - (err ** 2 + t2)) <= 1e-10 * a2
    return d.cpu(), err


def test_c3_full_size_properties():
    m, n, ell, q, k, noise, _ = bench.WORKLOADS["c3"]
    a = bench.gen_rows_device(torch, "c3", 0, m, torch.device("cuda", 0))
    cnt = P.PassCounter()
    f = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, seed=0), cnt)
    assert cnt.passes == 2 * (q + 1) + 1
    d, err = _check_factors(a, f, ell, k)
    assert d[k - 1] / d[k] > 10.0           # rank-100 signal above the 1e-4 noise
    assert err <= 1.01 * noise * math.sqrt(m * n)
    g = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, seed=0))
    assert torch.equal(f.t, g.t) and torch.equal(f.u, g.u)
    del a, f, g


def test_c5_full_size_properties():
    m, n, ell, q, k, noise, _ = bench.WORKLOADS["c5"]
    a = bench.gen_rows_device(torch, "c5", 0, m, torch.device("cuda", 0))
    f = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, seed=0))
    d, err = _check_factors(a, f, ell, k)
    # sigma_i = 0.99^i on a near-orthonormal 512-column factor: the optimal
    # rank-272 error is ~ sqrt(sum_{i > 272} 0.99^(2i)) = 0.454
    tail = math.sqrt(sum(0.99 ** (2 * i) for i in range(ell + 1, k + 1)))
    assert 0.8 * tail <= err <= 1.25 * tail
    assert abs(float(d[0]) - 0.99) < 0.1
    del a, f
