"""CUDA-graph replay of small fixed-shape decompositions (corutv_decompose):
the second call with the same (A, Omega, shape, ell, q) captures the whole
decomposition, later calls replay it.  Replays must be bitwise the ordinary
path, follow A's current contents, and raise the ordinary path's errors."""

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


def _mat(m, n, k, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    a = g.standard_normal((m, k)) @ g.standard_normal((k, n)) + 1e-6 * g.standard_normal((m, n))
    return torch.from_numpy(a).cuda()


@pytest.mark.parametrize("m,n,ell,q", [(1000, 1000, 15, 0), (700, 500, 40, 1), (4000, 3000, 50, 1)])
def test_graph_replay_is_bitwise_the_ordinary_path(m, n, ell, q):
    a = _mat(m, n, 10, 7)
    om = torch.from_numpy(P.gaussian_matrix(n, ell, 3)).cuda()
    cfg = P.SketchConfig(ell=ell, q_power=q)
    fs = [P.corutv(a, cfg, omega=om) for _ in range(4)]  # ordinary, capture + replay, replay, replay
    torch.cuda.synchronize()
    for f in fs[1:]:
        assert torch.equal(f.u, fs[0].u) and torch.equal(f.t, fs[0].t) and torch.equal(f.v, fs[0].v)
        pa = f.perm.cpu() if hasattr(f.perm, "cpu") else f.perm
        pb = fs[0].perm.cpu() if hasattr(fs[0].perm, "cpu") else fs[0].perm
        assert np.array_equal(np.asarray(pa), np.asarray(pb))
    # a fresh buffer (another pointer) takes the ordinary path: same bits
    f2 = P.corutv(a.clone(), cfg, omega=om.clone())
    assert torch.equal(f2.t, fs[0].t) and torch.equal(f2.u, fs[0].u)


def test_graph_replay_reads_current_contents():
    m, n, ell = 1000, 800, 20
    a = _mat(m, n, 8, 11)
    om = torch.from_numpy(P.gaussian_matrix(n, ell, 5)).cuda()
    cfg = P.SketchConfig(ell=ell, q_power=1)
    for _ in range(3):
        P.corutv(a, cfg, omega=om)
    a.copy_(_mat(m, n, 12, 12))  # same pointer, new matrix
    f = P.corutv(a, cfg, omega=om)  # replay
    g = P.corutv(a.clone(), cfg, omega=om.clone())  # ordinary path
    assert torch.equal(f.t, g.t) and torch.equal(f.v, g.v)
    a[3, 4] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        P.corutv(a, cfg, omega=om)
