"""The device QRCP kernels (one CTA, thread-block cluster, cooperative grid)
against the reference's own QRCP known-answer tests (pkg/tests/
test_dense.py:97-127, golden vectors made by the reference itself) and
against the oracle (dense.py:152-192) on exact-tie inputs and on cores past
the old 640 limit, through the C-ABI (corutv_qrcp_mn).

Bars: the permutation is compared EXACTLY (it is integer output; the
pivot rule -- max downdated norm, lowest current index on ties -- must be
reproduced, not approximated); |diag R| to 1e-14 of |R_00|; Q R = A[:, perm]
and Q'Q = I to 1e-12."""

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


def dev_qrcp(a):
    f = P.dense.qrcp(torch.from_numpy(np.ascontiguousarray(a)).cuda())
    return f.q.cpu().numpy(), f.r.cpu().numpy(), f.perm.cpu().numpy()


def check_invariants(a, q, r, perm, tol=1e-12):
    m, n = a.shape
    k = min(m, n)
    assert q.shape == (m, k) and r.shape == (k, n)
    assert sorted(perm.tolist()) == list(range(n))
    assert np.abs(q.T @ q - np.eye(k)).max() < tol
    assert np.linalg.norm(q @ r - a[:, perm]) <= tol * max(np.linalg.norm(a), 1e-300)
    assert np.abs(np.tril(r, -1)).max() == 0.0
    d = np.abs(np.diag(r))
    assert np.all(d[:-1] >= d[1:] * (1 - 1e-12))


@pytest.mark.parametrize("name", ["qrcp_diag", "qrcp_tie", "qrcp_rand", "qrcp_square"])
def test_device_qrcp_matches_reference_golden(golden, name):
    """test_dense.py:97-127 cases, golden from the reference itself:
    exact permutation, |diag R| to 1e-14 |R00|."""
    g = golden[name]
    q, r, perm = dev_qrcp(g["a"])
    assert perm.tolist() == g["perm"].tolist()
    d, dg = np.abs(np.diag(r)), np.abs(np.diag(g["r"]))
    assert np.abs(d - dg).max() <= 1e-14 * dg[0]
    check_invariants(g["a"], q, r, perm)


def test_device_qrcp_kat_diag_sorts():
    """test_dense.py:97-100: diag(1, 3, 2) -> perm [1, 2, 0], |diag R| 3, 2, 1."""
    q, r, perm = dev_qrcp(np.diag([1.0, 3.0, 2.0]))
    assert perm.tolist() == [1, 2, 0]
    assert np.abs(np.abs(np.diag(r)) - [3.0, 2.0, 1.0]).max() < 1e-14


def test_device_qrcp_kat_tie_lowest_index():
    """test_dense.py:103-107: columns 0 and 2 tie; the pivot is column 0."""
    q, r, perm = dev_qrcp(np.array([[2.0, 1.0, 2.0], [0.0, 0.5, 0.0]]))
    assert perm[0] == 0


def test_device_qrcp_kat_rank_reveal(golden):
    """test_dense.py:110-115 (the reference's rank-5 30 x 30 case): the
    leading five pivots are the reference's, and d[5] / d[0] < 1e-10.  Pivots
    past the numerical rank choose among residual norms at rounding level and
    are not part of the reference's assertion."""
    g = golden["qrcp_rank5"]
    q, r, perm = dev_qrcp(g["a"])
    assert perm[:5].tolist() == g["perm"][:5].tolist()
    d = np.abs(np.diag(r))
    assert d[5] / d[0] < 1e-10
    check_invariants(g["a"], q, r, perm)


def _tie_matrix(n, m=None, seed=0):
    """Diagonal-block matrix with many exact column-norm ties at every step
    (orthogonal columns keep the norms exact, so each pivot is decided by
    the lowest-current-index rule alone)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    m = n if m is None else m
    vals = rng.choice([1.0, 2.0, 3.0, 0.5], size=min(m, n))
    a = np.zeros((m, n))
    rows = rng.permutation(m)[:min(m, n)]
    cols = rng.permutation(n)[:min(m, n)]
    a[rows, cols] = vals
    return a


@pytest.mark.parametrize("shape", [(5, 5), (40, 40), (200, 200), (641, 641), (900, 900), (300, 700),
                                   (700, 300)])
def test_device_qrcp_tie_break_matches_oracle(shape):
    """One CTA (n <= 128), cluster (129..640) and grid (> 640, rectangular)
    kernels all reproduce the reference's physical-swap tie-break."""
    m, n = shape
    a = _tie_matrix(n, m, seed=m + n)
    q, r, perm = dev_qrcp(a)
    oq, orr, operm = O.qrcp(a)
    assert perm.tolist() == operm.tolist()
    assert np.abs(np.abs(np.diag(r)) - np.abs(np.diag(orr))).max() == 0.0
    check_invariants(a, q, r, perm)


@pytest.mark.parametrize("shape", [(1000, 1000), (700, 700), (1200, 800), (500, 900), (1, 7), (9, 1)])
def test_device_qrcp_grid_matches_oracle(shape):
    """Cores past the old 640 cap and rectangular inputs (grid kernel): a
    Gaussian matrix has well-separated pivot norms, so the whole permutation
    must agree."""
    m, n = shape
    rng = np.random.Generator(np.random.PCG64(m * 3 + n))
    a = rng.standard_normal((m, n))
    q, r, perm = dev_qrcp(a)
    oq, orr, operm = O.qrcp(a)
    assert perm.tolist() == operm.tolist()
    d, od = np.abs(np.diag(r)), np.abs(np.diag(orr))
    assert np.abs(d - od).max() <= 1e-12 * od[0]
    check_invariants(a, q, r, perm)


def test_device_qrcp_zero_columns():
    """Zero columns give no reflector (dense.py:109-110): R_jj = 0."""
    a = np.zeros((700, 700))
    a[:, 3] = 1.0
    a[:, 600] = 2.0
    q, r, perm = dev_qrcp(a)
    oq, orr, operm = O.qrcp(a)
    assert perm.tolist() == operm.tolist()
    assert np.abs(np.abs(np.diag(r)) - np.abs(np.diag(orr))).max() == 0.0
    assert np.linalg.norm(q @ r - a[:, perm]) <= 1e-12 * np.linalg.norm(a)
