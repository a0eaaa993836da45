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


def test_c4_full_size_matches_oracle_histories():
    # BASELINE configs[3] (C4, n = 10000): the ALM run on the device against
    # the CPU oracle's recorded run on the same M (tests/golden/c4_oracle.json,
    # tools/c4_parity.py): same mu0, identical iteration count and
    # cap / rank / nnz histories, residual to rounding; the device spectral
    # norm against the oracle's
    import json
    from pathlib import Path

    ref = json.loads((Path(__file__).parent / "golden" / "c4_oracle.json").read_text())
    dev = torch.device("cuda", 0)
    n, k = 10000, 50
    g = torch.Generator(device=dev)
    g.manual_seed(777)
    x = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
    y = torch.randn((n, k), generator=g, dtype=torch.float64, device=dev) / 100.0
    mat = x @ y.T
    nnz = n * n // 20
    pos = torch.randperm(n * n, generator=g, device=dev)[:nnz]
    vals = (torch.rand((nnz,), generator=g, dtype=torch.float64, device=dev) * 1000.0) - 500.0
    mat.view(-1)[pos] += vals
    s, it = P.dense.spectral_norm_iters(mat)
    assert abs(s - ref["spectral_norm"]) <= 1e-12 * ref["spectral_norm"]
    assert abs(it - ref["spectral_norm_iters"]) <= 1
    cfg = P.AlmConfig(ell=2 * k, lam=1 / math.sqrt(n), tol=1e-7, q_power=1, seed=0,
                      mu0=1.25 / ref["spectral_norm"])
    sol = P.alm_corutv(mat, cfg)
    assert sol.iterations == ref["iterations"]
    assert sol.ell_history == ref["ell_history"]
    assert sol.rank_history == ref["rank_history"]
    assert sol.rank_of_l == ref["rank_of_l"] and sol.nnz_of_s == ref["nnz_of_s"]
    assert abs(sol.residuals[-1] - ref["final_residual"]) <= 1e-6 * ref["final_residual"]
    del mat, sol


def test_c3_full_size_matches_oracle():
    # BASELINE configs[2] at full size against the CPU oracle on the same A
    # and seeded Omega (tools/full_parity.py; ~30 s of 16-core oracle time and
    # ~36 GB of host memory)
    import numpy as np
    import psutil

    import oracle as O

    if psutil.virtual_memory().available < 80 * 2 ** 30:
        pytest.skip("needs ~36 GB of free host memory for the oracle copy of A")
    m, n, ell, q, k, noise, _ = bench.WORKLOADS["c3"]
    a = bench.gen_rows_device(torch, "c3", 0, m, torch.device("cuda", 0))
    f = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, seed=0))
    a_host = a.cpu().numpy()
    ref = O.corutv(a_host, ell, q, seed=0)
    del a_host
    d_dev = f.t.diagonal().abs().cpu().numpy()
    d_ref = np.abs(np.diag(ref["t"]))
    assert np.abs(d_dev[:k] - d_ref[:k]).max() <= 1e-12 * d_ref[0]
    assert np.array_equal(np.asarray(f.perm.cpu())[:k], ref["perm"][:k])
    u, v = f.u[:, :k].cpu().numpy(), f.v[:, :k].cpu().numpy()
    su = np.sign(np.sum(u * ref["u"][:, :k], axis=0))
    sv = np.sign(np.sum(v * ref["v"][:, :k], axis=0))
    assert np.abs(u * su - ref["u"][:, :k]).max() <= 1e-10
    assert np.abs(v * sv - ref["v"][:, :k]).max() <= 1e-10
    e_dev = P.corutv_lowrank_error(a, P.SketchConfig(ell=ell, q_power=q, seed=0))
    # |A - U T V'| of the oracle's factors from the exact-d identity
    # |A|^2 = |A - U T V'|^2 + |T|^2 (U T V' = P1 A P2)
    a2 = float(P.dense.frobenius_norm(a)) ** 2
    e_ref = math.sqrt(max(a2 - float((ref["t"] ** 2).sum()), 0.0))
    assert abs(e_dev - e_ref) <= 1e-8 * e_ref
    del a, f


def test_c5_full_size_matches_oracle():
    # BASELINE configs[4] (C5, orthonormal U512 / V512, sigma_i = 0.99^i,
    # 1e-6 noise) at full size against the CPU oracle's recorded run on the
    # same device-generated A and seeded Omega (tests/golden/c5_oracle.json,
    # tools/c5_oracle.py): |diag T| to 1e-9 of T00, the whole QRCP
    # permutation, the reconstruction error to 1e-10, the pass count
    import json
    from pathlib import Path

    import numpy as np

    ref = json.loads((Path(__file__).parent / "golden" / "c5_oracle.json").read_text())
    m, n, ell, q, k, noise, _ = bench.WORKLOADS["c5"]
    a = bench.gen_rows_device(torch, "c5", 0, m, torch.device("cuda", 0))
    assert abs(float((a * a).sum()) - ref["a_fro2"]) <= 1e-12 * ref["a_fro2"]  # same A
    cnt = P.PassCounter()
    f = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, seed=0), cnt)
    assert cnt.passes == ref["passes"]
    d_dev = f.t.diagonal().abs().cpu().numpy()
    d_ref = np.asarray(ref["diag_t_abs"])
    assert np.abs(d_dev - d_ref).max() <= 1e-9 * d_ref[0]
    assert np.asarray(f.perm.cpu()).tolist() == ref["perm"]
    e_dev = P.corutv_lowrank_error(a, P.SketchConfig(ell=ell, q_power=q, seed=0))
    assert abs(e_dev - ref["err"]) <= 1e-10 * ref["err"]
    u0 = f.u[::4096, 0].cpu().numpy()
    s = np.sign(np.dot(u0, ref["u_col0_sample"]))
    assert np.abs(s * u0 - np.asarray(ref["u_col0_sample"])).max() <= 1e-9
    del a, f
