"""Row-sharded (N > 1) path on CPU with gloo, world_size 2.

The GPU box has one device, so the multi-rank logic is covered here:
row partitioning, the allreduce callback the native library calls (driven
through ctypes exactly as the library does, on host buffers), and the
sharded algorithm itself — a numpy mirror of the device schedule
(corutv_b200.cu: C2 / Gram / D all-reduces, adaptive CholeskyQR, redundant
Q2 + QRCP) — must reproduce the single-process oracle."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as tdist
import torch.multiprocessing as tmp

import oracle as O
from paper_1906_04572_b200.dist import RowShardComm, row_range

U = np.finfo(float).eps / 2


@pytest.mark.parametrize("m,world", [(10, 3), (131072, 8), (7, 8), (1000, 1), (4000, 2)])
def test_row_range_partitions(m, world):
    spans = [row_range(m, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == m
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cholqr_sharded(x_loc, m_glob, allreduce):
    """numpy mirror of cholqr() in corutv_b200.cu for a row-sharded X."""
    ell = x_loc.shape[1]
    coeff = 11.0 * (m_glob * ell + ell * (ell + 1)) * U
    plain = 0
    for _ in range(12):
        g = allreduce(x_loc.T @ x_loc)
        tr = np.trace(g)
        r = None
        try:
            r = np.linalg.cholesky(g).T
            ri = np.linalg.inv(r)
            kappa = np.linalg.norm(r) * np.linalg.norm(ri)
            shifted = not kappa <= 1e6
        except np.linalg.LinAlgError:
            shifted = True
        if shifted:
            r = np.linalg.cholesky(g + coeff * tr * np.eye(ell)).T
            ri = np.linalg.inv(r)
        x_loc = x_loc @ ri
        plain = 0 if shifted else plain + 1
        if plain == 2:
            return x_loc
    raise AssertionError("no convergence")


def _sharded_corutv(a_loc, m_glob, ell, q, omega, allreduce):
    x = omega
    for _ in range(q + 1):
        c1 = a_loc @ x
        x = allreduce(a_loc.T @ c1)
    q1 = _cholqr_sharded(c1, m_glob, allreduce)
    q2 = _cholqr_sharded(x, x.shape[0], lambda g: g)  # replicated
    d = allreduce(q1.T @ (a_loc @ q2))
    qd, rd, perm = O.qrcp(d)
    return q1 @ qd, rd, q2[:, perm], perm


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = RowShardComm(device="cpu")
        # 1) the exact callback the native library invokes
        buf = (ctypes.c_double * 4)(*[rank + 1.0 + i for i in range(4)])
        rc = comm.callback(None, ctypes.addressof(buf), 4, None)
        got_cb = list(buf)
        # 2) sharded algorithm mirror vs single-process oracle
        rng = np.random.Generator(np.random.PCG64(7))
        m, n, ell, q = 400, 120, 16, 1
        a = rng.standard_normal((m, 10)) @ rng.standard_normal((10, n)) + 1e-1 * rng.standard_normal((m, n))
        omega = O.gaussian_matrix(n, ell, 3)
        lo, hi = row_range(m, world, rank)

        def allreduce(x):
            import torch

            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).copy())
            tdist.all_reduce(t)
            return t.numpy()

        u_loc, t, v, perm = _sharded_corutv(a[lo:hi], m, ell, q, omega, allreduce)
        results[rank] = dict(rc=rc, cb=got_cb, u=u_loc, t=t, v=v, perm=perm, lo=lo, hi=hi,
                             calls=comm.calls)
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_sharded_path():
    world = 2
    port = _free_port()
    mgr = tmp.Manager()
    results = mgr.dict()
    tmp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    r0, r1 = results[0], results[1]
    # callback: in-place sum across ranks
    assert r0["rc"] == 0 and r1["rc"] == 0
    assert r0["cb"] == r1["cb"] == [3.0, 5.0, 7.0, 9.0]
    assert r0["calls"] == 1
    # replicated outputs identical on both ranks
    assert np.array_equal(r0["t"], r1["t"]) and np.array_equal(r0["v"], r1["v"])
    assert np.array_equal(r0["perm"], r1["perm"])
    # vs single-process oracle on the full matrix
    rng = np.random.Generator(np.random.PCG64(7))
    m, n, ell, q = 400, 120, 16, 1
    a = rng.standard_normal((m, 10)) @ rng.standard_normal((10, n)) + 1e-1 * rng.standard_normal((m, n))
    ref = O.corutv(a, ell, q, omega=O.gaussian_matrix(n, ell, 3))
    u = np.vstack([r0["u"], r1["u"]])
    f = dict(u=u, t=r0["t"], v=r0["v"])
    e_sh = O.corutv_lowrank_error(a, f)
    e_ref = O.corutv_lowrank_error(a, ref)
    assert abs(e_sh - e_ref) <= 1e-10 * e_ref
    assert np.abs(np.abs(np.diag(f["t"])) - np.abs(np.diag(ref["t"]))).max() <= 1e-9 * abs(ref["t"][0, 0])
    assert np.array_equal(r0["perm"][:10], ref["perm"][:10])
    assert np.abs(u.T @ u - np.eye(ell)).max() < 1e-12
