"""The row-sharded device path with two real ranks on the one
GPU of the test box: each rank runs the sm_100a decomposition on its block
of rows and the library's allreduce callback goes through
torch.distributed (gloo, on CUDA tensors; NCCL is the production backend).
No kernel waits on another rank -- the exchange points are host-side
collectives between ordinary launches -- so two processes may share the
device.  The factors must match the single-process run on the full matrix
(T, V replicated on both ranks, U row-stacked)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

M, N, ELL, Q = 3000, 700, 24, 1


def _matrix():
    rng = np.random.Generator(np.random.PCG64(77))
    return rng.standard_normal((M, 15)) @ rng.standard_normal((15, N)) + 1e-3 * rng.standard_normal((M, N))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, outdir, variant):
    import torch.distributed as tdist

    import paper_1906_04572_b200 as P
    from paper_1906_04572_b200.dist import RowShardComm, corutv_sharded, row_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = _matrix()
        lo, hi = row_range(M, world, rank)
        a_loc = torch.from_numpy(np.ascontiguousarray(a[lo:hi])).cuda()
        comm = RowShardComm(device="cuda")
        cnt = P.PassCounter()
        f = corutv_sharded(a_loc, P.SketchConfig(ell=ELL, q_power=Q, seed=3, variant=variant), comm, cnt)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), u=f.u.cpu().numpy(), t=f.t.cpu().numpy(),
                 v=f.v.cpu().numpy(), perm=f.perm.cpu().numpy(), passes=cnt.passes, calls=comm.calls)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("variant", ["exact-d", "approx-d"])
def test_two_ranks_on_device_match_single_process(tmp_path, variant):
    import torch.multiprocessing as tmp

    import paper_1906_04572_b200 as P

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    tmp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path), variant), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    torch.cuda.set_device(0)
    ref = P.corutv(torch.from_numpy(_matrix()).cuda(), P.SketchConfig(ell=ELL, q_power=Q, seed=3, variant=variant))
    t_ref, v_ref, u_ref = ref.t.cpu().numpy(), ref.v.cpu().numpy(), ref.u.cpu().numpy()
    # replicated factors are bit-identical across ranks
    assert np.array_equal(parts[0]["t"], parts[1]["t"]) and np.array_equal(parts[0]["v"], parts[1]["v"])
    assert all(int(p["calls"]) > 0 for p in parts)
    assert int(parts[0]["passes"]) == 2 * (Q + 1) + (1 if variant == "exact-d" else 0)
    # against the single-process run (different reduction order only)
    k = 15
    assert np.array_equal(parts[0]["perm"][:k], ref.perm.cpu().numpy()[:k])
    s0 = abs(t_ref[0, 0])
    assert np.abs(np.abs(np.diag(parts[0]["t"]))[:k] - np.abs(np.diag(t_ref))[:k]).max() <= 1e-10 * s0
    u = np.vstack([p["u"] for p in parts])
    sg = np.sign(np.sum(u[:, :k] * u_ref[:, :k], axis=0))
    assert np.abs(u[:, :k] * sg - u_ref[:, :k]).max() <= 1e-9
    sv = np.sign(np.sum(parts[0]["v"][:, :k] * v_ref[:, :k], axis=0))
    assert np.abs(parts[0]["v"][:, :k] * sv - v_ref[:, :k]).max() <= 1e-9


NA = 300


def _rpca_matrix():
    rng = np.random.Generator(np.random.PCG64(12))
    k = 15
    m = rng.standard_normal((NA, k)) @ rng.standard_normal((k, NA)) / NA
    pos = rng.choice(NA * NA, size=NA * NA // 20, replace=False)
    m.flat[pos] += rng.uniform(-5.0, 5.0, size=pos.size)
    return m


def _alm_rank_main(rank, world, port, outdir):
    import torch.distributed as tdist

    import paper_1906_04572_b200 as P
    from paper_1906_04572_b200.dist import RowShardComm, alm_corutv_sharded, row_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _rpca_matrix()
        lo, hi = row_range(NA, world, rank)
        m_loc = torch.from_numpy(np.ascontiguousarray(m[lo:hi])).cuda()
        comm = RowShardComm(device="cuda")
        sol = alm_corutv_sharded(m_loc, P.AlmConfig(ell=30, q_power=1, seed=2, tol=1e-7), comm, NA)
        np.savez(os.path.join(outdir, f"alm{rank}.npz"), l=sol.l.cpu().numpy(), s=sol.s.cpu().numpy(),
                 it=sol.iterations, ranks=np.array(sol.rank_history), caps=np.array(sol.ell_history),
                 nnz=np.array(sol.nnz_history), res=np.array(sol.residuals), rank_of_l=sol.rank_of_l,
                 calls=comm.calls)
    finally:
        tdist.destroy_process_group()


def test_two_rank_alm_matches_single_process(tmp_path):
    # BASELINE configs[3] "on 1 and 8 GPUs": the row-sharded ALM solver takes
    # the same decisions as the single-process one
    import torch.multiprocessing as tmp

    import paper_1906_04572_b200 as P
    from paper_1906_04572_b200.dist import row_range

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    tmp.spawn(_alm_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"alm{r}.npz") for r in range(world)]
    torch.cuda.set_device(0)
    m = _rpca_matrix()
    ref = P.alm_corutv(torch.from_numpy(m).cuda(), P.AlmConfig(ell=30, q_power=1, seed=2, tol=1e-7))
    for p in parts:
        assert int(p["calls"]) > 0
        assert int(p["it"]) == ref.iterations
        assert list(p["ranks"]) == ref.rank_history and list(p["caps"]) == ref.ell_history
        assert list(p["nnz"]) == ref.nnz_history and int(p["rank_of_l"]) == ref.rank_of_l
        assert np.allclose(p["res"], ref.residuals, rtol=1e-6, atol=0)
    l_ref, s_ref = ref.l.cpu().numpy(), ref.s.cpu().numpy()
    scale = np.abs(m).max()
    for r, p in enumerate(parts):
        lo, hi = row_range(NA, world, r)
        assert np.abs(p["l"] - l_ref[lo:hi]).max() <= 1e-8 * scale
        assert np.abs(p["s"] - s_ref[lo:hi]).max() <= 1e-8 * scale
