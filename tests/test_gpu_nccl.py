"""The native NCCL data plane of the row-sharded mode (SURVEY §8e,
corutv_nccl_comm_create / corutv_set_nccl): every exchange is an
ncclAllReduce the library enqueues on its own stream.  The test box has one
GPU, and NCCL refuses two ranks on one device, so the NCCL path is driven
as a one-rank communicator: the library then runs the full sharded code
path (Gram / sketch / core all-reduces through NCCL, the replicated QR,
the sharded spectral norm and ALM) and must reproduce the single-GPU
results.  Multi-rank correctness of the same exchange points is covered by
the 2-rank gloo tests (test_gpu_dist.py, test_dist_cpu.py)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1906_04572_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def nccl_comm():
    import torch.distributed as tdist

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    tdist.init_process_group("gloo", rank=0, world_size=1)
    from paper_1906_04572_b200.dist import RowShardComm

    comm = RowShardComm(device="cuda", native=True)
    yield comm
    comm.close()
    tdist.destroy_process_group()


def test_nccl_comm_is_native(nccl_comm):
    assert nccl_comm.native and nccl_comm.nccl
    assert nccl_comm.calls == 0  # no Python callback is ever used


@pytest.mark.parametrize("variant", ["exact-d", "approx-d"])
def test_sharded_corutv_over_nccl_matches_single(nccl_comm, variant):
    from paper_1906_04572_b200.dist import corutv_sharded

    rng = np.random.Generator(np.random.PCG64(5))
    a = rng.standard_normal((3000, 20)) @ rng.standard_normal((20, 700)) + 1e-3 * rng.standard_normal((3000, 700))
    A = torch.from_numpy(a).cuda()
    cfg = P.SketchConfig(ell=40, q_power=1, seed=3, variant=variant)
    cnt = P.PassCounter()
    f = corutv_sharded(A, cfg, nccl_comm, cnt)
    g = P.corutv(A, cfg)
    assert nccl_comm.calls == 0
    assert cnt.passes == (5 if variant == "exact-d" else 4)
    d, dg = f.t.diagonal().abs().cpu().numpy(), g.t.diagonal().abs().cpu().numpy()
    assert np.abs(d[:20] - dg[:20]).max() <= 1e-12 * dg[0]
    assert np.array_equal(f.perm.cpu().numpy()[:20], g.perm.cpu().numpy()[:20])
    ef = np.linalg.norm(a - f.u.cpu().numpy() @ (f.t.cpu().numpy() @ f.v.cpu().numpy().T))
    eg = np.linalg.norm(a - g.u.cpu().numpy() @ (g.t.cpu().numpy() @ g.v.cpu().numpy().T))
    assert abs(ef - eg) <= 1e-10 * np.linalg.norm(a)


def test_sharded_spectral_norm_over_nccl_matches_single(nccl_comm):
    from paper_1906_04572_b200 import _lib

    rng = np.random.Generator(np.random.PCG64(6))
    A = torch.from_numpy(rng.standard_normal((2000, 900))).cuda()
    ref, rit = P.dense.spectral_norm_iters(A)
    h = _lib.handle(0)
    nccl_comm.attach(h, 2000)
    try:
        val, it = P.dense.spectral_norm_iters(A)
    finally:
        nccl_comm.detach(h)
    assert abs(val - ref) <= 1e-13 * ref
    assert abs(it - rit) <= 1


def test_sharded_alm_over_nccl_matches_single(nccl_comm):
    import oracle as O
    from paper_1906_04572_b200.dist import alm_corutv_sharded

    m, _, _ = O.gen_rpca_instance(400, 10, 4000, seed=11)
    M = torch.from_numpy(m).cuda()
    cfg = P.AlmConfig(ell=20, q_power=1, seed=2)
    sol = alm_corutv_sharded(M, cfg, nccl_comm, 400)
    ref = P.alm_corutv(M, cfg)
    assert sol.iterations == ref.iterations
    assert sol.rank_history == ref.rank_history and sol.ell_history == ref.ell_history
    assert np.linalg.norm((sol.l - ref.l).cpu().numpy()) <= 1e-8 * np.linalg.norm(ref.l.cpu().numpy())
