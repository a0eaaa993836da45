"""Row-sharded (multi-GPU) CoR-UTV — SURVEY §8e.

One process per GPU; rank g owns a contiguous block of rows A_g.  The
native library does all the math; at the exchange points of the algorithm
it runs a sum-allreduce on the handle's stream -- ncclAllReduce on its own
communicator (``RowShardComm(native=True)``), or a callback into this
module (the gloo test path):

  * C2 = sum_g A_g' C1_g                 (n x ell, per power iteration)
  * Gram X'X of the row-sharded Q1 sketch (ell x ell, per CholeskyQR step)
  * D  = sum_g Q1_g' (A_g Q2)            (ell x ell)
  * the global row count, the non-finite flag, ALM (zeta^2, nnz) scalars

Everything replicated (Q2, the QRCP of D, V) is computed redundantly and
bit-identically on every rank from the all-reduced inputs.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as dev
from . import _lib
from .sketch import _VARIANT_CODE, CorUtvFactors, PassCounter, SketchConfig, pcg_state

__all__ = ["row_range", "RowShardComm", "corutv_sharded", "alm_corutv_sharded"]


def row_range(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of rows owned by ``rank``: the first m % world ranks
    get one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class _CudaBuffer:
    """Zero-copy view of a raw device pointer for torch.as_tensor."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3,
            "strides": None,
        }


class RowShardComm:
    """The row-sharded data plane over a torch.distributed process group.

    ``native=True`` (the production path on GPUs): the library gets its own
    NCCL communicator (rank 0 creates the id, the group broadcasts it, every
    rank joins) and enqueues every exchange as ncclAllReduce on its stream
    -- no Python runs per collective.  ``native=False``: a sum-allreduce
    callback into ``torch.distributed.all_reduce`` (the gloo test path);
    ``device``: "cuda" (pointers are device memory) or "cpu" (host
    pointers; used by the CPU tests of the marshalling)."""

    def __init__(self, group=None, device: str = "cuda", native: bool = False):
        import torch.distributed as tdist

        self.group = group
        self.rank = tdist.get_rank(group)
        self.world = tdist.get_world_size(group)
        self.device = device
        self.calls = 0
        self.callback = _lib.ALLREDUCE_FN(self._allreduce)
        self.native = native
        self.nccl = None
        if native:
            self._init_nccl()

    def _init_nccl(self):
        import torch
        import torch.distributed as tdist

        lib = _lib.load_library()
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            _lib.check(lib.corutv_nccl_unique_id(uid), None, "corutv_nccl_unique_id")
        box = [bytes(uid)]
        tdist.broadcast_object_list(box, src=tdist.get_global_rank(self.group, 0) if self.group else 0,
                                    group=self.group)
        uid = (ctypes.c_ubyte * 128).from_buffer_copy(box[0])
        comm = ctypes.c_void_p()
        _lib.check(lib.corutv_nccl_comm_create(torch.cuda.current_device(), uid, self.rank, self.world,
                                               ctypes.byref(comm)), None, "corutv_nccl_comm_create")
        self.nccl = comm

    def close(self):
        if self.nccl:
            _lib.load_library().corutv_nccl_comm_destroy(self.nccl)
            self.nccl = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _tensor(self, ptr: int, count: int):
        import torch

        if self.device == "cpu":
            arr = np.ctypeslib.as_array((ctypes.c_double * count).from_address(ptr))
            return torch.from_numpy(arr)
        return torch.as_tensor(_CudaBuffer(ptr, count), device="cuda")

    def _allreduce(self, user, buf, count, stream):  # noqa: ARG002
        import torch.distributed as tdist

        try:
            t = self._tensor(int(buf), int(count))
            tdist.all_reduce(t, op=tdist.ReduceOp.SUM, group=self.group)
            self.calls += 1
            return 0
        except Exception:  # pragma: no cover - surfaced as CORUTV_ERR_COMM
            return 1

    def global_rows(self, m_local: int) -> int:
        """Sum of the ranks' row counts (one host collective per sharded
        call; the library then needs no row-count exchange of its own)."""
        import torch
        import torch.distributed as tdist

        dev_ = "cuda" if self.device == "cuda" else "cpu"
        t = torch.tensor([float(m_local)], dtype=torch.float64, device=dev_)
        tdist.all_reduce(t, op=tdist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def attach(self, handle: "_lib.Handle", global_rows: int | None = None) -> None:
        if self.native:
            _lib.check(handle.lib.corutv_set_nccl(handle.ptr, self.nccl, self.rank, self.world), handle.ptr,
                       "corutv_set_nccl")
        else:
            _lib.check(handle.lib.corutv_set_comm(handle.ptr, self.callback, None, self.rank, self.world),
                       handle.ptr, "corutv_set_comm")
        if global_rows is not None:
            _lib.check(handle.lib.corutv_set_global_rows(handle.ptr, int(global_rows)), handle.ptr,
                       "corutv_set_global_rows")

    def detach(self, handle: "_lib.Handle") -> None:
        if self.native:
            handle.lib.corutv_set_nccl(handle.ptr, None, 0, 1)
        else:
            handle.lib.corutv_set_comm(handle.ptr, _lib.ALLREDUCE_FN(), None, 0, 1)


def corutv_sharded(a_local, cfg: SketchConfig, comm: RowShardComm, counter: PassCounter | None = None,
                   omega=None) -> CorUtvFactors:
    """CoR-UTV of the row-sharded global matrix whose rows
    ``row_range(m, world, rank)`` are ``a_local`` on this rank.  Returns the
    local rows of U plus the replicated T and V."""
    torch = dev.torch_mod()
    A, was_host = dev.to_device(a_local, "a")
    m_loc, n = A.shape
    ell = cfg.ell
    om = None
    if omega is not None:
        om = (omega if dev.is_device_tensor(omega) else torch.from_numpy(np.ascontiguousarray(omega)))
        om = om.to(A.device, torch.float64).contiguous()
    u = torch.empty((m_loc, ell), dtype=torch.float64, device=A.device)
    t = torch.empty((ell, ell), dtype=torch.float64, device=A.device)
    v = torch.empty((n, ell), dtype=torch.float64, device=A.device)
    perm = torch.empty((ell,), dtype=torch.int64, device=A.device)
    passes = ctypes.c_int64(0)
    h = _lib.handle(A.device.index)
    comm.attach(h, comm.global_rows(m_loc))
    try:
        if om is None:  # every rank draws the identical Omega on its device
            h.call("corutv_decompose_seeded", dev.ptr(A), m_loc, n, A.stride(0), ell, cfg.q_power,
                   _VARIANT_CODE[cfg.variant], pcg_state(cfg.seed), dev.ptr(u), dev.ptr(t),
                   dev.ptr(v), dev.ptr(perm), ctypes.byref(passes))
        else:
            h.call("corutv_decompose", dev.ptr(A), m_loc, n, A.stride(0), ell, cfg.q_power,
                   _VARIANT_CODE[cfg.variant], dev.ptr(om), dev.ptr(u), dev.ptr(t), dev.ptr(v),
                   dev.ptr(perm), ctypes.byref(passes))
    finally:
        comm.detach(h)
    if counter is not None:
        counter.add(passes.value)
    return CorUtvFactors(u=dev.to_output(u, was_host), t=dev.to_output(t, was_host),
                         v=dev.to_output(v, was_host), ell=ell, q_power=cfg.q_power,
                         variant=cfg.variant, perm=dev.to_output(perm, was_host))


def alm_corutv_sharded(m_local, cfg, comm: RowShardComm, global_rows: int):
    """alm_corutv (rpca.py:237-255) of the row-sharded global M whose rows
    ``row_range(global_rows, world, rank)`` are ``m_local`` on this rank
    (BASELINE configs[3] "on 1 and 8 GPUs").  Every exchange is inside the
    library: |M|_F and the spectral norm (mu0), the sketch products and
    Grams of each CoR-UTV, and the residual / support counts of the fused
    update are all-reduced, so the scalar decisions (rank, cap, mu, stop)
    are identical on all ranks.  Returns this rank's rows of L and S and the
    replicated histories."""
    from . import rpca

    if cfg.ell is None:
        raise ValueError("alm_corutv requires cfg.ell (sketch sample size)")
    torch = dev.torch_mod()
    device = m_local.device.index if dev.is_device_tensor(m_local) else torch.cuda.current_device()
    h = _lib.handle(device)
    comm.attach(h, global_rows)
    try:
        def step(g, delta, cap, j, state):
            scfg = SketchConfig(ell=cap, q_power=cfg.q_power, seed=(cfg.seed + j) % 2 ** 64)
            f, rank = rpca.corutv_truncated(g, scfg, delta)

            def sigma_of():
                sig = rpca.singular_values(f.t[:rank, :])
                return sig.cpu().numpy() if dev.is_device_tensor(sig) else sig

            return f.u, f.t, f.v, f.ell, rank, sigma_of, None

        return rpca._alm_loop(m_local, cfg, step, cap0=cfg.ell, global_rows=global_rows)
    finally:
        comm.detach(h)
