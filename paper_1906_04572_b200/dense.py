"""Dense kernels used on the hot path, device-backed — the subset of
/root/reference/pkg/src/corutv/dense.py that CoR-UTV and ALM-CoRUTV call.

* :func:`spectral_norm` — dense.py:405-442 (mu0 of the ALM solver)
* :func:`singular_values` — dense.py:379-387 (rank readout of L)
* :func:`frobenius_norm` — dense.py:94-96
* :func:`jacobi_svd` — dense.py:313-376 (sor_svd / tsr_svd cores, the
  InexactALM baseline's warm-started SVT)
* :func:`qrcp` — dense.py:152-192 (the QRCP of the compressed core, and the
  harness's deterministic full-matrix method)
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

from . import _device as dev
from . import _lib

__all__ = ["spectral_norm", "singular_values", "frobenius_norm", "spectral_norm_iters", "SvdFactors",
           "QrcpFactors", "qrcp", "jacobi_svd", "JACOBI_TOL", "JACOBI_MAX_SWEEPS"]

JACOBI_TOL = 1e-14        # dense.py:34
JACOBI_MAX_SWEEPS = 100   # dense.py:36


@dataclass
class SvdFactors:
    """dense.py:71-78: economy SVD factors, ``u * sigma @ v.T`` reconstructs
    the input; sigma non-negative and non-increasing."""

    u: object
    sigma: object
    v: object


def spectral_norm_iters(a, tol: float = 1e-10, max_iter: int = 5000):
    """(|A|_2, power iterations) — dense.py:405-442 schedule on the device:
    block size min(24, n), disjoint-support start, stop when
    |est - prev| <= 0.02 tol est; Jacobi path for min(m, n) <= 64."""
    A, _ = dev.to_device(a, "a")
    out = ctypes.c_double(0.0)
    it = ctypes.c_int(0)
    h = _lib.handle(A.device.index)
    try:
        h.call("corutv_spectral_norm", dev.ptr(A), A.shape[0], A.shape[1], A.stride(0), tol,
               max_iter, ctypes.byref(out), ctypes.byref(it))
    except ValueError:
        dev.raise_if_nonfinite(A, "a")
        raise
    if not math.isfinite(out.value):
        dev.raise_if_nonfinite(A, "a")
    return float(out.value), int(it.value)


def spectral_norm(a, tol: float = 1e-10, max_iter: int = 5000) -> float:
    """Largest singular value (dense.py:405-442)."""
    return spectral_norm_iters(a, tol, max_iter)[0]


def singular_values(a):
    """Singular values, descending (dense.py:379-387), one-sided Jacobi on
    the device (one CTA, or the cooperative grid above ~116 columns;
    min(m, n) <= 16384)."""
    torch = dev.torch_mod()
    A, was_host = dev.to_device(a, "a")
    dev.raise_if_nonfinite(A, "a")
    k = min(A.shape)
    sig = torch.empty((k,), dtype=torch.float64, device=A.device)
    h = _lib.handle(A.device.index)
    h.call("corutv_singular_values", dev.ptr(A), A.shape[0], A.shape[1], A.stride(0), dev.ptr(sig))
    return dev.to_output(sig, was_host)


def frobenius_norm(a) -> float:
    """dense.py:94-96 with a deterministic two-stage device reduction."""
    A, _ = dev.to_device(a, "a")
    out = ctypes.c_double(0.0)
    h = _lib.handle(A.device.index)
    try:
        h.call("corutv_sumsq", dev.ptr(A), A.shape[0], A.shape[1], A.stride(0), ctypes.byref(out))
    except ValueError:
        raise ValueError("a contains non-finite entries") from None
    return math.sqrt(out.value)


def _check_v_init(v_init, k: int):
    """dense.py:316-318: v_init must be the k x k right factor of the tall
    orientation."""
    V, _ = dev.to_device(v_init, "v_init")
    dev.raise_if_nonfinite(V, "v_init")
    if tuple(V.shape) != (k, k):
        raise ValueError(f"v_init must be {k}x{k}, got {tuple(V.shape)}")
    return V


@dataclass
class QrcpFactors:
    """dense.py:62-69: ``q @ r == a[:, perm]`` with ``|diag(r)|``
    non-increasing."""

    q: object
    r: object
    perm: object


def qrcp(a) -> QrcpFactors:
    """dense.py:152-192 on the device (corutv_qrcp_mn): Businger-Golub
    column pivoting on downdated norms with exact refresh, ties to the lowest
    column index; q is m x k, r is k x n, k = min(m, n)."""
    torch = dev.torch_mod()
    A, was_host = dev.to_device(a, "a")
    dev.raise_if_nonfinite(A, "a")
    m, n = A.shape
    k = min(m, n)
    q = torch.empty((m, k), dtype=torch.float64, device=A.device)
    r = torch.empty((k, n), dtype=torch.float64, device=A.device)
    perm = torch.empty((n,), dtype=torch.int64, device=A.device)
    h = _lib.handle(A.device.index)
    h.call("corutv_qrcp_mn", dev.ptr(A), m, n, A.stride(0), dev.ptr(q), k, dev.ptr(r), n, dev.ptr(perm))
    return QrcpFactors(q=dev.to_output(q, was_host), r=dev.to_output(r, was_host),
                       perm=dev.to_output(perm, was_host))


def jacobi_svd(a, tol: float = JACOBI_TOL, max_sweeps: int = JACOBI_MAX_SWEEPS,
               v_init=None) -> SvdFactors:
    """dense.py:357-376 on the device: economy SVD by one-sided Jacobi
    (min(m, n) <= 16384; one CTA when the core fits shared memory, else a
    cooperative grid, jacobi_grid.cuh).  ``v_init`` warm-starts the sweeps
    from the tall orientation's right factor (corutv_jacobi_svd_warm);
    exceeding ``max_sweeps`` raises :class:`ConvergenceError`."""
    torch = dev.torch_mod()
    A, was_host = dev.to_device(a, "a")
    dev.raise_if_nonfinite(A, "a")
    m, n = A.shape
    k = min(m, n)
    V0 = _check_v_init(v_init, k).contiguous() if v_init is not None else None
    u = torch.empty((m, k), dtype=torch.float64, device=A.device)
    s = torch.empty((k,), dtype=torch.float64, device=A.device)
    v = torch.empty((n, k), dtype=torch.float64, device=A.device)
    h = _lib.handle(A.device.index)
    h.call("corutv_jacobi_svd_warm", dev.ptr(A), m, n, A.stride(0), dev.ptr(V0) if V0 is not None else None,
           V0.stride(0) if V0 is not None else 0, float(tol), int(max_sweeps), dev.ptr(u), dev.ptr(s),
           dev.ptr(v))
    return SvdFactors(u=dev.to_output(u, was_host), sigma=dev.to_output(s, was_host), v=dev.to_output(v, was_host))
