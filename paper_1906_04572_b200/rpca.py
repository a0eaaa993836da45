"""ALM-CoRUTV robust PCA on the B200 — drop-in for ``corutv.rpca``.

Mirrors /root/reference/pkg/src/corutv/rpca.py: the same AlmConfig /
RpcaSolution types, the same iteration (rpca.py:175-234) and the same
history bookkeeping.  Per iteration the device does

  * CoR-UTV of G_j = M - S_j + Y_j / mu_j            (corutv_decompose)
  * one fused pass: L = U_r (T_r V') tile-by-tile, shrink, residual, dual
    update and G_{j+1}, with the residual norm and support count reduced
    deterministically on the device                  (corutv_alm_update)

and the host takes the same scalar decisions as the reference (rank count,
next cap, stop test, mu update) from a handful of bytes read back.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _device as dev
from . import _lib
from .dense import singular_values, spectral_norm
from .errors import ConvergenceError
from .sketch import SketchConfig, corutv, corutv_truncated  # noqa: F401  (rpca.corutv, as in the reference module)

__all__ = [
    "AlmConfig",
    "RpcaSolution",
    "shrink",
    "corutv_threshold",
    "alm_corutv",
    "inexact_alm",
    "svt",
    "write_telemetry_csv",
]

NNZ_EPS = 1e-12    # rpca.py:44 (hard-wired in the fused kernel)
RANK_RTOL = 1e-12  # rpca.py:46


@dataclass(frozen=True)
class AlmConfig:
    """rpca.py:49-80."""

    lam: float | None = None
    mu0: float | None = None
    rho: float = 1.5
    mu_bar: float | None = None
    tol: float = 1e-5
    max_iter: int = 1000
    ell: int | None = None
    q_power: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.rho <= 1:
            raise ValueError("rho must exceed 1")
        if self.mu_bar is not None and self.mu0 is not None and self.mu_bar < self.mu0:
            raise ValueError("mu_bar must be >= mu0")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")


@dataclass
class RpcaSolution:
    """rpca.py:83-96."""

    l: object
    s: object
    iterations: int
    residuals: list[float]
    rank_of_l: int
    nnz_of_s: int
    rank_history: list[int] = field(default_factory=list)
    nnz_history: list[int] = field(default_factory=list)
    mu_history: list[float] = field(default_factory=list)
    ell_history: list[int] = field(default_factory=list)


def shrink(x, delta: float):
    """rpca.py:99-104: sgn(x) max(|x| - delta, 0), on x's device."""
    if delta < 0:
        raise ValueError("delta must be >= 0")
    torch = dev.torch_mod()
    t, was_host = dev.to_device(x, "x")
    out = torch.empty(tuple(t.shape), dtype=torch.float64, device=t.device)
    h = _lib.handle(t.device.index)
    # one fused pass: the finiteness check of as_matrix and the shrinkage
    h.call("corutv_shrink", dev.ptr(t), t.shape[0], t.shape[1], t.stride(0), float(delta), dev.ptr(out),
           out.stride(0))
    return dev.to_output(out, was_host)


def _lowrank_device(u, t, v, r):
    """U[:, :r] (T[:r, :] V') on the device (rpca.py:129)."""
    torch = dev.torch_mod()
    rows, ell = u.shape
    cols = v.shape[0]
    out = torch.empty((rows, cols), dtype=torch.float64, device=u.device)
    h = _lib.handle(u.device.index)
    h.call("corutv_lowrank", dev.ptr(u), dev.ptr(t), dev.ptr(v), rows, cols, ell, r, dev.ptr(out))
    return out


def _numerical_rank(sig, shape) -> int:
    """rpca.py:161-164."""
    if sig.size == 0 or sig[0] <= 0.0:
        return 0
    return int((sig > max(shape) * sig[0] * RANK_RTOL).sum())


def _next_cap(cap: int, rank: int, limit: int, grow: int) -> int:
    """rpca.py:167-172."""
    if rank < cap:
        return max(1, min(rank + 1, limit))
    return max(1, min(rank + grow, limit))


def _truncate(f, delta):
    """rpca.py:122-132 with the count done on |diag T| read back (ell
    doubles) and L kept implicit."""
    d = f.t.diagonal().abs().cpu().numpy()
    return int((d > delta).sum())


def corutv_threshold(b, delta: float, cfg: SketchConfig):
    """rpca.py:107-119: keep the leading r rows of T, r = #(|diag T| > delta)."""
    if delta < 0:
        raise ValueError("delta must be >= 0")
    B, was_host = dev.to_device(b, "b")
    dev.raise_if_nonfinite(B, "b")
    f, r = corutv_truncated(B, cfg, delta)
    if r == 0:
        torch = dev.torch_mod()
        return dev.to_output(torch.zeros_like(B), was_host), 0
    return dev.to_output(_lowrank_device(f.u, f.t, f.v, r), was_host), r


def _svt_device(B, delta: float, cap, v_init):
    """_svt_warm rpca.py:146-158 on the device (corutv_svt): returns
    (u, t, v, k, r, kept) with u[:, :r] (t[:r, :] v') the thresholded matrix
    and v the warm start of the next call."""
    torch = dev.torch_mod()
    m_, n_ = B.shape
    k = min(m_, n_)
    V0 = None
    if v_init is not None:
        if tuple(v_init.shape) != (k, k):
            raise ValueError(f"v_init must be {k}x{k}, got {tuple(v_init.shape)}")
        V0 = v_init
    u = torch.empty((m_, k), dtype=torch.float64, device=B.device)
    v = torch.empty((n_, k), dtype=torch.float64, device=B.device)
    t = torch.empty((k, k), dtype=torch.float64, device=B.device)
    kept = torch.empty((k,), dtype=torch.float64, device=B.device)
    r = ctypes.c_int(0)
    h = _lib.handle(B.device.index)
    h.call("corutv_svt", dev.ptr(B), m_, n_, B.stride(0), delta, -1 if cap is None else int(cap),
           dev.ptr(V0) if V0 is not None else None, V0.stride(0) if V0 is not None else 0,
           dev.ptr(u), dev.ptr(kept), dev.ptr(v), dev.ptr(t), ctypes.byref(r))
    return u, t, v, k, int(r.value), kept


def svt(b, delta: float):
    """rpca.py:135-143: singular value thresholding by the full Jacobi SVD
    (device, min(m, n) <= 16384); returns ``(matrix, r)``."""
    if delta < 0:
        raise ValueError("delta must be >= 0")
    torch = dev.torch_mod()
    B, was_host = dev.to_device(b, "b")
    dev.raise_if_nonfinite(B, "b")
    u, t, v, k, r, _ = _svt_device(B, float(delta), None, None)
    if r == 0:
        return dev.to_output(torch.zeros_like(B), was_host), 0
    return dev.to_output(_lowrank_device(u, t, v, r), was_host), r


def _alm_loop(m, cfg: AlmConfig, step, cap0, global_rows: int | None = None) -> RpcaSolution:
    """rpca.py:175-234 on the device.  ``step(g, delta, cap, j, state)``
    returns (u, t, v, ell, rank, sigma_thunk, state): the thresholded iterate
    is u[:, :rank] (t[:rank, :] v'), kept implicit and fused into the ALM
    update (corutv_alm_update); sigma_thunk() gives the spectrum behind
    rank_of_l once the loop stops."""
    torch = dev.torch_mod()
    M, was_host = dev.to_device(m, "m")
    if M.stride(0) != M.shape[1]:
        M = M.contiguous()
    h_, w_ = M.shape           # local block (all rows unless row-sharded)
    hg = global_rows if global_rows is not None else h_
    handle = _lib.handle(M.device.index)
    lam = cfg.lam if cfg.lam is not None else 1.0 / np.sqrt(max(hg, w_))
    ss = ctypes.c_double(0.0)
    try:
        # the non-finite count is all-reduced with the sum: every rank raises
        handle.call("corutv_sumsq", dev.ptr(M), h_, w_, M.stride(0), ctypes.byref(ss))
    except ValueError:
        raise ValueError("m contains non-finite entries") from None
    norm_m = float(np.sqrt(ss.value))
    if norm_m == 0.0:
        zero = torch.zeros_like(M)
        return RpcaSolution(l=dev.to_output(zero, was_host), s=dev.to_output(zero.clone(), was_host),
                            iterations=1, residuals=[0.0], rank_of_l=0, nnz_of_s=0,
                            rank_history=[0], nnz_history=[0], mu_history=[0.0], ell_history=[0])
    mu = cfg.mu0 if cfg.mu0 is not None else 1.25 / spectral_norm(M)
    mu_bar = cfg.mu_bar if cfg.mu_bar is not None else 1e7 * mu
    limit = min(hg, w_)
    grow = max(1, round(0.05 * limit))
    cap = max(1, min(cap0 if cap0 is not None else limit, limit))
    y = torch.zeros_like(M)
    s = torch.zeros_like(M)
    g = torch.empty_like(M)
    src = M  # G_0 = M - 0 + 0/mu = M
    residuals, ranks, nnzs, mus, caps = [], [], [], [], []
    zeta2 = ctypes.c_double(0.0)
    nnz = ctypes.c_int64(0)
    state = None
    for j in range(cfg.max_iter):
        u, t, v, ell, rank, sigma_of, state = step(src, 1.0 / mu, cap, j, state)
        caps.append(cap)
        cap = _next_cap(cap, rank, limit, grow)
        mu_next = min(cfg.rho * mu, mu_bar)
        handle.call("corutv_alm_update", dev.ptr(M), dev.ptr(s), dev.ptr(y), dev.ptr(g), h_, w_,
                    dev.ptr(u), dev.ptr(t), dev.ptr(v), ell, rank, mu, lam / mu, mu_next,
                    ctypes.byref(zeta2), ctypes.byref(nnz))
        src = g
        zeta = float(np.sqrt(zeta2.value)) / norm_m
        residuals.append(zeta)
        ranks.append(rank)
        nnzs.append(int(nnz.value))
        mus.append(mu)
        if zeta < cfg.tol:
            if rank > 0:
                l_mat = _lowrank_device(u, t, v, rank)
                sig = sigma_of()
            else:
                l_mat = torch.zeros_like(M)
                sig = np.zeros(0)
            return RpcaSolution(
                l=dev.to_output(l_mat, was_host), s=dev.to_output(s, was_host), iterations=j + 1,
                residuals=residuals, rank_of_l=_numerical_rank(sig, (hg, w_)),
                nnz_of_s=int(nnz.value), rank_history=ranks, nnz_history=nnzs, mu_history=mus,
                ell_history=caps,
            )
        mu = mu_next
    raise ConvergenceError(
        f"ALM did not reach tol={cfg.tol:.1e} in {cfg.max_iter} iterations "
        f"(last residual {residuals[-1]:.3e})",
        residual=residuals[-1],
        history=residuals,
    )


def alm_corutv(m, cfg: AlmConfig) -> RpcaSolution:
    """rpca.py:237-255 (+ _alm_loop rpca.py:175-234) on the device."""
    if cfg.ell is None:
        raise ValueError("alm_corutv requires cfg.ell (sketch sample size)")

    def step(g, delta, cap, j, state):
        scfg = SketchConfig(ell=cap, q_power=cfg.q_power, seed=(cfg.seed + j) % 2 ** 64)
        # Omega = gaussian_matrix(w, cap, seed + j) drawn on the device; the
        # rank count r = #(|diag T| > 1/mu) comes back with the factors
        f, rank = corutv_truncated(g, scfg, delta)

        def sigma_of():
            sig = singular_values(f.t[:rank, :])
            return sig.cpu().numpy() if dev.is_device_tensor(sig) else sig

        return f.u, f.t, f.v, f.ell, rank, sigma_of, None

    return _alm_loop(m, cfg, step, cap0=cfg.ell)


def inexact_alm(m, cfg: AlmConfig) -> RpcaSolution:
    """rpca.py:258-273: the InexactALM baseline on the device.  Each
    iteration thresholds G_j by a full one-sided Jacobi SVD warm-started
    from the previous right factor (corutv_svt), the kept rank capped by the
    same prediction schedule; the thresholded iterate stays implicit
    (u, diag(kept), v) and feeds the same fused ALM update."""

    def step(g, delta, cap, j, state):
        u, t, v, k, r, kept = _svt_device(g, delta, cap, state)
        return u, t, v, k, r, (lambda: kept[:r].cpu().numpy()), v

    # cap0 = cfg.ell, else min(m.shape) (rpca.py:272)
    return _alm_loop(m, cfg, step, cap0=cfg.ell)


def write_telemetry_csv(solution: RpcaSolution, path) -> None:
    """rpca.py:276-283: iter,zeta,rank_l,nnz_s,mu."""
    with open(path, "w", encoding="ascii", newline="\n") as fh:
        fh.write("iter,zeta,rank_l,nnz_s,mu\n")
        rows = zip(solution.residuals, solution.rank_history, solution.nnz_history,
                   solution.mu_history)
        for i, (zeta, rank, nz, mu) in enumerate(rows, start=1):
            fh.write(f"{i},{zeta!r},{rank},{nz},{mu!r}\n")
