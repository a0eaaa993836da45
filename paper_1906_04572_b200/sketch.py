"""CoR-UTV on the B200 — drop-in for the reference's ``corutv.sketch``.

Same names, signatures, validation messages and result types as
/root/reference/pkg/src/corutv/sketch.py; the numerics run in the sm_100a
library (``corutv_decompose``, include/corutv_b200.h).

Additive API: ``corutv(..., omega=None)`` accepts a
caller-supplied n x ell Gaussian test matrix (default: ``gaussian_matrix(n,
ell, seed)`` exactly as sketch.py:174), and :func:`corutv_kpq` takes the
north-star's (A, k, p, q, omega) form with ell = k + p.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from . import _lib
from .dense import SvdFactors

__all__ = [
    "VARIANT_EXACT",
    "VARIANT_APPROX",
    "SketchConfig",
    "CorUtvFactors",
    "PassCounter",
    "gaussian_matrix",
    "corutv",
    "corutv_kpq",
    "corutv_lowrank_error",
    "count_passes",
    "flop_estimate",
    "svd_flop_estimate",
    "sor_svd",
    "tsr_svd",
    "SvdFactors",
]

SECOND_STREAM_OFFSET = 0x9E3779B9  # sketch.py:60

VARIANT_EXACT = "exact-d"   # sketch.py:53
VARIANT_APPROX = "approx-d"  # sketch.py:55
_VARIANTS = (VARIANT_EXACT, VARIANT_APPROX)
_VARIANT_CODE = {VARIANT_EXACT: _lib.EXACT_D, VARIANT_APPROX: _lib.APPROX_D}


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """sketch.py:63-68: numpy PCG64(seed) ziggurat normals, host side.

    The test matrix is an *input* of the decomposition; it is drawn with the
    same numpy generator as the reference so that results are comparable on
    identical seeds (SURVEY §7 "Omega parity")."""
    if rows < 1 or cols < 1:
        raise ValueError(f"gaussian_matrix needs positive dims, got {rows}x{cols}")
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((rows, cols))


@dataclass(frozen=True)
class SketchConfig:
    """sketch.py:71-98 — ell (sample size), q_power, seed, variant."""

    ell: int
    q_power: int = 0
    seed: int = 0
    variant: str = VARIANT_EXACT

    def __post_init__(self):
        if self.ell < 1:
            raise ValueError(f"ell must be >= 1, got {self.ell}")
        if self.q_power < 0:
            raise ValueError(f"q_power must be >= 0, got {self.q_power}")
        if self.variant not in _VARIANTS:
            raise ValueError(f"variant must be one of {_VARIANTS}, got {self.variant!r}")

    def validated_for(self, m: int, n: int) -> "SketchConfig":
        if self.ell > min(m, n):
            raise ValueError(
                f"ell={self.ell} exceeds min(m, n)={min(m, n)} for a {m}x{n} input"
            )
        return self


@dataclass
class CorUtvFactors:
    """sketch.py:101-123 — u (m x ell), t (ell x ell upper), v (n x ell).

    Arrays are numpy for host inputs and torch CUDA tensors for device
    inputs.  ``perm`` (extra) is the QRCP column permutation."""

    u: object
    t: object
    v: object
    ell: int
    q_power: int
    variant: str
    perm: object = None

    def lowrank(self):
        """The rank-ell approximation u @ (t @ v.T) (sketch.py:117-119)."""
        if dev.is_device_tensor(self.u):
            from .rpca import _lowrank_device

            return _lowrank_device(self.u, self.t, self.v, self.ell)
        return self.u @ (self.t @ self.v.T)

    def diag_abs(self):
        """|diag(t)| (sketch.py:121-123)."""
        if dev.is_device_tensor(self.t):
            return self.t.diagonal().abs()
        return np.abs(np.diag(self.t))


@dataclass
class PassCounter:
    """sketch.py:126-133 — full sweeps over the data matrix."""

    passes: int = 0

    def add(self, n: int = 1) -> None:
        self.passes += n


def pcg_state(seed: int):
    """numpy's PCG64(seed) starting state as {state_hi, state_lo, inc_hi,
    inc_lo} (SeedSequence expansion on the host; the draws themselves are
    generated on the device, bit-identical to gaussian_matrix)."""
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    return (ctypes.c_uint64 * 4)(s >> 64, s & m64, inc >> 64, inc & m64)


def gaussian_matrix_device(rows: int, cols: int, seed: int, device=None):
    """gaussian_matrix(rows, cols, seed) generated on the B200 (PCG64 +
    ziggurat, bit-identical to numpy)."""
    torch = dev.torch_mod()
    if rows < 1 or cols < 1:
        raise ValueError(f"gaussian_matrix needs positive dims, got {rows}x{cols}")
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    out = torch.empty((rows, cols), dtype=torch.float64, device=device)
    h = _lib.handle(out.device.index)
    h.call("corutv_gaussian", pcg_state(seed), rows, cols, dev.ptr(out), cols)
    return out


def _omega_device(omega, n, ell, seed, device_like):
    torch = dev.torch_mod()
    if omega is None:
        omega = gaussian_matrix(n, ell, seed)
    if dev.is_device_tensor(omega):
        om = omega.to(torch.float64).contiguous()
    else:
        om = torch.from_numpy(np.ascontiguousarray(omega, dtype=np.float64)).to(device_like.device)
    if tuple(om.shape) != (n, ell):
        raise ValueError(f"omega must be {n}x{ell}, got {tuple(om.shape)}")
    return om


def corutv(a, cfg: SketchConfig, counter: PassCounter | None = None, omega=None) -> CorUtvFactors:
    """Compressed randomized UTV (sketch.py:182-208) on the B200.

    Requires m >= n.  ``a``: numpy-compatible host array (copied to the
    current CUDA device) or a CUDA tensor (used in place).  ``omega``:
    optional caller-supplied n x ell test matrix."""
    torch = dev.torch_mod()
    a = dev.shape_check(a, "a")
    m, n = (tuple(a.shape))
    if m < n or cfg.ell > min(m, n):
        # reference order: as_matrix's finiteness check comes first (dense.py:48)
        t, _ = dev.to_device(a, "a")
        dev.raise_if_nonfinite(t, "a")
        if m < n:
            raise ValueError(f"corutv requires rows >= cols, got {m}x{n}")
        cfg.validated_for(m, n)
    if not dev.is_device_tensor(a):
        return _corutv_host(a, cfg, counter, omega)
    A, was_host = dev.to_device(a, "a")
    ell = cfg.ell
    u = torch.empty((m, ell), dtype=torch.float64, device=A.device)
    t = torch.empty((ell, ell), dtype=torch.float64, device=A.device)
    v = torch.empty((n, ell), dtype=torch.float64, device=A.device)
    perm = torch.empty((ell,), dtype=torch.int64, device=A.device)
    passes = ctypes.c_int64(0)
    h = _lib.handle(A.device.index)
    if omega is None:
        # Omega = gaussian_matrix(n, ell, seed) drawn on the device (sketch.py:174)
        h.call("corutv_decompose_seeded", dev.ptr(A), m, n, A.stride(0), ell, cfg.q_power,
               _VARIANT_CODE[cfg.variant], pcg_state(cfg.seed), dev.ptr(u), dev.ptr(t),
               dev.ptr(v), dev.ptr(perm), ctypes.byref(passes))
    else:
        om = _omega_device(omega, n, ell, cfg.seed, A)
        h.call("corutv_decompose", dev.ptr(A), m, n, A.stride(0), ell, cfg.q_power,
               _VARIANT_CODE[cfg.variant], dev.ptr(om), dev.ptr(u), dev.ptr(t), dev.ptr(v),
               dev.ptr(perm), ctypes.byref(passes))
    if counter is not None:
        counter.add(passes.value)
    return CorUtvFactors(u=dev.to_output(u, was_host), t=dev.to_output(t, was_host),
                         v=dev.to_output(v, was_host), ell=ell, q_power=cfg.q_power,
                         variant=cfg.variant, perm=dev.to_output(perm, was_host))


def _host_source(a):
    """(keep-alive source, host pointer, ld, output kind) of a host matrix:
    numpy arrays come back as numpy, host torch tensors as host tensors."""
    torch = dev.torch_mod()
    if dev.is_host_tensor(a):
        src = a if (a.dtype == torch.float64 and a.stride(1) == 1) else a.to(torch.float64).contiguous()
        return src, src.data_ptr(), src.stride(0), "torch"
    src = np.ascontiguousarray(a, dtype=np.float64)
    return src, src.ctypes.data, src.shape[1], True


def _staged_outputs(tensors, kind, device):
    """D2H through pinned staging (torch's host caching allocator recycles
    the blocks call to call), one synchronisation."""
    torch = dev.torch_mod()
    outs = []
    for x in tensors:
        y = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        y.copy_(x, non_blocking=True)
        outs.append(y)
    torch.cuda.current_stream(device).synchronize()
    return [y.numpy() for y in outs] if kind is True else outs


def _corutv_host(a, cfg: SketchConfig, counter: PassCounter | None, omega) -> CorUtvFactors:
    """corutv of a host-resident matrix: the library streams A into a device
    buffer in row chunks and overlaps the copy with Omega and the first
    sketch sweep (corutv_decompose_host); results are bit-identical to the
    device-resident call.  Factors come back as numpy arrays (host torch
    tensors for a host torch input)."""
    torch = dev.torch_mod()
    src, host_ptr, ld_host, kind = _host_source(a)
    m, n = src.shape
    ell = cfg.ell
    device = torch.device("cuda", torch.cuda.current_device())
    ld_dev = n + (n & 1)
    a_dev = torch.empty((m, ld_dev), dtype=torch.float64, device=device)
    u = torch.empty((m, ell), dtype=torch.float64, device=device)
    t = torch.empty((ell, ell), dtype=torch.float64, device=device)
    v = torch.empty((n, ell), dtype=torch.float64, device=device)
    perm = torch.empty((ell,), dtype=torch.int64, device=device)
    passes = ctypes.c_int64(0)
    h = _lib.handle(device.index)
    om = None if omega is None else _omega_device(omega, n, ell, cfg.seed, a_dev)
    h.call("corutv_decompose_host", host_ptr, m, n, ld_host, dev.ptr(a_dev), ld_dev, ell, cfg.q_power,
           _VARIANT_CODE[cfg.variant], None if om is None else dev.ptr(om),
           None if om is not None else pcg_state(cfg.seed), dev.ptr(u), dev.ptr(t), dev.ptr(v),
           dev.ptr(perm), ctypes.byref(passes))
    del src
    if counter is not None:
        counter.add(passes.value)
    outs = _staged_outputs((u, t, v, perm), kind, device)
    return CorUtvFactors(u=outs[0], t=outs[1], v=outs[2], ell=ell, q_power=cfg.q_power, variant=cfg.variant,
                         perm=outs[3])


def corutv_truncated(A, cfg: SketchConfig, delta: float, counter: PassCounter | None = None):
    """CoR-UTV of a CUDA tensor for the ALM thresholding step
    (rpca.py:122-132): returns (factors, r) with r = #(|diag T| > delta); the
    QRCP stops at step r, so only U[:, :r] and T[:r, :] are formed (the rest
    of U / T is not meaningful) -- L = U_r (T_r V') is unchanged."""
    torch = dev.torch_mod()
    m, n = A.shape
    ell = cfg.ell
    u = torch.empty((m, ell), dtype=torch.float64, device=A.device)
    t = torch.empty((ell, ell), dtype=torch.float64, device=A.device)
    v = torch.empty((n, ell), dtype=torch.float64, device=A.device)
    perm = torch.empty((ell,), dtype=torch.int64, device=A.device)
    passes = ctypes.c_int64(0)
    r = ctypes.c_int(0)
    h = _lib.handle(A.device.index)
    h.call("corutv_decompose_truncated", dev.ptr(A), m, n, A.stride(0), ell, cfg.q_power,
           _VARIANT_CODE[cfg.variant], None, pcg_state(cfg.seed), float(delta), dev.ptr(u),
           dev.ptr(t), dev.ptr(v), dev.ptr(perm), ctypes.byref(passes), ctypes.byref(r))
    if counter is not None:
        counter.add(passes.value)
    return CorUtvFactors(u=u, t=t, v=v, ell=ell, q_power=cfg.q_power, variant=cfg.variant,
                         perm=perm), int(r.value)


def _svd_outputs(u, sigma, v, was_host):
    return SvdFactors(u=dev.to_output(u, was_host), sigma=dev.to_output(sigma, was_host),
                      v=dev.to_output(v, was_host))


def _svd_host(kind_name, a, cfg, counter, g1, g2) -> SvdFactors:
    """sor_svd / tsr_svd of a host matrix, streamed (corutv_{sor,tsr}_svd_host)."""
    torch = dev.torch_mod()
    src, host_ptr, ld_host, kind = _host_source(a)
    m, n = src.shape
    ell = cfg.ell
    device = torch.device("cuda", torch.cuda.current_device())
    ld_dev = n + (n & 1)
    a_dev = torch.empty((m, ld_dev), dtype=torch.float64, device=device)
    u = torch.empty((m, ell), dtype=torch.float64, device=device)
    s = torch.empty((ell,), dtype=torch.float64, device=device)
    v = torch.empty((n, ell), dtype=torch.float64, device=device)
    passes = ctypes.c_int64(0)
    h = _lib.handle(device.index)
    if kind_name == "sor":
        om = None if g1 is None else _omega_device(g1, n, ell, cfg.seed, a_dev)
        h.call("corutv_sor_svd_host", host_ptr, m, n, ld_host, dev.ptr(a_dev), ld_dev, ell, cfg.q_power,
               _VARIANT_CODE[cfg.variant], None if om is None else dev.ptr(om),
               None if om is not None else pcg_state(cfg.seed), dev.ptr(u), dev.ptr(s), dev.ptr(v),
               ctypes.byref(passes))
    else:
        ps = None if g1 is None else _omega_device(g1, n, ell, cfg.seed, a_dev)
        ph = None if g2 is None else _omega_device(g2, m, ell, cfg.seed, a_dev)
        h.call("corutv_tsr_svd_host", host_ptr, m, n, ld_host, dev.ptr(a_dev), ld_dev, ell,
               None if ps is None else dev.ptr(ps), None if ps is not None else pcg_state(cfg.seed),
               None if ph is None else dev.ptr(ph),
               None if ph is not None else pcg_state((cfg.seed + SECOND_STREAM_OFFSET) % 2 ** 64),
               dev.ptr(u), dev.ptr(s), dev.ptr(v), ctypes.byref(passes))
    del src
    if counter is not None:
        counter.add(passes.value)
    outs = _staged_outputs((u, s, v), kind, device)
    return SvdFactors(u=outs[0], sigma=outs[1], v=outs[2])


def sor_svd(a, cfg: SketchConfig, counter: PassCounter | None = None, omega=None) -> SvdFactors:
    """sketch.py:244-262: the corutv pipeline finished by a Jacobi SVD of the
    compressed core (corutv_sor_svd)."""
    torch = dev.torch_mod()
    a = dev.shape_check(a, "a")
    m, n = tuple(a.shape)
    if m < n or cfg.ell > min(m, n):
        # reference order: as_matrix's finiteness check comes first (dense.py:48);
        # otherwise the first sweep flags non-finite entries on the device
        t_, _ = dev.to_device(a, "a")
        dev.raise_if_nonfinite(t_, "a")
        if m < n:
            raise ValueError(f"sor_svd requires rows >= cols, got {m}x{n}")
        cfg.validated_for(m, n)
    if not dev.is_device_tensor(a):
        return _svd_host("sor", a, cfg, counter, omega, None)
    A, was_host = dev.to_device(a, "a")
    ell = cfg.ell
    u = torch.empty((m, ell), dtype=torch.float64, device=A.device)
    s = torch.empty((ell,), dtype=torch.float64, device=A.device)
    v = torch.empty((n, ell), dtype=torch.float64, device=A.device)
    om = None if omega is None else _omega_device(omega, n, ell, cfg.seed, A)
    passes = ctypes.c_int64(0)
    h = _lib.handle(A.device.index)
    h.call("corutv_sor_svd", dev.ptr(A), m, n, A.stride(0), ell, cfg.q_power, _VARIANT_CODE[cfg.variant],
           None if om is None else dev.ptr(om), None if om is not None else pcg_state(cfg.seed),
           dev.ptr(u), dev.ptr(s), dev.ptr(v), ctypes.byref(passes))
    if counter is not None:
        counter.add(passes.value)
    return _svd_outputs(u, s, v, was_host)


def tsr_svd(a, cfg: SketchConfig, counter: PassCounter | None = None, psi=None, phi=None) -> SvdFactors:
    """sketch.py:220-241: two-sided randomized SVD, psi = G(n, ell, seed),
    phi = G(m, ell, seed + 0x9E3779B9 mod 2^64) drawn on the device
    (corutv_tsr_svd).  One algorithmic pass (counted as the reference's
    fused sweep)."""
    torch = dev.torch_mod()
    a = dev.shape_check(a, "a")
    m, n = tuple(a.shape)
    if cfg.ell > min(m, n):
        t_, _ = dev.to_device(a, "a")
        dev.raise_if_nonfinite(t_, "a")  # reference order (dense.py:48)
        cfg.validated_for(m, n)
    if not dev.is_device_tensor(a):
        return _svd_host("tsr", a, cfg, counter, psi, phi)
    A, was_host = dev.to_device(a, "a")
    ell = cfg.ell
    u = torch.empty((m, ell), dtype=torch.float64, device=A.device)
    s = torch.empty((ell,), dtype=torch.float64, device=A.device)
    v = torch.empty((n, ell), dtype=torch.float64, device=A.device)
    ps = None if psi is None else _omega_device(psi, n, ell, cfg.seed, A)
    ph = None if phi is None else _omega_device(phi, m, ell, cfg.seed, A)
    passes = ctypes.c_int64(0)
    h = _lib.handle(A.device.index)
    h.call("corutv_tsr_svd", dev.ptr(A), m, n, A.stride(0), ell,
           None if ps is None else dev.ptr(ps), None if ps is not None else pcg_state(cfg.seed),
           None if ph is None else dev.ptr(ph),
           None if ph is not None else pcg_state((cfg.seed + SECOND_STREAM_OFFSET) % 2 ** 64),
           dev.ptr(u), dev.ptr(s), dev.ptr(v), ctypes.byref(passes))
    if counter is not None:
        counter.add(passes.value)
    return _svd_outputs(u, s, v, was_host)


def corutv_kpq(a, k: int, p: int, q: int, omega=None, seed: int = 0,
               variant: str = VARIANT_EXACT) -> CorUtvFactors:
    """North-star form: target rank k, oversampling p (ell = k + p), q power
    iterations, optional caller-supplied Gaussian test matrix."""
    return corutv(a, SketchConfig(ell=k + p, q_power=q, seed=seed, variant=variant), omega=omega)


def corutv_lowrank_error(a, cfg: SketchConfig, counter: PassCounter | None = None) -> float:
    """sketch.py:211-217: |A - U T V'|_F, evaluated on the device without
    materialising U T V' (one fused GEMM + residual pass)."""
    torch = dev.torch_mod()
    A, _ = dev.to_device(a, "a")
    f = corutv(A, cfg, counter)
    out = ctypes.c_double(0.0)
    h = _lib.handle(A.device.index)
    h.call("corutv_lowrank_error", dev.ptr(A), A.shape[0], A.shape[1], A.stride(0),
           dev.ptr(f.u), dev.ptr(f.t), dev.ptr(f.v), f.ell, ctypes.byref(out))
    del torch
    return float(out.value)


def count_passes(fn, a, cfg: SketchConfig) -> int:
    """sketch.py:265-269."""
    counter = PassCounter()
    fn(a, cfg, counter)
    return counter.passes


def flop_estimate(m: int, n: int, ell: int, q_power: int = 0, variant: str = VARIANT_EXACT) -> int:
    """sketch.py:272-296 — the algorithmic flop count (metric numerator)."""
    if min(m, n, ell) < 1:
        raise ValueError("dimensions must be positive")
    if variant not in _VARIANTS:
        raise ValueError(f"variant must be one of {_VARIANTS}, got {variant!r}")
    reps = q_power + 1
    total = n * ell
    total += reps * 2 * m * n * ell
    total += reps * 2 * m * n * ell
    total += 2 * m * ell ** 2 + 2 * n * ell ** 2
    if variant == VARIANT_EXACT:
        total += m * ell ** 2 + 2 * m * n * ell
    else:
        total += 2 * m * ell ** 2 + 2 * n * ell ** 2 + 3 * ell ** 3
    total += (8 * ell ** 3) // 3
    total += 2 * m * ell ** 2 + 2 * n * ell
    return total


def svd_flop_estimate(m: int, n: int) -> int:
    """sketch.py:299-304: textbook flop count of a full economy SVD."""
    if m < n:
        m, n = n, m
    return 14 * m * n ** 2 + 8 * n ** 3
