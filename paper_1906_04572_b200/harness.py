"""Experiment harness on the device — drop-in for the reference's
``corutv.bench`` experiments (bench.py:165-290).

Same configs, methods, report rows and CSV bytes as the reference's
``run_sv_compare`` / ``run_lowrank_error`` / ``run_rpca_recovery``, with
every method on the device:

* ``svd``        — singular_values (one-sided Jacobi; the cooperative-grid
                   kernel for n above ~116)
* ``qrcp``       — corutv_qrcp (Businger-Golub, one CTA or a cluster)
* ``corutv`` / ``utv-approx`` / ``tsr-svd`` / ``sor-svd`` — the device
  decompositions; low-rank errors |A - approx|_F by the fused residual
  kernel (corutv_lowrank_error[_rank]), so no approximation is ever formed

The input matrix is uploaded once and shared.  The randomized methods'
trials (seeds base_seed + t) run on a pool of worker threads, each with its
own CUDA stream and native handle, so the trials' latency-bound small
kernels (Cholesky steps, QRCP, Jacobi cores) overlap on the GPU; results are
assembled in trial order and are bitwise independent of the scheduling
(each trial's arithmetic is fixed by its plan), so reports are
byte-identical across re-runs (bench.py:1-16's contract).  Worker count:
``CORUTV_THREADS`` as in the reference (bench.py:59-65), default 8 here.
"""

from __future__ import annotations

import ctypes
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _device as dev
from . import _lib
from .dense import singular_values
from .errors import CorutvError
from .rpca import AlmConfig, alm_corutv, inexact_alm, write_telemetry_csv
from .sketch import VARIANT_EXACT, SketchConfig, corutv, flop_estimate, sor_svd, svd_flop_estimate, tsr_svd
from .synth import NoisyLowRankSpec, RpcaInstanceSpec, gen_noisy_lowrank, gen_rpca_instance

__all__ = [
    "EXPERIMENTS", "METHODS", "SOLVERS", "ExperimentConfig", "run_sv_compare", "run_lowrank_error",
    "run_rpca_recovery", "solver_flops", "svd_flop_estimate", "write_csv", "run_trials",
]

EXPERIMENTS = ("sv-compare", "lowrank-error", "rpca-recovery")
METHODS = ("svd", "qrcp", "utv-approx", "corutv", "tsr-svd", "sor-svd")
SOLVERS = ("inexact-alm", "alm-corutv")
_RANDOMIZED = {"corutv", "tsr-svd", "sor-svd", "utv-approx"}

SV_COMPARE_HEADER = "index,method,value,trial_mean,trial_std"
LOWRANK_HEADER = "ell,method,ek_mean,ek_std,svd_optimal"
RPCA_HEADER = "n,solver,rank_l,nnz_s,iters,zeta,flops_est"


def _max_workers() -> int:
    """bench.py:59-65, device default 8."""
    raw = os.environ.get("CORUTV_THREADS", "8")
    try:
        w = int(raw)
    except ValueError:
        raise ValueError(f"CORUTV_THREADS must be an integer, got {raw!r}")
    return max(1, w)


_POOL = {"workers": 0, "pool": None}
_STREAMS = threading.local()


def _pool(workers: int) -> ThreadPoolExecutor:
    # one persistent pool: its threads keep their native handles (arena,
    # pinned buffers) and CUDA streams across experiments
    if _POOL["workers"] != workers:
        if _POOL["pool"] is not None:
            _POOL["pool"].shutdown(wait=True)
        _POOL["pool"] = ThreadPoolExecutor(max_workers=workers, thread_name_prefix="corutv-trial")
        _POOL["workers"] = workers
    return _POOL["pool"]


def run_trials(fn, trials: int):
    """bench.py:68-79: fn(t) for t in range(trials), in trial order.  Each
    worker thread launches on its own CUDA stream (native handles are per
    thread, bound to the thread's current stream)."""
    torch = dev.torch_mod()
    workers = min(_max_workers(), trials)
    if workers == 1:
        return [fn(t) for t in range(trials)]
    device = torch.cuda.current_device()
    torch.cuda.current_stream().synchronize()  # inputs ready before the side streams read them

    def run(t):
        torch.cuda.set_device(device)
        streams = getattr(_STREAMS, "by_device", None)
        if streams is None:
            streams = _STREAMS.by_device = {}
        st = streams.get(device)
        if st is None:
            st = streams[device] = torch.cuda.Stream(device=device)
        with torch.cuda.stream(st):
            out = fn(t)
            st.synchronize()
        return out

    return list(_pool(_max_workers()).map(run, range(trials)))


@dataclass(frozen=True)
class ExperimentConfig:
    """bench.py:82-137."""

    experiment: str
    n: int = 400
    k: int = 20
    ell: int | None = None
    ell_sweep: tuple = ()
    q_power: int = 0
    trials: int = 20
    base_seed: int = 1
    matrix_seed: int = 0
    methods: tuple = ("svd", "corutv", "tsr-svd", "sor-svd", "qrcp")
    noise_coeff: float = 0.1
    sizes: tuple = ()
    rank_fraction: float = 0.05
    sparsity_fraction: float = 0.05
    amplitude: float = 80.0
    solvers: tuple = SOLVERS
    out_path: str | None = None
    telemetry_prefix: str | None = None

    def __post_init__(self):
        if self.experiment not in EXPERIMENTS:
            raise ValueError(f"experiment must be one of {EXPERIMENTS}")
        if self.trials < 1:
            raise ValueError("trials must be >= 1")
        for m in self.methods:
            if m not in METHODS:
                raise ValueError(f"unknown method {m!r}, expected one of {METHODS}")
        for s in self.solvers:
            if s not in SOLVERS:
                raise ValueError(f"unknown solver {s!r}, expected one of {SOLVERS}")
        for ell in self.ell_sweep:
            if not self.k <= ell <= self.n:
                raise ValueError(f"sweep value ell={ell} outside [k, n] = [{self.k}, {self.n}]")

    def resolved_ell(self) -> int:
        return self.ell if self.ell is not None else 2 * self.k

    def resolved_sweep(self) -> tuple:
        if self.ell_sweep:
            return self.ell_sweep
        k = self.k
        return (k, k + k // 2, 2 * k, 3 * k)


def _fmt(x) -> str:
    if isinstance(x, float):
        return repr(x)
    return str(x)


def write_csv(path, header: str, rows) -> None:
    """bench.py:146-150."""
    with open(path, "w", encoding="ascii", newline="\n") as fh:
        fh.write(header + "\n")
        for row in rows:
            fh.write(",".join(_fmt(x) for x in row) + "\n")


# ------------------------------------------------------------ device methods

def _qrcp(A):
    torch = dev.torch_mod()
    n = A.shape[0]
    if A.shape[1] != n:
        raise ValueError("the harness qrcp method needs a square matrix")
    q = torch.empty((n, n), dtype=torch.float64, device=A.device)
    r = torch.empty((n, n), dtype=torch.float64, device=A.device)
    perm = torch.empty((n,), dtype=torch.int64, device=A.device)
    _lib.handle(A.device.index).call("corutv_qrcp", dev.ptr(A), n, A.stride(0), dev.ptr(q), dev.ptr(r),
                                     dev.ptr(perm))
    return q, r, perm


def _resid(A, u, t, v, ell, r) -> float:
    out = ctypes.c_double(0.0)
    _lib.handle(A.device.index).call("corutv_lowrank_error_rank", dev.ptr(A), A.shape[0], A.shape[1],
                                     A.stride(0), dev.ptr(u), dev.ptr(t), dev.ptr(v), ell, r,
                                     ctypes.byref(out))
    return float(out.value)


def _method_sigma(method: str, A, ell: int, q_power: int, seed: int) -> np.ndarray:
    """bench.py:140-162 on the device."""
    n = min(A.shape)
    if method == "svd":
        return singular_values(A)[:ell].cpu().numpy()
    if method == "qrcp":
        _, r, _ = _qrcp(A)
        return r.diagonal().abs()[:ell].cpu().numpy()
    if method == "utv-approx":
        cfg = SketchConfig(ell=n, q_power=q_power, seed=seed, variant=VARIANT_EXACT)
        return corutv(A, cfg).diag_abs()[:ell].cpu().numpy()
    cfg = SketchConfig(ell=ell, q_power=q_power, seed=seed)
    if method == "corutv":
        return corutv(A, cfg).diag_abs().cpu().numpy()
    if method == "tsr-svd":
        return tsr_svd(A, cfg).sigma.cpu().numpy()
    if method == "sor-svd":
        return sor_svd(A, cfg).sigma.cpu().numpy()
    raise ValueError(f"unknown method {method!r}")


def _method_lowrank_error(method: str, A, sig: np.ndarray, ell: int, q_power: int, seed: int) -> float:
    """bench.py:201-226 on the device: |A - approx|_F by the fused residual
    kernel, the approximation kept as u (t v')."""
    torch = dev.torch_mod()
    if method == "svd":
        return float(np.sqrt((sig[ell:] ** 2).sum()))
    if method == "qrcp":
        # A[:, perm] - Q_l R_l  ==  A - Q_l (R_l P'),  P[perm[c], c] = 1
        q, r, perm = _qrcp(A)
        n = A.shape[1]
        p = torch.zeros((n, n), dtype=torch.float64, device=A.device)
        p[perm, torch.arange(n, device=A.device)] = 1.0
        return _resid(A, q, r, p, n, ell)
    cfg = SketchConfig(ell=ell, q_power=q_power, seed=seed)
    if method == "utv-approx":
        f = corutv(A, SketchConfig(ell=min(A.shape), q_power=q_power, seed=seed))
        return _resid(A, f.u, f.t, f.v, f.ell, ell)
    if method == "corutv":
        f = corutv(A, cfg)
        return _resid(A, f.u, f.t, f.v, f.ell, f.ell)
    if method in ("tsr-svd", "sor-svd"):
        f = (tsr_svd if method == "tsr-svd" else sor_svd)(A, cfg)
        k = f.sigma.shape[0]
        return _resid(A, f.u, torch.diag(f.sigma).contiguous(), f.v, k, k)
    raise ValueError(f"unknown method {method!r}")


def _input(cfg: ExperimentConfig):
    spec = NoisyLowRankSpec(n=cfg.n, k=cfg.k, seed=cfg.matrix_seed, noise_coeff=cfg.noise_coeff)
    a, _ = gen_noisy_lowrank(spec)
    A, _ = dev.to_device(a, "a")
    return A


def run_sv_compare(cfg: ExperimentConfig):
    """bench.py:165-196: per-index singular-value estimates per method,
    mean / std over trials for the randomized methods."""
    A = _input(cfg)
    ell = cfg.resolved_ell()
    rows = []
    for method in cfg.methods:
        if method in _RANDOMIZED:
            ests = run_trials(lambda t, m=method: _method_sigma(m, A, ell, cfg.q_power, cfg.base_seed + t),
                              cfg.trials)
            stack = np.vstack(ests)
            mean = stack.mean(axis=0)
            std = stack.std(axis=0)
        else:
            est = _method_sigma(method, A, ell, cfg.q_power, cfg.base_seed)
            mean = est
            std = np.zeros_like(est)
        for i in range(len(mean)):
            rows.append((i + 1, method, float(mean[i]), float(mean[i]), float(std[i])))
    if cfg.out_path:
        write_csv(cfg.out_path, SV_COMPARE_HEADER, rows)
    return rows


def run_lowrank_error(cfg: ExperimentConfig):
    """bench.py:229-256: mean low-rank error per (sample size, method)."""
    A = _input(cfg)
    sig = singular_values(A).cpu().numpy()
    rows = []
    for ell in cfg.resolved_sweep():
        optimal = float(np.sqrt((sig[ell:] ** 2).sum()))
        for method in cfg.methods:
            if method in _RANDOMIZED:
                errs = run_trials(lambda t, m=method: _method_lowrank_error(m, A, sig, ell, cfg.q_power,
                                                                            cfg.base_seed + t),
                                  cfg.trials)
                errs = np.array(errs)
                mean, std = float(errs.mean()), float(errs.std())
            else:
                mean = _method_lowrank_error(method, A, sig, ell, cfg.q_power, cfg.base_seed)
                std = 0.0
            rows.append((ell, method, mean, std, optimal))
    if cfg.out_path:
        write_csv(cfg.out_path, LOWRANK_HEADER, rows)
    return rows


def solver_flops(solver: str, n: int, q_power: int, sol) -> int:
    """bench.py:259-273."""
    total = 0
    for i, r in enumerate(sol.rank_history):
        if solver == "alm-corutv":
            ell = max(1, sol.ell_history[i])
            total += flop_estimate(n, n, ell, q_power, VARIANT_EXACT)
            total += 2 * r * ell * n
        else:
            total += svd_flop_estimate(n, n)
        total += 2 * n * n * r
        total += 8 * n * n
    return total


def run_rpca_recovery(cfg: ExperimentConfig):
    """bench.py:276-306: recovery statistics per (size, solver)."""
    sizes = cfg.sizes if cfg.sizes else (cfg.n,)
    rows = []
    for n in sizes:
        k = max(1, round(cfg.rank_fraction * n))
        s = round(cfg.sparsity_fraction * n * n)
        spec = RpcaInstanceSpec(n=n, k=k, s=s, amplitude=cfg.amplitude, seed=cfg.matrix_seed)
        m_mat, _, _ = gen_rpca_instance(spec)
        M, _ = dev.to_device(m_mat, "m")
        ell = cfg.ell if cfg.ell is not None else 2 * k
        for solver in cfg.solvers:
            alm_cfg = AlmConfig(ell=ell, q_power=max(cfg.q_power, 1), seed=cfg.base_seed)
            try:
                sol = (alm_corutv if solver == "alm-corutv" else inexact_alm)(M, alm_cfg)
                flops = solver_flops(solver, n, alm_cfg.q_power, sol)
                rows.append((n, solver, sol.rank_of_l, sol.nnz_of_s, sol.iterations, float(sol.residuals[-1]),
                             flops))
                if cfg.telemetry_prefix:
                    write_telemetry_csv(sol, f"{cfg.telemetry_prefix}.{n}.{solver}.csv")
            except CorutvError:
                rows.append((n, solver, -1, -1, -1, float("nan"), -1))
    if cfg.out_path:
        write_csv(cfg.out_path, RPCA_HEADER, rows)
    return rows
