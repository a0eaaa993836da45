"""CoR-UTV / ALM-CoRUTV benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c3|c2|c1|c5] [--no-e2e] [--no-rpca] [--no-cpu] [--no-extra]

Metric (BASELINE.json): "CoR-UTV GFLOP/s & % FP64 TC peak at 1/2/4/8 B200;
RPCA ms/iter".  A step is one full CoR-UTV (sketch.py:182-208) of the
workload matrix; GFLOP/s uses the reference's own algorithmic flop count
(corutv.flop_estimate, sketch.py:272-296).  Default workload = BASELINE
configs[2] (C3): A = X Y' + 1e-4 G, 131072 x 32768 (34.4 GB), X, Y with 100
columns scaled 1/sqrt(n), k = 100, p = 10 (ell = 110), q = 2 -- the config
quoted at 1/2/4/8 B200, row-sharded across ranks (strong scaling).  The
same line carries the RPCA ms/iter of configs[3] (C4, n = 10000) under
"rpca" and, at N = 1, configs[0], [1] and [4] (C1, C2, C5) under
"workloads", each with its roofline fraction; "tsr_svd_ell8" there times tsr_svd on
the resident C3 matrix with one pass over A against two sweeps.

Inputs are synthetic (seeded, generated on the device; no dataset).  A is
34 GB >> the 126 MB L2, so every timed step streams it from HBM (no flush
needed).  Timing: CUDA events on the library's stream over exactly K steps
bracketed by barrier + synchronize, max over ranks.

--impl reference runs the reference package itself (baseline/_ref, the
unmodified corutv installed by pip --target) on the host cores, on the
FULL workload matrix -- the identical A (same device generator, copied to
the host) and the identical seeded Omega -- so both lines share one config.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (m, n, ell, q, rank, noise, description)
    "c1": (1000, 1000, 15, 0, 10, 1e-3, "BASELINE configs[0]: 1000x1000 X Y' + E (E ~ N(0,1e-6)), k=10 p=5 q=0"),
    "c2": (4000, 3000, 50, 1, 40, None, "BASELINE configs[1]: 4000x3000 U diag(1 (i<=40), 0.8^(i-40)) V', k=40 p=10 q=1"),
    "c3": (131072, 32768, 110, 2, 100, 1e-4, "BASELINE configs[2]: 131072x32768 X Y'/n + 1e-4 G (X,Y 100 cols, 1/sqrt(n)), k=100 p=10 q=2"),
    "c5": (262144, 32768, 272, 2, 512, 1e-6, "BASELINE configs[4]: 262144x32768 U512 diag(0.99^i) V512' + 1e-6 G, k=256 p=16 q=2"),
}
CHUNK = 4096  # rows per generation chunk (global matrix is independent of N)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-rpca", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the C1 / C2 / C5 records")
    p.add_argument("--e2e-steps", type=int, default=3)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def flop_estimate(m, n, ell, q):
    from paper_1906_04572_b200.sketch import flop_estimate as fe

    return fe(m, n, ell, q)


# ---------------------------------------------------------------- inputs
def gen_rows_device(torch, wl, lo, hi, device, seed=1234):
    """Rows [lo, hi) of the workload matrix, generated chunk by chunk with
    per-chunk seeds so the global matrix does not depend on the rank count."""
    m, n, ell, q, k, noise, _ = WORKLOADS[wl]
    out = torch.empty((hi - lo, n), dtype=torch.float64, device=device)
    g = torch.Generator(device=device)
    if wl in ("c1", "c3"):
        g.manual_seed(seed)
        y = torch.randn((n, k), generator=g, dtype=torch.float64, device=device)
        if wl == "c3":
            y /= math.sqrt(n)
        for c0 in range(lo - lo % CHUNK, hi, CHUNK):
            g.manual_seed(seed + 1 + c0 // CHUNK)
            rows = min(CHUNK, m - c0)
            x = torch.randn((rows, k), generator=g, dtype=torch.float64, device=device)
            if wl == "c3":
                x /= math.sqrt(n)
            blk = x @ y.T
            blk += noise * torch.randn((rows, n), generator=g, dtype=torch.float64, device=device)
            a0, a1 = max(lo, c0), min(hi, c0 + rows)
            out[a0 - lo:a1 - lo] = blk[a0 - c0:a1 - c0]
        return out
    if wl == "c2":
        g.manual_seed(seed)
        u = torch.linalg.qr(torch.randn((m, n), generator=g, dtype=torch.float64, device=device))[0]
        v = torch.linalg.qr(torch.randn((n, n), generator=g, dtype=torch.float64, device=device))[0]
        i = torch.arange(1, n + 1, dtype=torch.float64, device=device)
        sig = torch.where(i <= 40, torch.ones_like(i), 0.8 ** (i - 40))
        return ((u * sig) @ v.T)[lo:hi].contiguous()
    # c5 (BASELINE configs[4]): A = U512 diag(0.99^i) V512' + 1e-6 G, i = 1..512,
    # U512 (262144 x 512) and V512 (32768 x 512) orthonormal: QR of Gaussian
    # matrices on the device (cuSOLVER, deterministic); every rank forms the
    # full U512 (1 GB) and keeps its rows
    g.manual_seed(seed)
    vq = torch.linalg.qr(torch.randn((n, k), generator=g, dtype=torch.float64, device=device))[0]
    uq = torch.linalg.qr(torch.randn((m, k), generator=g, dtype=torch.float64, device=device))[0]
    sig = 0.99 ** torch.arange(1, k + 1, dtype=torch.float64, device=device)
    w = (vq * sig).T.contiguous()  # diag(sigma) V512'
    del vq
    for c0 in range(lo - lo % CHUNK, hi, CHUNK):
        g.manual_seed(seed + 1 + c0 // CHUNK)
        rows = min(CHUNK, m - c0)
        blk = uq[c0:c0 + rows] @ w
        blk += noise * torch.randn((rows, n), generator=g, dtype=torch.float64, device=device)
        a0, a1 = max(lo, c0), min(hi, c0 + rows)
        out[a0 - lo:a1 - lo] = blk[a0 - c0:a1 - c0]
    del uq, w
    return out


# ---------------------------------------------------------------- clocks
REASONS = ["gpu_idle", "applications_clocks_setting", "sw_power_cap", "hw_slowdown", "sync_boost",
           "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_power_brake_slowdown",
           "display_clock_setting"]


class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                mask = int(parts[3], 16) if parts[3].startswith("0x") else int(parts[3])
            except ValueError:
                continue
            for bit, name in enumerate(REASONS):
                if mask & (1 << bit) and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- helpers
def measured_dgemm_tflops(torch, device):
    """Live FP64 roofline denominator: cuBLAS DGEMM 8192^3, best of 5."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device=device)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=device)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * 8192 ** 3 / best / 1e9


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(p.read_text())
    except (OSError, ValueError):
        return {}


def ncu_traffic(wl):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/ncu_summary.json), if one matches this workload."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        return d.get("traffic_bytes_per_launch", {}).get(wl)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------- reference arm
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def all_blas_threads():
    """BLAS thread pool sized to every usable host core (torchrun exports
    OMP_NUM_THREADS=1 to each rank, which would starve the CPU arm)."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(limits=host_cores(), user_api="blas")


def load_reference():
    """The unmodified reference package installed in baseline/_ref (pip
    install --target baseline/_ref /root/reference/pkg), or None."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "corutv" / "__init__.py").exists():
        return None
    if str(ref_dir) not in sys.path:
        sys.path.insert(0, str(ref_dir))
    try:
        import corutv
    except ImportError:
        return None
    if not str(getattr(corutv, "__file__", "")).startswith(str(ref_dir)):
        return None
    return corutv


def reference_corutv(ell, q):
    """(callable(a) -> |diag T|, kind, label): the reference's own corutv
    (sketch.py:182-208) from baseline/_ref with the seeded Omega of
    SketchConfig(seed=0); the oracle port only if the install is missing."""
    ref = load_reference()
    if ref is not None:
        cfg = ref.SketchConfig(ell=ell, q_power=q, seed=0)
        return (lambda a: np.abs(np.diag(ref.corutv(a, cfg).t))), "reference", \
            "the reference package (baseline/_ref corutv.corutv, unmodified, numpy/OpenBLAS)"
    import oracle as O

    return (lambda a: np.abs(np.diag(O.corutv(a, ell, q, seed=0)["t"]))), "port", \
        "oracle (numpy restatement of corutv; baseline/_ref missing)"


def host_matrix(wl, lo=0, hi=None):
    """Rows [lo, hi) of the workload matrix as a host numpy array, generated
    by the SAME device generator as the b200 arm (so both arms factor the
    identical A), copied down in chunks.  Input generation only."""
    import torch

    m, n = WORKLOADS[wl][:2]
    hi = m if hi is None else hi
    dev = torch.device("cuda", 0)
    a_dev = gen_rows_device(torch, wl, lo, hi, dev)
    out = np.empty((hi - lo, n), dtype=np.float64)
    step = max(1, (1 << 30) // (8 * n))
    for r0 in range(0, hi - lo, step):
        out[r0:r0 + step] = a_dev[r0:r0 + step].cpu().numpy()
    del a_dev
    torch.cuda.empty_cache()
    return out


def bench_config(wl):
    """The workload description both arms print (identical dicts, so the
    driver can match them); how the b200 arm sharded it is reported under
    the line's "sharding" key."""
    m, n, ell, q, *_ = WORKLOADS[wl]
    l2_resident = 8 * m * n < 2 * 126 * 2 ** 20
    return {"workload": wl, "desc": WORKLOADS[wl][6], "m": m, "n": n, "ell": ell, "q": q,
            "variant": "exact-d",
            "l2": ("L2 flushed between steps (512 MB write), steps timed individually (A = %.3f GB)"
                   % (8 * m * n / 1e9)) if l2_resident else
                  "inputs larger than L2 (A = %.1f GB)" % (8 * m * n / 1e9),
            "flops_per_step": flop_estimate(m, n, ell, q),
            "omega": "gaussian_matrix(n, ell, seed 0) (numpy PCG64)",
            "matrix": "bench.gen_rows_device(%r), seed 1234" % wl}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU corutv on the FULL workload
    matrix (the b200 arm's A, identical: same device generator; the same
    seeded Omega), all host cores, K timed steps.  The W warm-up steps run
    on the first 1/8 of the rows (they only page in code and BLAS pools; a
    full-size warm-up would double the CPU arm's ~1 min/step run time)."""
    if rank != 0:
        return 0
    _pool = all_blas_threads()  # noqa: F841  (held for the run)
    wl = args.workload
    m, n, ell, q, *_ = WORKLOADS[wl]
    a = host_matrix(wl)
    run, kind, label = reference_corutv(ell, q)
    for _ in range(args.warmup):
        run(a[: max(n, m // 8)])
    times = []
    d = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        d = run(a)
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    val = flop_estimate(m, n, ell, q) / t / 1e9
    cores = host_cores()
    line = {
        "impl": "reference", "metric": "corutv_gflops", "value": round(val, 3), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(wl),
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": cores, "kind": kind,
                         "sample": f"{label}: corutv(A, SketchConfig(ell={ell}, q_power={q}, seed=0)) on the full "
                                   f"{m}x{n} {wl} matrix (the b200 arm's A), mean of {args.steps} runs "
                                   f"({min(times):.1f}-{max(times):.1f} s); {args.warmup} warm-up runs on "
                                   f"the first {max(n, m // 8)} rows"},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "check": {"diag_t_abs_head": [float(x) for x in d[:4]], "diag_t_abs_sum": float(d.sum())},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- device arm
def time_steps(torch, h, stream, step, a, omega, steps, l2_resident):
    """K steps of `step(a, omega)` on CUDA events (the library's stream):
    back to back for inputs larger than L2, else each step on its own events
    with L2 flushed (512 MB write) outside them.  Returns (ms/step, last)."""
    f = None
    if not l2_resident:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            f = step(a, omega)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps, f
    flush = torch.empty(2 ** 26, dtype=torch.float64, device=a.device)
    evs = []
    for _ in range(steps):
        flush.fill_(0.0)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        f = step(a, omega)
        b1.record(stream)
        evs.append((b0, b1))
    torch.cuda.synchronize()
    return sum(b0.elapsed_time(b1) for b0, b1 in evs) / steps, f


def roofline_time(m, n, ell, q, peak_tflops, bw_gbs):
    """Lower bound of one CoR-UTV: each of the 2q+3 A sweeps needs
    max(2 m n ell / P, 8 m n / BW)."""
    sweep = max(2.0 * m * n * ell / (peak_tflops * 1e12), 8.0 * m * n / (bw_gbs * 1e9))
    return (2 * q + 3) * sweep


def extra_workload(torch, P, h, device, wl, steps, warmup, peak, bw):
    """One more BASELINE config measured in the same run (N = 1): ms/step,
    GFLOP/s, roofline fraction."""
    m, n, ell, q, *_ = WORKLOADS[wl]
    a = gen_rows_device(torch, wl, 0, m, device)
    omega = torch.from_numpy(P.gaussian_matrix(n, ell, 0)).to(device)
    cfg = P.SketchConfig(ell=ell, q_power=q, seed=0)

    def step(x, om):
        return P.corutv(x, cfg, omega=om)

    for _ in range(warmup):
        step(a, omega)
    torch.cuda.synchronize()
    h.bind_stream()
    l2_resident = 8 * m * n < 2 * 126 * 2 ** 20
    h.lib.corutv_profile_begin(h.ptr)
    ms, f = time_steps(torch, h, torch.cuda.current_stream(device), step, a, omega, steps, l2_resident)
    prof = (ctypes.c_double * 12)()
    nl = ctypes.c_int64(0)
    h.lib.corutv_profile_end(h.ptr, prof, ctypes.byref(nl))
    fl = flop_estimate(m, n, ell, q)
    t_roof = roofline_time(m, n, ell, q, peak, bw)
    out = {"workload": wl, "desc": WORKLOADS[wl][6], "ms_per_step": round(ms, 4),
           "gflops": round(fl / (ms / 1e3) / 1e9, 3), "steps": steps, "warmup": warmup,
           "roofline": {"t_roofline_ms": round(t_roof * 1e3, 4), "frac": round(t_roof * 1e3 / ms, 4),
                        "bound": "tensor" if 2 * ell / 8 > peak * 1e3 / bw else "hbm",
                        "model": "(2q+3) x max(2 m n ell / P_fp64, 8 m n / BW_hbm)",
                        "sweep_gemm_ms_per_step": round(prof[3] / steps, 4),
                        "sweep_gemm_tflops": round(prof[5] / (prof[3] / 1e3) / 1e12, 3) if prof[3] > 0 else None},
           "l2": "flushed between steps (512 MB write), each step on its own events" if l2_resident
                 else "A larger than L2, steps back to back",
           "gpu_launches_per_step": round(nl.value / steps, 1),
           "check": {"diag_t_abs_head": [float(x) for x in f.t.diagonal().abs()[:4].cpu()]}}
    del a, f
    torch.cuda.empty_cache()
    return out


def tsr_record(torch, P, a, bw, ell=8, reps=3):
    """tsr_svd(a, ell) on the device-resident matrix, one pass over A (the
    default for ell <= 8) and two sweeps (CORUTV_DUAL_OFF=1): ms per call with
    CUDA events on the current stream; A is far larger than L2."""
    m, n = a.shape
    cfg = P.SketchConfig(ell=ell, seed=3)
    out = {"workload": "tsr_svd", "desc": f"tsr_svd (sketch.py:220-241) on the resident {m}x{n} matrix, ell={ell}",
           "a_bytes": 8 * m * n, "l2": "inputs larger than L2"}
    old = os.environ.get("CORUTV_DUAL_OFF")
    try:
        for key, off in (("one_pass", "0"), ("two_sweeps", "1")):
            os.environ["CORUTV_DUAL_OFF"] = off
            f = P.tsr_svd(a, cfg)  # warm-up (workspace)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                f = P.tsr_svd(a, cfg)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out[key] = {"ms_per_call": round(ms, 3), "sigma_0": float(f.sigma[0]),
                        "a_reads": 1 if off == "0" else 2}
        out["hbm_frac_one_pass"] = round(8.0 * m * n / (out["one_pass"]["ms_per_call"] * 1e-3) / (bw * 1e9), 4)
    finally:
        if old is None:
            os.environ.pop("CORUTV_DUAL_OFF", None)
        else:
            os.environ["CORUTV_DUAL_OFF"] = old
    return out


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    import torch
    import torch.distributed as tdist

    import paper_1906_04572_b200 as P
    from paper_1906_04572_b200 import _lib
    from paper_1906_04572_b200.dist import RowShardComm, corutv_sharded, row_range

    # one rank per GPU; CORUTV_BENCH_BACKEND=gloo (and more ranks than GPUs)
    # is only for dry runs of the multi-rank logic on a one-GPU box
    backend = os.environ.get("CORUTV_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=device)
        else:
            tdist.init_process_group(backend)
    wl = args.workload
    m, n, ell, q, *_ = WORKLOADS[wl]
    lo, hi = row_range(m, world, rank)
    a = gen_rows_device(torch, wl, lo, hi, device)
    omega_host = P.gaussian_matrix(n, ell, 0)
    omega = torch.from_numpy(omega_host).to(device)
    cfg = P.SketchConfig(ell=ell, q_power=q, seed=0)
    # NCCL ranks: the library's own communicator (every exchange an
    # ncclAllReduce on its stream); the gloo dry run keeps the callback
    comm = RowShardComm(native=(backend == "nccl")) if world > 1 else None
    h = _lib.handle(local)

    def step(x, om):
        if comm is not None:
            return corutv_sharded(x, cfg, comm, omega=om)
        return P.corutv(x, cfg, omega=om)

    def barrier():
        if world > 1:
            tdist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=device)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 0)):
        step(a, omega)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    h.bind_stream()
    h.lib.corutv_profile_begin(h.ptr)
    stream = torch.cuda.current_stream(device)
    # A per rank larger than twice the 126 MB L2: steps run back to back.
    # Smaller (C1, C2): every step is timed on its own events and L2 is
    # flushed between steps by writing a 512 MB buffer (outside the events).
    l2_resident = 8 * (hi - lo) * n < 2 * 126 * 2 ** 20
    ms_local, f = time_steps(torch, h, stream, step, a, omega, args.steps, l2_resident)
    barrier()
    torch.cuda.synchronize()
    prof = (ctypes.c_double * 12)()
    nl = ctypes.c_int64(0)
    h.lib.corutv_profile_end(h.ptr, prof, ctypes.byref(nl))
    clk = clocks.stop()
    ms = max_over_ranks(ms_local)
    flops = flop_estimate(m, n, ell, q)
    value = flops / (ms / 1e3) / 1e9
    bw = measured_peaks().get("hbm_gbs") or 6453.7

    # dominant kernel: the DMMA GEMMs that sweep A (K1 A*X, K2 A'*C1, K5 A*Q2)
    sweep_ms, sweep_n, sweep_fl = prof[3], prof[4], prof[5]
    other_ms = prof[6]
    result = {}
    peak = measured_dgemm_tflops(torch, device)
    if rank == 0:
        achieved = sweep_fl / (sweep_ms / 1e3) / 1e12 if sweep_ms > 0 else None
        result["roofline"] = {
            "bound": "tensor", "achieved": round(achieved, 3) if achieved else None,
            "peak": round(peak, 3), "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4) if achieved else None,
            "traffic": ncu_traffic(wl),
            "kernel": "gemm_kernel (TMA + DMMA.884 FP64; A sweeps K1/K2/K5)",
            "peak_source": "cuBLAS DGEMM 8192^3 (torch.matmul f64) measured in this run, best of 5; "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "algorithmic_flops_per_launch": round(sweep_fl / max(sweep_n, 1)),
            "launches": int(sweep_n), "avg_launch_ms": round(sweep_ms / max(sweep_n, 1), 4),
            "share_of_step": round(sweep_ms / (ms * args.steps), 4) if ms > 0 else None,
            "other_gemm_ms_per_step": round(other_ms / args.steps, 4),
            "hbm_bytes_per_launch": 8 * (hi - lo) * n,
            "hbm_peak_gbs": bw,
            "step_vs_roofline": round(roofline_time(m, n, ell, q, peak, bw) * 1e3 / ms, 4),
        }
    # parity spot-check of the measured result (size-independent property):
    # |A|^2 = |A - U T V'|^2 + |T|^2 for exact-d (U T V' = P1 A P2); and the
    # leading |diag T| (the reference arm prints the same for the same A)
    d_head = [float(x) for x in f.t.diagonal().abs()[:4].cpu()]
    check = {"t_fro2": float((f.t ** 2).sum()), "diag_t_abs_head": d_head,
             "diag_t_abs_sum": float(f.t.diagonal().abs().sum())}
    del f

    # ------------------------------------------------------------- CPU leg
    # the reference's own corutv (baseline/_ref) on the first 32768 rows of
    # the SAME A (C3: 1/4 of it, ~10-15 s on 16 cores); the full-size CPU run
    # is the reference arm (--impl reference)
    # tsr_svd's sketches on the same resident matrix: one pass over A (l <= 8,
    # csrc/dual_sketch.cuh, the reference's fused_sketch sketch.py:160-163)
    # against two DMMA sweeps -- a record next to the other workloads
    tsr = None
    if world == 1 and not args.no_extra:
        try:
            tsr = tsr_record(torch, P, a, bw)
        except Exception as exc:  # the headline line must still print
            tsr = {"workload": "tsr_svd", "error": str(exc)[:200]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rows = min(m, 32768)
        sample = a[:rows].cpu().numpy()
        run, kind, label = reference_corutv(ell, q)
        with all_blas_threads():
            t0 = time.perf_counter()
            run(sample)
            tc = time.perf_counter() - t0
        del sample
        cpu = {"value": round(flop_estimate(rows, n, ell, q) / tc / 1e9, 3), "unit": "GFLOP/s",
               "cores": host_cores(), "kind": kind,
               "sample": f"{label}: corutv on the first {rows} rows ({rows}x{n}) of the same {wl} matrix, "
                         f"ell={ell}, q={q}, seeded Omega, 1 run, {tc:.2f} s"}

    # ------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        try:
            a_host = torch.empty((hi - lo, n), dtype=torch.float64, pin_memory=True)
            a_host.copy_(a)
            del a
            torch.cuda.empty_cache()
            # public API exactly as a reference user calls it: corutv(a, cfg) with
            # the seeded Omega (drawn on the device, bit-identical to numpy)
            step(a_host, None)  # warm-up (allocations)
            torch.cuda.synchronize()
            barrier()
            k2 = max(1, args.e2e_steps)
            t0 = time.perf_counter()
            for _ in range(k2):
                fo = step(a_host, None)
                _ = fo.t[0, 0].item() if hasattr(fo.t, "item") else fo.t[0, 0]
            torch.cuda.synchronize()
            dt = max_over_ranks((time.perf_counter() - t0) / k2)
            e2e = {"value": round(flops / dt / 1e9, 3), "unit": "GFLOP/s",
                   "h2d_bytes_per_step": int(a_host.numel() * 8),
                   "d2h_bytes_per_step": int(((hi - lo) * ell + ell * ell + n * ell) * 8),
                   "ms_per_step": round(dt * 1e3, 3), "steps": k2,
                   "path": "paper_1906_04572_b200.corutv(pinned host tensor, SketchConfig(seed=0)) -> "
                           "corutv_decompose_host: A streamed H2D in 1 GiB row chunks, overlapped with the device "
                           "Omega (PCG64+ziggurat), C1 = A Omega per chunk and the split-K slices of C2 = A' C1; "
                           "then the resident sweeps; D2H of U,T,V via pinned staging"}
            # the case a reference user actually has: a pageable numpy array
            # (the library stages it through pinned buffers itself)
            try:
                a_np = np.empty(tuple(a_host.shape), dtype=np.float64)
                a_np[...] = a_host.numpy()
                del a_host
                step(a_np, None)
                torch.cuda.synchronize()
                barrier()
                t0 = time.perf_counter()
                for _ in range(k2):
                    fo = step(a_np, None)
                    _ = fo.t[0, 0]
                torch.cuda.synchronize()
                dtp = max_over_ranks((time.perf_counter() - t0) / k2)
                e2e["pageable"] = {"value": round(flops / dtp / 1e9, 3), "unit": "GFLOP/s",
                                   "ms_per_step": round(dtp * 1e3, 3), "steps": k2,
                                   "path": "paper_1906_04572_b200.corutv(pageable numpy array, SketchConfig(seed=0)) "
                                           "-> corutv_decompose_host (staged through pinned buffers)"}
                del a_np
            except (RuntimeError, MemoryError) as exc:
                e2e["pageable"] = {"value": None, "error": str(exc)[:200]}
            a_host = None
        except RuntimeError as exc:  # e.g. pinned allocation failure
            e2e = {"value": None, "unit": "GFLOP/s", "error": str(exc)[:200],
                   "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    else:
        del a
    torch.cuda.empty_cache()

    # ------------------------------------------------------------- RPCA (C4)
    rpca = None
    if not args.no_rpca and world == 1:
        rpca = bench_rpca(torch, P, device, peak=peak, bw=bw, cpu=(rank == 0 and not args.no_cpu))
    elif not args.no_rpca:
        try:
            rpca = bench_rpca(torch, P, device, world, rank, tdist, comm, peak=peak, bw=bw)
        except Exception as exc:  # the headline line must still print
            rpca = {"workload": "c4", "ranks": world, "error": str(exc)[:200]}

    # ------------------------------------------- the other BASELINE configs
    extra = None
    if world == 1 and not args.no_extra:
        extra = {}
        for x in ("c1", "c2", "c5"):
            if x == wl:
                continue
            try:
                extra[x] = extra_workload(torch, P, h, device, x, 20 if x != "c5" else 3,
                                          5 if x != "c5" else 1, peak, bw)
            except Exception as exc:  # the headline line must still print
                extra[x] = {"workload": x, "error": str(exc)[:200]}
        if tsr is not None:
            extra["tsr_svd_ell8"] = tsr

    if rank == 0:
        line = {
            "metric": "corutv_gflops", "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(wl),
            "sharding": {"parallelism": f"row-shard x{world}" if world > 1 else "single",
                         "rows_per_rank": hi - lo},
            "fp64_pct_of_peak": round(100 * value / 1e3 / peak, 2),
            "roofline": result["roofline"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(nl.value),
            "clocks": clk,
            "rpca": rpca,
            "workloads": extra,
            "check": check,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


def c4_matrix(torch, device):
    """BASELINE configs[3] (C4): M = X Y' + S, n = 10000, X, Y 10000 x 50
    N(0, 1/10000), 5% spikes U[-500, 500] at uniform positions."""
    n, k = 10000, 50
    g = torch.Generator(device=device)
    g.manual_seed(777)
    x = torch.randn((n, k), generator=g, dtype=torch.float64, device=device) / 100.0
    y = torch.randn((n, k), generator=g, dtype=torch.float64, device=device) / 100.0
    mat = x @ y.T
    nnz = n * n // 20
    pos = torch.randperm(n * n, generator=g, device=device)[:nnz]
    vals = (torch.rand((nnz,), generator=g, dtype=torch.float64, device=device) * 1000.0) - 500.0
    mat.view(-1)[pos] += vals
    return mat


def rpca_roofline(n, q, sol, snorm_iters, peak, bw):
    """Lower bounds (seconds) of the C4 solve and of mu0 from the run's own
    histories: per iteration the 2q+3 sweeps of G at ell_j (each
    max(2 n^2 ell / P, 8 n^2 / BW)) plus the fused update (read M, Y, write
    S, Y, G: 40 B/element, and 2 r n^2 flops); per spectral-norm iteration
    two b = 24 sweeps."""
    P_, B_ = peak * 1e12, bw * 1e9
    t = 0.0
    for ell, r in zip(sol.ell_history, sol.rank_history):
        t += (2 * q + 3) * max(2.0 * n * n * ell / P_, 8.0 * n * n / B_)
        t += max(2.0 * n * n * r / P_, 40.0 * n * n / B_)
    t_mu0 = snorm_iters * 2 * max(2.0 * n * n * 24 / P_, 8.0 * n * n / B_)
    return t, t_mu0


def rpca_cpu_baseline(mat_host, lam, mu0, iters=3):
    """The reference's own solver (baseline/_ref rpca.alm_corutv, else the
    oracle port) on the same M, all host cores: its spectral norm (mu0) in
    full, and the first `iters` ALM iterations as a bounded sample (the full
    30-iteration solve is ~3 min of 16-core time)."""
    ref = load_reference()
    with all_blas_threads():
        t0 = time.perf_counter()
        if ref is not None:
            ref.dense.spectral_norm(mat_host)
        else:
            import oracle as O

            O.spectral_norm(mat_host)
        t_snorm = time.perf_counter() - t0
        t0 = time.perf_counter()
        try:
            if ref is not None:
                ref.alm_corutv(mat_host, ref.AlmConfig(lam=lam, tol=1e-7, ell=100, q_power=1, seed=0, mu0=mu0,
                                                       max_iter=iters))
            else:
                import oracle as O

                O.alm_corutv(mat_host, ell=100, lam=lam, mu0=mu0, tol=1e-7, q_power=1, seed=0, max_iter=iters)
        except Exception:  # ConvergenceError after `iters` iterations: the sample ends here
            pass
        t_alm = time.perf_counter() - t0
    kind = "reference" if ref is not None else "port"
    label = "the reference package (baseline/_ref)" if ref is not None else "oracle port"
    return {"ms_per_iter": round(1e3 * t_alm / iters, 1), "unit": "ms/iter", "cores": host_cores(), "kind": kind,
            "spectral_norm_s": round(t_snorm, 2),
            "sample": f"{label}: alm_corutv on the same C4 M, first {iters} iterations (caps 100, 600, 1: the "
                      f"costliest and a cheap one) of the 30, {t_alm:.1f} s; spectral_norm (mu0) in full"}


def bench_rpca(torch, P, device, world=1, rank=0, tdist=None, comm=None, peak=35.4, bw=6453.7, cpu=False):
    """BASELINE configs[3] (C4): lam = 1/sqrt(n), tol = 1e-7, ell0 = 2k =
    100, q = 1.  mu0 = 1.25/|M|_2 is timed separately (spectral_norm) and
    passed in.  world > 1: M row-sharded over the ranks
    (dist.alm_corutv_sharded; every rank builds the same M and keeps its
    rows), wall time the max over ranks."""
    n, k = 10000, 50
    mat = c4_matrix(torch, device)
    mat_host = mat.cpu().numpy() if cpu else None
    if world > 1:
        from paper_1906_04572_b200.dist import alm_corutv_sharded, row_range

        lo, hi = row_range(n, world, rank)
        mat = mat[lo:hi].contiguous()
        h = P._lib.handle(device.index)
        comm.attach(h, n)
        try:
            torch.cuda.synchronize()
            tdist.barrier()
            t0 = time.perf_counter()
            snorm, sit = P.dense.spectral_norm_iters(mat)
            t_snorm = time.perf_counter() - t0
        finally:
            comm.detach(h)
        cfg = P.AlmConfig(lam=1 / math.sqrt(n), tol=1e-7, ell=2 * k, q_power=1, seed=0, mu0=1.25 / snorm)

        def solve():
            return alm_corutv_sharded(mat, cfg, comm, n)
    else:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        snorm, sit = P.dense.spectral_norm_iters(mat)
        t_snorm = time.perf_counter() - t0
        cfg = P.AlmConfig(lam=1 / math.sqrt(n), tol=1e-7, ell=2 * k, q_power=1, seed=0, mu0=1.25 / snorm)

        def solve():
            return P.alm_corutv(mat, cfg)
    # warm-up solve (lazy kernel loading, workspace growth), then the timed one
    solve()
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    t0 = time.perf_counter()
    sol = solve()
    torch.cuda.synchronize()
    t_alm = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t_alm, t_snorm], dtype=torch.float64, device=device)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_alm, t_snorm = float(tt[0]), float(tt[1])
    t_roof, t_roof_mu0 = rpca_roofline(n, 1, sol, sit, peak, bw)
    out = {"workload": "c4", "n": n, "ms_per_iter": round(1e3 * t_alm / sol.iterations, 3),
           "iterations": sol.iterations, "alm_total_s": round(t_alm, 3),
           "spectral_norm_s": round(t_snorm, 3), "spectral_norm_iters": sit,
           "spectral_norm_ms_per_iter": round(1e3 * t_snorm / max(sit, 1), 4),
           "rank_of_l": sol.rank_of_l, "nnz_of_s": sol.nnz_of_s,
           "final_residual": sol.residuals[-1], "ell_history": sol.ell_history,
           "rank_history": sol.rank_history,
           "ranks": world,
           "roofline": {"t_roofline_s": round(t_roof, 4), "frac": round(t_roof / t_alm, 4),
                        "mu0_t_roofline_s": round(t_roof_mu0, 4), "mu0_frac": round(t_roof_mu0 / t_snorm, 4),
                        "model": "per iteration (2q+3) max(2 n^2 ell_j / P, 8 n^2 / BW) + max(2 r_j n^2 / P, "
                                 "40 n^2 / BW); mu0: 2 max(2 n^2 24 / P, 8 n^2 / BW) per power iteration; "
                                 "P = in-run cuBLAS DGEMM, BW = MEASURED_PEAKS hbm_gbs"},
           "timing": "wall clock around alm_corutv (host decisions included), sync on both sides, "
                     "after one untimed warm-up solve" + ("; row-sharded, max over ranks" if world > 1 else "")}
    del mat, sol
    torch.cuda.empty_cache()
    if mat_host is not None:
        out["cpu_baseline"] = rpca_cpu_baseline(mat_host, 1 / math.sqrt(n), 1.25 / snorm)
        del mat_host
    return out


if __name__ == "__main__":
    sys.exit(main())
