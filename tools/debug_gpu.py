"""Quick device checks used while bringing up kernels (prints, no asserts)."""
import sys, time, traceback
sys.path.insert(0, '.')
import numpy as np, torch, ctypes
import paper_1906_04572_b200 as P
from paper_1906_04572_b200 import _lib
import oracle as O

torch.cuda.set_device(0)
h = _lib.handle(0)
rng = np.random.Generator(np.random.PCG64(1))
def gemm(trans, M, N, K):
    a = rng.standard_normal((K, M) if trans else (M, K)); b = rng.standard_normal((K, N))
    A = torch.from_numpy(a).cuda(); B = torch.from_numpy(b).cuda(); C = torch.zeros((M, N), dtype=torch.float64, device='cuda')
    h.call("corutv_gemm", trans, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(), C.stride(0))
    torch.cuda.synchronize()
    ref = (a.T if trans else a) @ b
    err = np.abs(C.cpu().numpy() - ref).max() / max(1e-300, np.abs(ref).max())
    return err
for trans in (0, 1):
    for (M, N, K) in ((1, 1, 1), (7, 3, 5), (128, 16, 16), (130, 15, 33), (1000, 15, 1000), (4000, 50, 3000), (3000, 50, 4000), (520, 110, 700), (300, 272, 513), (64, 600, 200)):
        try:
            print("gemm trans", trans, (M, N, K), "relerr %.2e" % gemm(trans, M, N, K), flush=True)
        except Exception as e:
            traceback.print_exc(); break
z = np.load('tests/golden/golden.npz')
for name in ("cu_replay", "cu_rank8_q0", "cu_rank8_q2", "cu_noisy_q1", "cu_full_ell", "cu_ell1", "cu_c2small_q2", "cu_rank8_q2_approx"):
    try:
        a = z[f"{name}/a"]; t = z[f"{name}/t"]; ell = t.shape[0]; om = z[f"{name}/omega"]
        q = {"cu_replay": 1, "cu_rank8_q0": 0, "cu_rank8_q2": 2, "cu_rank8_q2_approx": 2, "cu_noisy_q1": 1, "cu_full_ell": 1, "cu_ell1": 1, "cu_c2small_q2": 2}[name]
        var = "approx-d" if "approx" in name else "exact-d"
        cnt = P.PassCounter()
        f = P.corutv(a, P.SketchConfig(ell=ell, q_power=q, variant=var), cnt, omega=om)
        dd = np.abs(np.abs(np.diag(f.t)) - np.abs(np.diag(t))).max() / np.abs(t).max()
        err = np.linalg.norm(a - f.lowrank()); errref = float(z[f"{name}/err"])
        orth = np.abs(f.u.T @ f.u - np.eye(ell)).max()
        print(name, "passes", cnt.passes, int(z[f"{name}/passes"]), "diag %.2e" % dd, "err %.3e ref %.3e" % (err, errref), "orth %.1e" % orth, flush=True)
    except Exception:
        traceback.print_exc()
for name in ("snorm_block", "snorm_direct"):
    try:
        v, it = P.dense.spectral_norm_iters(z[f"{name}/a"]); print(name, v, float(z[f"{name}/val"]), it)
    except Exception:
        traceback.print_exc()
try:
    print("sv", np.abs(P.singular_values(z["sv/a"]) - z["sv/sig"]).max())
except Exception:
    traceback.print_exc()
for n in (60, 100):
    try:
        m = z[f"alm_n{n}/m"]; k = max(1, round(0.05*n)); cs = {60: 11, 100: 5}[n]
        sol = P.alm_corutv(m, P.AlmConfig(ell=2*k, q_power=1, seed=cs))
        print("alm", n, sol.iterations, int(z[f"alm_n{n}/iterations"]), "L err %.2e" % (np.linalg.norm(sol.l - z[f"alm_n{n}/l"]) / np.linalg.norm(z[f"alm_n{n}/l"])), sol.rank_of_l, int(z[f"alm_n{n}/rank_of_l"]), sol.ell_history == list(z[f"alm_n{n}/ell_history"]))
    except Exception:
        traceback.print_exc()
# timing of C2-like and a C3-like sharded size
for (m, n, ell, q) in ((4000, 3000, 50, 1), (32768, 32768, 110, 2)):
    A = torch.randn(m, n, dtype=torch.float64, device='cuda')
    cfg = P.SketchConfig(ell=ell, q_power=q)
    om = torch.from_numpy(P.gaussian_matrix(n, ell, 0)).cuda()
    P.corutv(A, cfg, omega=om); torch.cuda.synchronize()
    t0 = time.perf_counter(); 
    for _ in range(3): P.corutv(A, cfg, omega=om)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
    print("corutv", (m, n, ell, q), "%.3f ms" % (dt * 1e3), "%.1f GFLOP/s" % (P.flop_estimate(m, n, ell, q) / dt / 1e9), flush=True)
    # raw gemm speed
    X = torch.randn(n, ell, dtype=torch.float64, device='cuda'); C = torch.empty(m, ell, dtype=torch.float64, device='cuda')
    Y = torch.randn(m, ell, dtype=torch.float64, device='cuda'); C2 = torch.empty(n, ell, dtype=torch.float64, device='cuda')
    for trans, BB, CC, MM in ((0, X, C, m), (1, Y, C2, n)):
        h.call("corutv_gemm", trans, MM, ell, (n if trans == 0 else m), A.data_ptr(), A.stride(0), BB.data_ptr(), BB.stride(0), CC.data_ptr(), CC.stride(0))
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            h.call("corutv_gemm", trans, MM, ell, (n if trans == 0 else m), A.data_ptr(), A.stride(0), BB.data_ptr(), BB.stride(0), CC.data_ptr(), CC.stride(0))
        e1.record(); e1.synchronize(); ms = e0.elapsed_time(e1) / 5
        print("  gemm trans", trans, "%.3f ms %.2f TFLOP/s" % (ms, 2 * m * n * ell / ms / 1e9), flush=True)
