"""Generate golden vectors from the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``corutv`` from /root/reference/pkg/src (read-only), runs the
reference functions on seeded inputs and writes ``tests/golden/golden.npz``.
The GPU box never runs this script; tests only read the committed .npz.
Every case records the reference call it came from.
"""

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
import corutv as ref  # noqa: E402
from corutv import dense as rdense, rpca as rrpca, sketch as rsketch, synth as rsynth  # noqa: E402

out = {}
meta = {"numpy": np.__version__, "cases": {}}


def put(name, what, **arrs):
    meta["cases"][name] = what
    for k, v in arrs.items():
        out[f"{name}/{k}"] = np.asarray(v)


def rank_k(seed, m, n, k, scale=1.0):  # pkg/tests/test_sketch.py:21-23
    rng = np.random.Generator(np.random.PCG64(seed))
    return scale * rng.standard_normal((m, k)) @ rng.standard_normal((k, n))


# ---- householder_qr (dense.py:132) ------------------------------------
for seed in range(3):
    a = np.random.Generator(np.random.PCG64(seed)).standard_normal((50, 10))
    f = rdense.householder_qr(a)
    put(f"qr{seed}", "dense.householder_qr(PCG64(seed).standard_normal((50,10)))", a=a, q=f.q, r=f.r)

# ---- qrcp (dense.py:152) ------------------------------------------------
for name, a in {
    "qrcp_diag": np.diag([1.0, 3.0, 2.0]),                       # test_dense.py:97-100
    "qrcp_tie": np.array([[2.0, 1.0, 2.0], [0.0, 0.5, 0.0]]),    # test_dense.py:103-107
    "qrcp_rand": np.random.Generator(np.random.PCG64(100)).standard_normal((25, 18)),
    "qrcp_square": np.random.Generator(np.random.PCG64(101)).standard_normal((40, 40)),
    "qrcp_rank5": (lambda g: g.standard_normal((30, 5)) @ g.standard_normal((5, 30)))(
        np.random.Generator(np.random.PCG64(20240917))),
}.items():
    f = rdense.qrcp(a)
    put(name, "dense.qrcp", a=a, q=f.q, r=f.r, perm=f.perm)

# ---- singular values / pinv / spectral norm -----------------------------
g = np.random.Generator(np.random.PCG64(7))
a = g.standard_normal((12, 20))
put("sv", "dense.singular_values", a=a, sig=rdense.singular_values(a))
a = g.standard_normal((9, 9))
put("pinv", "dense.pseudoinverse", a=a, pinv=rdense.pseudoinverse(a))
a = g.standard_normal((120, 90))
put("snorm_block", "dense.spectral_norm (block power path)", a=a, val=rdense.spectral_norm(a))
a = g.standard_normal((50, 40))
put("snorm_direct", "dense.spectral_norm (Jacobi path)", a=a, val=rdense.spectral_norm(a))

# ---- gaussian_matrix (sketch.py:63) -------------------------------------
put("omega", "sketch.gaussian_matrix(30, 7, 12345)", val=rsketch.gaussian_matrix(30, 7, 12345))

# ---- corutv (sketch.py:182) ---------------------------------------------
cases = [
    ("cu_replay", rank_k(17, 60, 50, 5), 12, 1, 123, "exact-d"),       # test_sketch.py:73-79
    ("cu_rank8_q0", rank_k(3, 200, 150, 8), 20, 0, 5, "exact-d"),      # test_sketch.py:50-57
    ("cu_rank8_q2", rank_k(3, 200, 150, 8), 20, 2, 5, "exact-d"),
    ("cu_rank8_q2_approx", rank_k(3, 200, 150, 8), 20, 2, 5, "approx-d"),
    ("cu_noisy_q1", rsynth.gen_noisy_lowrank(rsynth.NoisyLowRankSpec(n=120, k=8, seed=21))[0], 16, 1, 9, "exact-d"),
    ("cu_full_ell", rank_k(5, 40, 24, 24), 24, 1, 2, "exact-d"),         # ell == min(m, n)
    ("cu_ell1", rank_k(6, 70, 30, 3), 1, 1, 3, "exact-d"),
]
# C2-shaped at reduced size: orthonormal factors, sigma_i = 1 (i<=40), 0.8^(i-40)
g = np.random.Generator(np.random.PCG64(4242))
uu = np.linalg.qr(g.standard_normal((400, 300)))[0]
vv = np.linalg.qr(g.standard_normal((300, 300)))[0]
sig = np.where(np.arange(1, 301) <= 40, 1.0, 0.8 ** (np.arange(1, 301) - 40))
cases.append(("cu_c2small_q2", (uu * sig) @ vv.T, 50, 2, 77, "exact-d"))
for name, a, ell, q, seed, variant in cases:
    cnt = rsketch.PassCounter()
    f = rsketch.corutv(a, rsketch.SketchConfig(ell=ell, q_power=q, seed=seed, variant=variant), cnt)
    err = rsketch.corutv_lowrank_error(a, rsketch.SketchConfig(ell=ell, q_power=q, seed=seed, variant=variant))
    put(name, f"sketch.corutv(a, SketchConfig(ell={ell}, q_power={q}, seed={seed}, variant={variant!r}))",
        a=a, u=f.u, t=f.t, v=f.v, passes=cnt.passes, err=err,
        omega=rsketch.gaussian_matrix(a.shape[1], ell, seed),
        flops=rsketch.flop_estimate(a.shape[0], a.shape[1], ell, q, variant))

# ---- jacobi_svd (dense.py:357), sor_svd / tsr_svd (sketch.py:220-262) ------
g = np.random.Generator(np.random.PCG64(31))
for name, a in {
    "svd_tall": g.standard_normal((15, 9)),
    "svd_wide": g.standard_normal((7, 12)),
    "svd_square": g.standard_normal((10, 10)),
    "svd_zero_cols": np.diag([3.0, 0.0, 2.0, 0.0, 1.0]),          # zero-sigma completion
}.items():
    f = rdense.jacobi_svd(a)
    put(name, "dense.jacobi_svd", a=a, u=f.u, sigma=f.sigma, v=f.v)
svd_cases = [
    ("sor_q1", "sor", rank_k(41, 120, 80, 7), 14, 1, 8, "exact-d"),
    ("sor_q0_approx", "sor", rank_k(42, 90, 60, 5), 10, 0, 3, "approx-d"),
    ("sor_c2small", "sor", (uu * sig) @ vv.T, 50, 2, 77, "exact-d"),
    ("tsr_tall", "tsr", rank_k(43, 80, 60, 6), 12, 0, 4, "exact-d"),
    ("tsr_wide", "tsr", rank_k(44, 50, 90, 5), 10, 0, 6, "exact-d"),
    ("tsr_noisy", "tsr", rsynth.gen_noisy_lowrank(rsynth.NoisyLowRankSpec(n=100, k=6, seed=22))[0], 20, 0, 1, "exact-d"),
]
for name, kind, a, ell, q, seed, variant in svd_cases:
    cnt = rsketch.PassCounter()
    cfg = rsketch.SketchConfig(ell=ell, q_power=q, seed=seed, variant=variant)
    f = (rsketch.sor_svd if kind == "sor" else rsketch.tsr_svd)(a, cfg, cnt)
    put(name, f"sketch.{kind}_svd(a, SketchConfig(ell={ell}, q_power={q}, seed={seed}, variant={variant!r}))",
        a=a, u=f.u, sigma=f.sigma, v=f.v, passes=cnt.passes)

# ---- ALM-CoRUTV (rpca.py:237) -------------------------------------------
def instance(n, seed):  # test_rpca.py:104-108
    k = max(1, round(0.05 * n))
    s = round(0.05 * n * n)
    return (k, s) + rsynth.gen_rpca_instance(rsynth.RpcaInstanceSpec(n=n, k=k, s=s, seed=seed))

for n, seed, cseed in ((60, 7, 11), (100, 3, 5)):
    k, s, m, l0, s0 = instance(n, seed)
    cfg = rrpca.AlmConfig(ell=2 * k, q_power=1, seed=cseed)
    sol = rrpca.alm_corutv(m, cfg)
    mu0 = 1.25 / rdense.spectral_norm(m)
    put(f"alm_n{n}", f"rpca.alm_corutv(gen_rpca_instance(n={n}, seed={seed}), AlmConfig(ell={2*k}, q_power=1, seed={cseed}))",
        m=m, l=sol.l, s=sol.s, iterations=sol.iterations, residuals=sol.residuals,
        rank_of_l=sol.rank_of_l, nnz_of_s=sol.nnz_of_s, rank_history=sol.rank_history,
        nnz_history=sol.nnz_history, mu_history=sol.mu_history, ell_history=sol.ell_history, mu0=mu0)

# desk scale n=400 (test_rpca.py:160-173): histories + support only (M is regenerated)
k, s, m, l0, s0 = instance(400, 0)
sol = rrpca.alm_corutv(m, rrpca.AlmConfig(ell=2 * k, q_power=1, seed=1))
put("alm_n400", "rpca.alm_corutv(gen_rpca_instance(n=400, seed=0), AlmConfig(ell=40, q_power=1, seed=1)); M regenerated by oracle.gen_rpca_instance",
    iterations=sol.iterations, residuals=sol.residuals, rank_of_l=sol.rank_of_l, nnz_of_s=sol.nnz_of_s,
    rank_history=sol.rank_history, nnz_history=sol.nnz_history, mu_history=sol.mu_history,
    ell_history=sol.ell_history, l_norm=np.linalg.norm(sol.l), s_norm=np.linalg.norm(sol.s),
    m_sum=m.sum(), m_norm=np.linalg.norm(m),
    s_support=np.flatnonzero(np.abs(sol.s) > 1e-12).astype(np.int32),
    l_sample=sol.l[::37, ::41], s_sample=sol.s[::37, ::41])

# ---- warm-started Jacobi SVD (dense.py:313-376, v_init) ------------------
g = np.random.Generator(np.random.PCG64(31))
a = g.standard_normal((24, 24))
v0 = rdense.jacobi_svd(a + 1e-3 * g.standard_normal((24, 24))).v
f = rdense.jacobi_svd(a, v_init=v0)
put("svdwarm_sq", "dense.jacobi_svd(a, v_init=jacobi_svd(a + 1e-3 E).v), 24x24", a=a, v_init=v0, u=f.u,
    sigma=f.sigma, v=f.v)
a = g.standard_normal((30, 17))
v0 = rdense.jacobi_svd(a + 1e-3 * g.standard_normal((30, 17))).v
f = rdense.jacobi_svd(a, v_init=v0)
put("svdwarm_tall", "dense.jacobi_svd(a, v_init=...), 30x17 (odd width: pad column)", a=a, v_init=v0, u=f.u,
    sigma=f.sigma, v=f.v)
a = g.standard_normal((13, 29))
v0 = rdense.jacobi_svd(a.T + 1e-3 * g.standard_normal((29, 13))).v
f = rdense.jacobi_svd(a, v_init=v0)
put("svdwarm_wide", "dense.jacobi_svd(a, v_init=...), 13x29 (v_init: right factor of a')", a=a, v_init=v0,
    u=f.u, sigma=f.sigma, v=f.v)

# ---- svt (rpca.py:135-158) -------------------------------------------------
g = np.random.Generator(np.random.PCG64(41))
for name, b, delta in (("svt_diag", np.diag([3.0, 1.0]), 2.0),          # test_rpca.py:52-55
                       ("svt_zero", g.standard_normal((6, 5)), 0.0),    # test_rpca.py:58-62
                       ("svt_nuc", g.standard_normal((20, 20)), 1.5),   # test_rpca.py:65-72
                       ("svt_wide", g.standard_normal((9, 16)), 0.8),
                       ("svt_rank", rank_k(42, 40, 40, 4) + 1e-3 * g.standard_normal((40, 40)), 0.5)):
    mat, r = rrpca.svt(b, delta)
    put(name, f"rpca.svt(b, {delta})", b=b, delta=delta, mat=mat, r=r)

# ---- InexactALM baseline (rpca.py:258-273) ---------------------------------
for n, seed in ((60, 7), (100, 3)):
    k, s, m, l0, s0 = instance(n, seed)
    sol = rrpca.inexact_alm(m, rrpca.AlmConfig(ell=2 * k))
    put(f"ialm_n{n}", f"rpca.inexact_alm(gen_rpca_instance(n={n}, seed={seed}), AlmConfig(ell={2*k}))",
        m=m, l=sol.l, s=sol.s, iterations=sol.iterations, residuals=sol.residuals,
        rank_of_l=sol.rank_of_l, nnz_of_s=sol.nnz_of_s, rank_history=sol.rank_history,
        nnz_history=sol.nnz_history, mu_history=sol.mu_history, ell_history=sol.ell_history)
k, s, m, l0, s0 = instance(80, 3)  # test_rpca.py:139-143: max_iter error carries the history
try:
    rrpca.inexact_alm(m, rrpca.AlmConfig(max_iter=2))
except rdense.ConvergenceError as exc:
    put("ialm_maxiter", "rpca.inexact_alm(gen_rpca_instance(n=80, seed=3), AlmConfig(max_iter=2)) -> ConvergenceError",
        m=m, history=exc.history, residual=exc.residual)
# desk scale n=400 (test_rpca.py:176-180): histories + support only
k, s, m, l0, s0 = instance(400, 0)
sol = rrpca.inexact_alm(m, rrpca.AlmConfig(ell=2 * k))
put("ialm_n400", "rpca.inexact_alm(gen_rpca_instance(n=400, seed=0), AlmConfig(ell=40)); M regenerated by oracle.gen_rpca_instance",
    iterations=sol.iterations, residuals=sol.residuals, rank_of_l=sol.rank_of_l, nnz_of_s=sol.nnz_of_s,
    rank_history=sol.rank_history, nnz_history=sol.nnz_history, mu_history=sol.mu_history,
    ell_history=sol.ell_history, m_sum=m.sum(),
    s_support=np.flatnonzero(np.abs(sol.s) > 1e-12).astype(np.int32),
    l_sample=sol.l[::37, ::41], s_sample=sol.s[::37, ::41])

# ---- experiment harness (bench.py:165-306) -------------------
from corutv import bench as rbench  # noqa: E402

for exp in ("sv-compare", "lowrank-error"):
    cfg = rbench.ExperimentConfig(experiment=exp, n=80, k=6, trials=3, q_power=1,
                                  methods=("svd", "qrcp", "utv-approx", "corutv", "tsr-svd", "sor-svd"))
    rows = (rbench.run_sv_compare if exp == "sv-compare" else rbench.run_lowrank_error)(cfg)
    cols = list(zip(*rows))
    put(f"harness_{exp.replace('-', '_')}",
        f"bench.run_{exp.replace('-', '_')}(ExperimentConfig({exp!r}, n=80, k=6, trials=3, q_power=1, all methods))",
        c0=np.array(cols[0]), method=np.array(cols[1]), c2=np.array(cols[2]), c3=np.array(cols[3]),
        c4=np.array(cols[4]))
a_h, _ = rsynth.gen_noisy_lowrank(rsynth.NoisyLowRankSpec(n=80, k=6, seed=0, noise_coeff=0.1))
a_0, _ = rsynth.gen_noisy_lowrank(rsynth.NoisyLowRankSpec(n=50, k=4, seed=3, noise_coeff=0.0))
put("synth_noisy", "synth.gen_noisy_lowrank(NoisyLowRankSpec(n=80, k=6, seed=0)) and (n=50, k=4, seed=3, noise 0)",
    a=a_h, a_noiseless=a_0)
cfg = rbench.ExperimentConfig(experiment="rpca-recovery", sizes=(60, 80))
rows = rbench.run_rpca_recovery(cfg)
cols = list(zip(*rows))
put("harness_rpca_recovery", "bench.run_rpca_recovery(ExperimentConfig('rpca-recovery', sizes=(60, 80)))",
    n=np.array(cols[0]), solver=np.array(cols[1]), rank_l=np.array(cols[2]), nnz_s=np.array(cols[3]),
    iters=np.array(cols[4]), zeta=np.array(cols[5]), flops=np.array(cols[6]))

here = Path(__file__).resolve().parent
np.savez_compressed(here / "golden.npz", **out)
(here / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
print("wrote", len(out), "arrays")
