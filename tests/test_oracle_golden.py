"""Pin the CPU oracle against golden vectors produced by the reference
itself (tests/golden/make_golden.py) and against the reference's own
known-answer tests.  No GPU needed."""

import numpy as np
import pytest

import oracle as O


def _sign_align(x, y):
    """Align columns of x to y by sign (column signs are free in QR)."""
    s = np.sign(np.sum(x * y, axis=0))
    s[s == 0] = 1.0
    return x * s


@pytest.mark.parametrize("seed", range(3))
def test_qr_matches_reference(golden, seed):
    c = golden[f"qr{seed}"]
    q, r = O.householder_qr(c["a"])
    assert np.abs(q - c["q"]).max() < 1e-13
    assert np.abs(r - c["r"]).max() < 1e-13
    assert np.abs(np.tril(r, -1)).max() == 0.0


@pytest.mark.parametrize("name", ["qrcp_diag", "qrcp_tie", "qrcp_rand", "qrcp_square", "qrcp_rank5"])
def test_qrcp_matches_reference(golden, name):
    c = golden[name]
    q, r, perm = O.qrcp(c["a"])
    assert np.array_equal(perm, c["perm"])
    scale = max(1.0, np.abs(c["a"]).max())
    assert np.abs(q - c["q"]).max() < 1e-12
    assert np.abs(r - c["r"]).max() < 1e-12 * scale


def test_qrcp_known_answers():
    # pkg/tests/test_dense.py:97-107
    q, r, perm = O.qrcp(np.diag([1.0, 3.0, 2.0]))
    assert list(perm) == [1, 2, 0]
    assert np.abs(np.abs(np.diag(r)) - [3.0, 2.0, 1.0]).max() < 1e-14
    _, _, perm = O.qrcp(np.array([[2.0, 1.0, 2.0], [0.0, 0.5, 0.0]]))
    assert perm[0] == 0


def test_singular_values_pinv_snorm(golden):
    c = golden["sv"]
    assert np.abs(O.jacobi_singular_values(c["a"]) - c["sig"]).max() < 1e-13
    c = golden["pinv"]
    assert np.abs(O.pseudoinverse(c["a"]) - c["pinv"]).max() < 1e-11
    for name in ("snorm_block", "snorm_direct"):
        c = golden[name]
        val, _ = O.spectral_norm(c["a"])
        assert abs(val - float(c["val"])) <= 1e-13 * float(c["val"])


def test_gaussian_stream(golden):
    # same numpy => bit-identical PCG64/ziggurat stream (sketch.py:63-68)
    assert np.array_equal(O.gaussian_matrix(30, 7, 12345), golden["omega"]["val"])


CU = ["cu_replay", "cu_rank8_q0", "cu_rank8_q2", "cu_rank8_q2_approx", "cu_noisy_q1",
      "cu_full_ell", "cu_ell1", "cu_c2small_q2"]


@pytest.mark.parametrize("name", CU)
def test_corutv_matches_reference(golden, name):
    c = golden[name]
    ell = c["t"].shape[0]
    info = name
    variant = "approx-d" if "approx" in info else "exact-d"
    # recover q/seed from the golden: omega is stored, so pass it explicitly
    q = {"cu_replay": 1, "cu_rank8_q0": 0, "cu_rank8_q2": 2, "cu_rank8_q2_approx": 2,
         "cu_noisy_q1": 1, "cu_full_ell": 1, "cu_ell1": 1, "cu_c2small_q2": 2}[name]
    f = O.corutv(c["a"], ell, q, omega=c["omega"], variant=variant)
    assert f["passes"] == int(c["passes"])
    a = c["a"]
    err = O.corutv_lowrank_error(a, f)
    assert abs(err - float(c["err"])) <= 1e-10 * np.linalg.norm(a) + 1e-10 * float(c["err"])
    assert np.abs(np.abs(np.diag(f["t"])) - np.abs(np.diag(c["t"]))).max() <= 1e-9 * np.abs(c["t"]).max()
    # leading columns (well separated) agree to ~1e-9 up to sign
    u = _sign_align(f["u"], c["u"])
    v = _sign_align(f["v"], c["v"])
    assert np.abs(u - c["u"]).max() < 1e-8
    assert np.abs(v - c["v"]).max() < 1e-8
    assert O.flop_estimate(a.shape[0], a.shape[1], ell, q, variant) == int(c["flops"])


@pytest.mark.parametrize("n", [60, 100])
def test_alm_matches_reference(golden, n):
    c = golden[f"alm_n{n}"]
    k = max(1, round(0.05 * n))
    cseed = {60: 11, 100: 5}[n]
    sol = O.alm_corutv(c["m"], ell=2 * k, q_power=1, seed=cseed)
    assert sol["iterations"] == int(c["iterations"])
    assert sol["ell_history"] == list(c["ell_history"])
    assert sol["rank_history"] == list(c["rank_history"])
    assert sol["nnz_history"] == list(c["nnz_history"])
    assert sol["rank_of_l"] == int(c["rank_of_l"]) and sol["nnz_of_s"] == int(c["nnz_of_s"])
    assert abs(sol["mu0"] - float(c["mu0"])) <= 1e-12 * float(c["mu0"])
    nl = np.linalg.norm(c["l"])
    assert np.linalg.norm(sol["l"] - c["l"]) <= 1e-8 * nl
    assert np.linalg.norm(sol["s"] - c["s"]) <= 1e-8 * max(np.linalg.norm(c["s"]), 1.0)


def test_rpca_generator_matches_reference(golden):
    c = golden["alm_n60"]
    m, _, _ = O.gen_rpca_instance(60, 3, 180, seed=7)
    assert np.array_equal(m, c["m"])


@pytest.mark.slow
def test_alm_desk_scale_matches_reference(golden):
    c = golden["alm_n400"]
    m, _, _ = O.gen_rpca_instance(400, 20, 8000, seed=0)
    assert m.sum() == float(c["m_sum"])
    sol = O.alm_corutv(m, ell=40, q_power=1, seed=1)
    assert sol["iterations"] == int(c["iterations"])
    assert sol["ell_history"] == list(c["ell_history"])
    assert np.array_equal(np.flatnonzero(np.abs(sol["s"]) > 1e-12), c["s_support"])


@pytest.mark.parametrize("name", ["svd_tall", "svd_wide", "svd_square", "svd_zero_cols"])
def test_jacobi_svd_matches_reference(golden, name):
    c = golden[name]
    u, s, v = O.jacobi_svd(c["a"])
    assert np.array_equal(s, c["sigma"])
    assert np.array_equal(u, c["u"]) and np.array_equal(v, c["v"])


@pytest.mark.parametrize("name", ["sor_q1", "sor_q0_approx", "sor_c2small", "tsr_tall", "tsr_wide", "tsr_noisy"])
def test_svd_sketches_match_reference(golden, name):
    c = golden[name]
    q, seed = {"sor_q1": (1, 8), "sor_q0_approx": (0, 3), "sor_c2small": (2, 77), "tsr_tall": (0, 4),
               "tsr_wide": (0, 6), "tsr_noisy": (0, 1)}[name]
    ell = c["sigma"].size
    if name.startswith("sor"):
        variant = O.VARIANT_APPROX if "approx" in name else O.VARIANT_EXACT
        f = O.sor_svd(c["a"], ell, q, seed, variant)
    else:
        f = O.tsr_svd(c["a"], ell, seed)
    assert f["passes"] == int(c["passes"])
    assert np.array_equal(f["sigma"], c["sigma"])
    assert np.array_equal(f["u"], c["u"]) and np.array_equal(f["v"], c["v"])


# ---- InexactALM baseline pieces --------------------------------

@pytest.mark.parametrize("name", ["svdwarm_sq", "svdwarm_tall", "svdwarm_wide"])
def test_warm_jacobi_svd_matches_reference(golden, name):
    c = golden[name]
    u, s, v = O.jacobi_svd(c["a"], c["v_init"])
    assert np.array_equal(s, c["sigma"])
    assert np.array_equal(u, c["u"]) and np.array_equal(v, c["v"])


def test_warm_jacobi_rejects_wrong_v_init(golden):
    c = golden["svdwarm_wide"]
    with pytest.raises(ValueError, match="v_init must be 13x13"):
        O.jacobi_svd(c["a"], np.eye(29))


@pytest.mark.parametrize("name", ["svt_diag", "svt_zero", "svt_nuc", "svt_wide", "svt_rank"])
def test_svt_matches_reference(golden, name):
    c = golden[name]
    mat, r = O.svt(c["b"], float(c["delta"]))
    assert r == int(c["r"])
    assert np.array_equal(mat, c["mat"])


@pytest.mark.parametrize("n", [60, 100])
def test_inexact_alm_matches_reference(golden, n):
    c = golden[f"ialm_n{n}"]
    sol = O.inexact_alm(c["m"], ell=int(c["ell_history"][0]))
    assert sol["iterations"] == int(c["iterations"])
    for key in ("rank_history", "nnz_history", "ell_history"):
        assert sol[key] == [int(x) for x in c[key]]
    assert np.array_equal(np.array(sol["residuals"]), c["residuals"])
    assert np.array_equal(np.array(sol["mu_history"]), c["mu_history"])
    assert sol["rank_of_l"] == int(c["rank_of_l"]) and sol["nnz_of_s"] == int(c["nnz_of_s"])
    assert np.array_equal(sol["l"], c["l"]) and np.array_equal(sol["s"], c["s"])


def test_inexact_alm_max_iter_history_matches_reference(golden):
    c = golden["ialm_maxiter"]
    with pytest.raises(O.OracleConvergenceError) as exc:
        O.inexact_alm(c["m"], max_iter=2)
    assert np.array_equal(np.array(exc.value.history), c["history"])


def test_inexact_alm_zero_matrix():
    sol = O.inexact_alm(np.zeros((30, 30)))
    assert sol["iterations"] == 1 and not sol["l"].any() and not sol["s"].any()
