"""numpy restatement of the reference CoR-UTV / ALM-CoRUTV algorithms.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): this module is the
checker the CUDA path is compared against and the CPU baseline that
``bench.py`` times.  It is never imported by the product package.

Every function restates the reference algorithm it names (file:line under
``/root/reference/pkg/src/corutv/``) in plain numpy — same operations, same
pivot / sign / tie-break / stopping rules, so that on identical inputs it
reproduces the reference to round-off (pinned by tests/test_oracle_golden.py
against vectors produced by the reference itself).

Randomness: ``gaussian_matrix`` draws from numpy's PCG64 + ziggurat normal
stream exactly as ``sketch.py:63-68`` does; numpy does not promise stream
stability across versions, so golden vectors record the numpy version.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "VARIANT_EXACT", "VARIANT_APPROX",
    "as_matrix", "gaussian_matrix",
    "householder_qr", "qrcp", "jacobi_singular_values", "jacobi_svd",
    "pseudoinverse", "spectral_norm",
    "corutv", "corutv_lowrank_error", "flop_estimate", "sor_svd", "tsr_svd", "SECOND_STREAM_OFFSET",
    "shrink", "truncate_utv", "numerical_rank", "next_cap", "alm_corutv",
    "svt", "svt_warm", "inexact_alm",
    "solver_flops",
]

VARIANT_EXACT = "exact-d"   # sketch.py:53
VARIANT_APPROX = "approx-d"  # sketch.py:55
SECOND_STREAM_OFFSET = 0x9E3779B9  # sketch.py:60 (tsr_svd's second Gaussian stream)
NNZ_EPS = 1e-12              # rpca.py:44
RANK_RTOL = 1e-12            # rpca.py:46
JACOBI_TOL = 1e-14           # dense.py:34
JACOBI_MAX_SWEEPS = 100      # dense.py:36


class OracleConvergenceError(RuntimeError):
    """Mirror of errors.py:8-18 for the oracle (carries residual/history)."""

    def __init__(self, message, residual=None, history=None):
        super().__init__(message)
        self.residual = residual
        self.history = list(history) if history is not None else None


# --------------------------------------------------------------------------
# input handling and randomness
# --------------------------------------------------------------------------

def as_matrix(a, name="matrix", require_finite=True):
    """dense.py:41-50 — float64, 2-D, positive dims, finite."""
    x = np.asarray(a, dtype=float)
    if x.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {x.shape}")
    if min(x.shape) < 1:
        raise ValueError(f"{name} must have positive dimensions, got {x.shape}")
    if require_finite and not np.isfinite(x).all():
        raise ValueError(f"{name} contains non-finite entries")
    return x


def gaussian_matrix(rows, cols, seed):
    """sketch.py:63-68 — PCG64(seed) ziggurat standard normals, C order."""
    if rows < 1 or cols < 1:
        raise ValueError(f"gaussian_matrix needs positive dims, got {rows}x{cols}")
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((rows, cols))


# --------------------------------------------------------------------------
# Householder QR / QRCP  (dense.py:104-192)
# --------------------------------------------------------------------------

def _house(x):
    """dense.py:104-114: v = x + sign(x0)|x| e1 (sign(0) = +1), tau = 2/v'v;
    a zero column yields no reflector."""
    norm = np.sqrt((x * x).sum())
    if norm == 0.0:
        return None
    v = np.array(x, copy=True)
    v[0] = v[0] + (norm if v[0] >= 0.0 else -norm)
    return v, 2.0 / (v * v).sum()


def _reflect(block, refl):
    """block <- (I - tau v v') block, applied as in dense.py:126-128/145-147."""
    v, tau = refl
    w = tau * (v @ block)
    block -= np.outer(v, w)


def _form_q(reflectors, rows, ncols):
    """dense.py:117-129: explicit thin Q by reverse accumulation on I."""
    q = np.zeros((rows, ncols))
    idx = np.arange(ncols)
    q[idx, idx] = 1.0
    for j in reversed(range(len(reflectors))):
        if reflectors[j] is not None:
            _reflect(q[j:, :], reflectors[j])
    return q


def householder_qr(a):
    """dense.py:132-149 — thin Householder QR, returns (q, r) with r = triu."""
    a = as_matrix(a, "a")
    m, n = a.shape
    if m < n:
        raise ValueError(f"householder_qr requires rows >= cols, got {m}x{n}")
    r = a.copy()
    refl = []
    for j in range(n):
        h = _house(r[j:, j].copy())
        refl.append(h)
        if h is not None:
            _reflect(r[j:, j:], h)
    return _form_q(refl, m, n), np.triu(r[:n, :])


def qrcp(a):
    """dense.py:152-192 — Businger-Golub column pivoting.

    Pivot = argmax of the downdated residual norms^2 (first index on ties),
    norms downdated by the new row of R, clamped at 0, and recomputed exactly
    where they fall below 1e-10 of their reference value.
    Returns (q, r, perm).
    """
    a = as_matrix(a, "a")
    m, n = a.shape
    k = min(m, n)
    r = a.copy()
    perm = np.arange(n)
    nrm = np.einsum("ij,ij->j", r, r)
    ref = nrm.copy()
    refl = []
    for j in range(k):
        p = j + int(np.argmax(nrm[j:]))
        if p != j:
            for arr in (perm, nrm, ref):
                arr[[j, p]] = arr[[p, j]]
            r[:, [j, p]] = r[:, [p, j]]
        h = _house(r[j:, j].copy())
        refl.append(h)
        if h is not None:
            _reflect(r[j:, j:], h)
        if j + 1 < n:
            tail = slice(j + 1, None)
            nrm[tail] -= r[j, tail] * r[j, tail]
            np.maximum(nrm[tail], 0.0, out=nrm[tail])
            stale = np.nonzero(nrm[tail] < 1e-10 * ref[tail])[0] + (j + 1)
            if stale.size:
                fresh = np.einsum("ij,ij->j", r[j + 1:, stale], r[j + 1:, stale])
                nrm[stale] = fresh
                ref[stale] = fresh
    return _form_q(refl, m, k), np.triu(r[:k, :]), perm


# --------------------------------------------------------------------------
# one-sided Jacobi SVD (dense.py:200-387) — small matrices only
# --------------------------------------------------------------------------

def _round_robin(n):
    """dense.py:200-210: n-1 rounds of n/2 disjoint pairs (n even)."""
    ring = list(range(n))
    out = []
    for _ in range(n - 1):
        out.append((np.array([ring[0]] + ring[1:n // 2]),
                    np.array(ring[n // 2:][::-1])))
        ring = [ring[0], ring[-1]] + ring[1:-1]
    return out


def _jacobi_rotate(x, tol, max_sweeps, want_v):
    """dense.py:223-282: cyclic one-sided Jacobi with cached column norms."""
    n = x.shape[1]
    if n == 1:
        return (np.eye(1) if want_v else None)
    v = np.eye(n) if want_v else None
    nrm = np.einsum("ij,ij->j", x, x)
    sched = _round_robin(n)
    off = 0.0
    for _ in range(max_sweeps):
        off = 0.0
        for top, bot in sched:
            xt, xb = x[:, top], x[:, bot]
            gam = np.einsum("ij,ij->j", xt, xb)
            al, be = nrm[top], nrm[bot]
            den = np.sqrt(al * be)
            with np.errstate(invalid="ignore", divide="ignore"):
                rel = np.where(den > 0.0, np.abs(gam) / den, 0.0)
            off = max(off, float(rel.max()))
            sel = rel > tol
            if not sel.any():
                continue
            ia, ib, g = top[sel], bot[sel], gam[sel]
            aa, bb = al[sel], be[sel]
            zeta = (bb - aa) / (2.0 * g)
            t = np.sign(zeta) / (np.abs(zeta) + np.sqrt(1.0 + zeta * zeta))
            c = 1.0 / np.sqrt(1.0 + t * t)
            s = c * t
            xa, xc = xt[:, sel], xb[:, sel]
            x[:, ia] = c * xa - s * xc
            x[:, ib] = s * xa + c * xc
            nrm[ia] = np.maximum(aa - t * g, 0.0)
            nrm[ib] = np.maximum(bb + t * g, 0.0)
            if want_v:
                va, vb = v[:, ia], v[:, ib]
                v[:, ia] = c * va - s * vb
                v[:, ib] = s * va + c * vb
        if off <= tol:
            return v
        nrm = np.einsum("ij,ij->j", x, x)
    raise OracleConvergenceError(
        f"one-sided Jacobi did not converge in {max_sweeps} sweeps", residual=off)


def _jacobi_tall(a, want_uv, v_init=None):
    """dense.py:313-354: warm start X = A v_init when given, else
    QR-precondition when m > n; pad odd widths with a zero column, sort
    descending (stable); V = v_init Vrot when warm-started."""
    m, n = a.shape
    q0 = None
    if v_init is not None:
        v_init = as_matrix(v_init, "v_init")
        if v_init.shape != (n, n):
            raise ValueError(f"v_init must be {n}x{n}, got {v_init.shape}")
        x = np.asfortranarray(a @ v_init)
    elif m > n:
        q0, x = householder_qr(a)
        x = np.asfortranarray(x)
    else:
        x = np.array(a, order="F")
    pad = n % 2 == 1 and n > 1
    if pad:
        x = np.asfortranarray(np.concatenate([x, np.zeros((x.shape[0], 1))], axis=1))
    vr = _jacobi_rotate(x, JACOBI_TOL, JACOBI_MAX_SWEEPS, want_uv)
    if pad:
        x = x[:, :-1]
        if want_uv:
            vr = vr[:-1, :-1]
    sig = np.sqrt(np.einsum("ij,ij->j", x, x))
    order = np.argsort(-sig, kind="stable")
    sig = sig[order]
    if not want_uv:
        return None, sig, None
    u = x[:, order].copy()
    nz = sig > 0.0
    u[:, nz] /= sig[nz]
    if (~nz).any():
        _complete_orthonormal(u, np.nonzero(~nz)[0])   # dense.py:347-349
    if q0 is not None:
        u = q0 @ u
    v = vr[:, order]
    if v_init is not None:
        v = v_init @ v
    return u, sig, v


def jacobi_singular_values(a):
    """dense.py:379-387."""
    a = as_matrix(a, "a")
    if a.shape[0] < a.shape[1]:
        a = a.T
    return _jacobi_tall(a, False)[1]


def _complete_orthonormal(u, fill):
    """dense.py:285-310: replace the columns ``fill`` (zero singular values)
    by unit-vector candidates e_0, e_1, ... Gram-Schmidt'ed (twice) against
    the kept columns, accepted when their residual norm exceeds 0.1."""
    m = u.shape[0]
    keep = [j for j in range(u.shape[1]) if j not in set(int(f) for f in fill)]
    basis = [u[:, j] for j in keep]
    cand = 0
    for j in fill:
        while True:
            if cand >= m:
                raise OracleConvergenceError("orthonormal completion ran out of candidates")
            w = np.zeros(m)
            w[cand] = 1.0
            cand += 1
            for _ in range(2):
                for b in basis:
                    w -= (b @ w) * b
            nw = np.sqrt((w * w).sum())
            if nw > 0.1:
                w /= nw
                break
        u[:, j] = w
        basis.append(w)


def jacobi_svd(a, v_init=None):
    """dense.py:357-376.  Returns (u, sigma, v)."""
    a = as_matrix(a, "a")
    if a.shape[0] >= a.shape[1]:
        return _jacobi_tall(a, True, v_init)
    u, s, v = _jacobi_tall(a.T, True, v_init)
    return v, s, u


def pseudoinverse(a):
    """dense.py:390-402: cutoff max(m,n)*sigma0*1e-12."""
    a = as_matrix(a, "a")
    u, s, v = jacobi_svd(a)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((a.shape[1], a.shape[0]))
    cut = max(a.shape) * s[0] * 1e-12
    inv = np.where(s > cut, 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return (v * inv) @ u.T


def spectral_norm(a, tol=1e-10, max_iter=5000):
    """dense.py:405-442 — Jacobi for min dim <= 64, else block power
    iteration (b = min(24, n)) from disjoint-support unit blocks, stop when
    |est - prev| <= 0.02 tol est.  Returns (estimate, iterations)."""
    a = as_matrix(a, "a")
    m, n = a.shape
    if min(m, n) <= 64:
        return float(jacobi_singular_values(a)[0]), 0
    if m < n:
        a = a.T
        m, n = n, m
    b = min(24, n)
    v = np.zeros((n, b))
    for j in range(b):
        v[j::b, j] = 1.0
    v /= np.sqrt(np.einsum("ij,ij->j", v, v))
    prev = 0.0
    for it in range(max_iter):
        w = a @ v
        est = float(jacobi_singular_values(householder_qr(w)[1])[0])
        if est == 0.0:
            return 0.0, it + 1
        if abs(est - prev) <= 0.02 * tol * est:
            return est, it + 1
        prev = est
        v = householder_qr(a.T @ w)[0]
    raise OracleConvergenceError("spectral norm power iteration did not converge",
                                 residual=prev)


# --------------------------------------------------------------------------
# CoR-UTV (sketch.py:166-217, 272-296)
# --------------------------------------------------------------------------

def corutv(a, ell, q_power=0, seed=0, variant=VARIANT_EXACT, omega=None,
           counter=None):
    """sketch.py:182-208 (with _power_sketch sketch.py:166-179).

    Returns dict(u, t, v, perm, passes).  ``omega`` overrides the seeded
    Gaussian draw (the north-star's caller-supplied test matrix).
    """
    a = as_matrix(a, "a")
    m, n = a.shape
    if m < n:
        raise ValueError(f"corutv requires rows >= cols, got {m}x{n}")
    if ell > min(m, n):
        raise ValueError(f"ell={ell} exceeds min(m, n)={min(m, n)} for a {m}x{n} input")
    passes = 0
    c2 = gaussian_matrix(n, ell, seed) if omega is None else np.asarray(omega, float)
    for _ in range(q_power + 1):
        c2_in = c2
        c1 = a @ c2
        c2 = a.T @ c1
        passes += 2
    q1, _ = householder_qr(c1)
    q2, _ = householder_qr(c2)
    if variant == VARIANT_EXACT:
        d = q1.T @ (a @ q2)
        passes += 1
    else:
        d = (q1.T @ c1) @ pseudoinverse(q2.T @ c2_in)
    qd, rd, perm = qrcp(d)
    if counter is not None:
        counter.passes += passes
    return dict(u=q1 @ qd, t=rd, v=q2[:, perm], perm=perm, passes=passes)


def sor_svd(a, ell, q_power=0, seed=0, variant=VARIANT_EXACT, omega=None):
    """sketch.py:244-262: the corutv pipeline finished by jacobi_svd of the
    compressed core instead of qrcp.  Returns dict(u, sigma, v, passes)."""
    a = as_matrix(a, "a")
    m, n = a.shape
    if m < n:
        raise ValueError(f"sor_svd requires rows >= cols, got {m}x{n}")
    if ell > min(m, n):
        raise ValueError(f"ell={ell} exceeds min(m, n)={min(m, n)} for a {m}x{n} input")
    passes = 0
    c2 = gaussian_matrix(n, ell, seed) if omega is None else np.asarray(omega, float)
    for _ in range(q_power + 1):
        c2_in = c2
        c1 = a @ c2
        c2 = a.T @ c1
        passes += 2
    q1, _ = householder_qr(c1)
    q2, _ = householder_qr(c2)
    if variant == VARIANT_EXACT:
        d = q1.T @ (a @ q2)
        passes += 1
    else:
        d = (q1.T @ c1) @ pseudoinverse(q2.T @ c2_in)
    fu, fs, fv = jacobi_svd(d)
    return dict(u=q1 @ fu, sigma=fs, v=q2 @ fv, passes=passes)


def tsr_svd(a, ell, seed=0, psi=None, phi=None):
    """sketch.py:220-241: psi = G(n, ell, seed), phi = G(m, ell, seed +
    0x9E3779B9 mod 2^64); y = A psi, z = A' phi in one (fused) pass; core =
    (Q1' y) pinv(Q2' psi); jacobi_svd(core) lifted.  No m >= n requirement."""
    a = as_matrix(a, "a")
    m, n = a.shape
    if ell > min(m, n):
        raise ValueError(f"ell={ell} exceeds min(m, n)={min(m, n)} for a {m}x{n} input")
    psi = gaussian_matrix(n, ell, seed) if psi is None else np.asarray(psi, float)
    phi = (gaussian_matrix(m, ell, (seed + SECOND_STREAM_OFFSET) % 2 ** 64) if phi is None
           else np.asarray(phi, float))
    y, z = a @ psi, a.T @ phi
    q1, _ = householder_qr(y)
    q2, _ = householder_qr(z)
    core = (q1.T @ y) @ pseudoinverse(q2.T @ psi)
    fu, fs, fv = jacobi_svd(core)
    return dict(u=q1 @ fu, sigma=fs, v=q2 @ fv, passes=1)


def corutv_lowrank_error(a, f):
    """sketch.py:211-217 numerator: |A - U T V'|_F."""
    r = a - f["u"] @ (f["t"] @ f["v"].T)
    return float(np.sqrt((r * r).sum()))


def flop_estimate(m, n, ell, q_power=0, variant=VARIANT_EXACT):
    """sketch.py:272-296 — the metric numerator (algorithmic flops)."""
    reps = q_power + 1
    tot = n * ell + reps * 4 * m * n * ell + 2 * (m + n) * ell ** 2
    if variant == VARIANT_EXACT:
        tot += m * ell ** 2 + 2 * m * n * ell
    else:
        tot += 2 * (m + n) * ell ** 2 + 3 * ell ** 3
    tot += (8 * ell ** 3) // 3 + 2 * m * ell ** 2 + 2 * n * ell
    return tot


# --------------------------------------------------------------------------
# ALM-CoRUTV robust PCA (rpca.py:99-255)
# --------------------------------------------------------------------------

def shrink(x, delta):
    """rpca.py:99-104."""
    return np.sign(x) * np.maximum(np.abs(x) - delta, 0.0)


def truncate_utv(f, delta):
    """rpca.py:122-132: r = #(|diag T| > delta); L = U_r (T_r V')."""
    d = np.abs(np.diag(f["t"]))
    r = int((d > delta).sum())
    if r == 0:
        return np.zeros((f["u"].shape[0], f["v"].shape[0])), 0, np.zeros(0)
    head = f["t"][:r, :]
    return f["u"][:, :r] @ (head @ f["v"].T), r, jacobi_singular_values(head)


def numerical_rank(sig, shape):
    """rpca.py:161-164."""
    if sig.size == 0 or sig[0] <= 0.0:
        return 0
    return int((sig > max(shape) * sig[0] * RANK_RTOL).sum())


def next_cap(cap, rank, limit, grow):
    """rpca.py:167-172."""
    if rank < cap:
        return max(1, min(rank + 1, limit))
    return max(1, min(rank + grow, limit))


def svt_warm(b, delta, v_init=None, cap=None):
    """rpca.py:146-158 (_svt_warm): threshold the Jacobi spectrum of b.
    Returns (matrix, r, v, kept[:r])."""
    if delta < 0:
        raise ValueError("delta must be >= 0")
    b = as_matrix(b, "b")
    u, sig, v = jacobi_svd(b, v_init)
    kept = np.maximum(sig - delta, 0.0)
    r = int((kept > 0.0).sum())
    if cap is not None:
        r = min(r, cap)
    if r == 0:
        return np.zeros_like(b), 0, v, np.zeros(0)
    return (u[:, :r] * kept[:r]) @ v[:, :r].T, r, v, kept[:r]


def svt(b, delta):
    """rpca.py:135-143."""
    mat, r, _, _ = svt_warm(b, delta)
    return mat, r


def _alm_loop(m_mat, step, cap0, lam=None, mu0=None, rho=1.5, mu_bar=None, tol=1e-5, max_iter=1000):
    """rpca.py:175-234: step(g, delta, cap, j, state) -> (L, rank, sig, state)."""
    m_mat = as_matrix(m_mat, "m")
    h, w = m_mat.shape
    lam = lam if lam is not None else 1.0 / np.sqrt(max(h, w))
    norm_m = float(np.sqrt((m_mat * m_mat).sum()))
    if norm_m == 0.0:
        z = np.zeros_like(m_mat)
        return dict(l=z, s=z.copy(), iterations=1, residuals=[0.0], rank_of_l=0,
                    nnz_of_s=0, rank_history=[0], nnz_history=[0],
                    mu_history=[0.0], ell_history=[0], mu0=0.0)
    mu = mu0 if mu0 is not None else 1.25 / spectral_norm(m_mat)[0]
    mu_first = mu
    mu_bar = mu_bar if mu_bar is not None else 1e7 * mu
    limit = min(h, w)
    grow = max(1, round(0.05 * limit))
    cap = max(1, min(cap0, limit))
    y = np.zeros_like(m_mat)
    s = np.zeros_like(m_mat)
    hist = dict(residuals=[], rank_history=[], nnz_history=[], mu_history=[],
                ell_history=[])
    state = None
    for j in range(max_iter):
        l, rank, sig, state = step(m_mat - s + y / mu, 1.0 / mu, cap, j, state)
        hist["ell_history"].append(cap)
        cap = next_cap(cap, rank, limit, grow)
        g = m_mat - l + y / mu
        s = np.sign(g) * np.maximum(np.abs(g) - lam / mu, 0.0)
        z = m_mat - l - s
        y = y + mu * z
        zeta = float(np.sqrt((z * z).sum())) / norm_m
        nnz = int((np.abs(s) > NNZ_EPS).sum())
        hist["residuals"].append(zeta)
        hist["rank_history"].append(rank)
        hist["nnz_history"].append(nnz)
        hist["mu_history"].append(mu)
        if zeta < tol:
            return dict(l=l, s=s, iterations=j + 1, rank_of_l=numerical_rank(sig, m_mat.shape),
                        nnz_of_s=nnz, mu0=mu_first, **hist)
        mu = min(rho * mu, mu_bar)
    raise OracleConvergenceError(
        f"ALM did not reach tol={tol:.1e} in {max_iter} iterations",
        residual=hist["residuals"][-1], history=hist["residuals"])


def alm_corutv(m_mat, ell, lam=None, mu0=None, rho=1.5, mu_bar=None, tol=1e-5,
               max_iter=1000, q_power=1, seed=0):
    """rpca.py:237-255 (alm_corutv + _alm_loop).  Returns a dict with the
    RpcaSolution fields (l, s, iterations, residuals, rank_of_l, nnz_of_s,
    rank_history, nnz_history, mu_history, ell_history) plus ``mu0``."""

    def step(g, delta, cap, j, state):
        f = corutv(g, cap, q_power, (seed + j) % 2 ** 64)
        l, rank, sig = truncate_utv(f, delta)
        return l, rank, sig, None

    return _alm_loop(m_mat, step, ell, lam, mu0, rho, mu_bar, tol, max_iter)


def inexact_alm(m_mat, ell=None, lam=None, mu0=None, rho=1.5, mu_bar=None, tol=1e-5,
                max_iter=1000):
    """rpca.py:258-273: the same loop with the warm-started SVT step."""

    def step(g, delta, cap, j, state):
        mat, r, v, kept = svt_warm(g, delta, state, cap)
        return mat, r, kept, v

    m_arr = as_matrix(m_mat, "m")
    cap0 = ell if ell is not None else min(m_arr.shape)
    return _alm_loop(m_arr, step, cap0, lam, mu0, rho, mu_bar, tol, max_iter)


def solver_flops(n, q_power, rank_history, ell_history):
    """bench.py:251-264 (alm-corutv branch): per-iteration flop numerator."""
    tot = 0
    for r, ell in zip(rank_history, ell_history):
        ell = max(1, ell)
        tot += flop_estimate(n, n, ell, q_power, VARIANT_EXACT) + 2 * r * ell * n
        tot += 2 * n * n * r + 8 * n * n
    return tot


# --------------------------------------------------------------------------
# seeded test-input generators (synth.py:77-99, 123-134)
# --------------------------------------------------------------------------

def gen_noisy_lowrank(n, k, noise_coeff=0.1, sigma_max=1.0, sigma_min=1e-9, seed=0):
    """synth.py:77-99 with the default spectral noise normalisation and the
    "full" ramp (synth.py:67-74)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = householder_qr(rng.standard_normal((n, k)))[0]
    v = householder_qr(rng.standard_normal((n, k)))[0]
    sig = np.zeros(n)
    sig[:k] = np.linspace(sigma_max, sigma_min, n)[:k]
    a = (u * sig[:k]) @ v.T
    if noise_coeff > 0:
        e = rng.standard_normal((n, n))
        e /= spectral_norm(e)[0]
        a = a + (noise_coeff * sig[k - 1]) * e
    return a, sig


def gen_rpca_instance(n, k, s, amplitude=80.0, seed=0):
    """synth.py:123-134: Gaussian rank-k product plus s signed spikes at
    distinct uniform positions.  Returns (m, l_true, s_true)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    l_true = rng.standard_normal((n, k)) @ rng.standard_normal((k, n))
    s_true = np.zeros((n, n))
    if s > 0:
        pos = rng.choice(n * n, size=s, replace=False)
        signs = rng.integers(0, 2, size=s) * 2 - 1
        s_true.flat[pos] = amplitude * signs
    return l_true + s_true, l_true, s_true


__all__ += ["gen_noisy_lowrank", "gen_rpca_instance", "OracleConvergenceError"]
