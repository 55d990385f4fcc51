"""TEST INFRASTRUCTURE ONLY — CPU oracle for PbP-QLP.

Used by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) as the checker / the timed CPU reference.  The product
package never imports it.

This is a restatement of the reference path at the numpy level, call for call:

* ``oracle_gaussian``   ↔ ``gaussian_matrix``  (pbpqlp/linalg.py:83-93)
* ``oracle_qr``         ↔ ``householder_qr`` + ``_fix_signs`` (linalg.py:96-115)
* ``oracle_orth``       ↔ ``orth``             (linalg.py:142-165)
* ``oracle_pbp_qlp``    ↔ ``pbp_qlp``          (algorithms.py:209-260)
* ``oracle_r_svd``       ↔ ``r_svd``         (algorithms.py:263-292)
* ``oracle_spectral_norm`` ↔ ``spectral_norm`` (linalg.py:168-207)
* ``oracle_error_curve``   ↔ ``error_curve``   (analysis.py:213-247, pbp_qlp)
* ``oracle_column_pivoted_qr`` ↔ ``column_pivoted_qr`` (linalg.py:118-129; scipy
  1.18 → LAPACK dgeqp3)
* ``oracle_cor_utv``     ↔ ``cor_utv``        (algorithms.py:295-363)

``cpqr_pivots_restated`` restates LAPACK dlaqp2's pivot rule (first-max
pivot, norm downdating with the √ε recompute test) without a LAPACK call; it
cross-checks scipy's pivots and is the rule the device kernel implements.

The arithmetic lives in numpy 2.3.5 (the reference pins only numpy>=1.24,
pyproject.toml:11-15): dgemm for products, LAPACK dgeqrf+dorgqr (via
``np.linalg.qr``) for QR, Philox4x64-10 + ziggurat for the sketch.  Because the
calls are the reference's own, the oracle reproduces the reference bit for bit
on the same machine (pinned in tests/test_oracle.py against /root/reference
when present and against the committed tests/golden/ fixtures everywhere).

``householder_qr_restated`` is an independent column-by-column restatement of
LAPACK's dgeqr2/dorg2r Householder algorithm (no LAPACK call), used to
cross-check ``oracle_qr`` on small inputs.
"""
import ctypes
import os

import numpy as np

RANK_DEFICIENCY_RTOL = 1e-14  # linalg.py:48

_HERE = os.path.dirname(os.path.abspath(__file__))
_CLIB = os.path.join(_HERE, "_build", "libpbq_oracle.so")
_clib = None


def build_c_oracle():
    """Compile sketch_oracle.c (gcc) into oracle/_build/."""
    import subprocess

    os.makedirs(os.path.join(_HERE, "_build"), exist_ok=True)
    src = os.path.join(_HERE, "sketch_oracle.c")
    if not os.path.exists(_CLIB) or os.path.getmtime(_CLIB) < os.path.getmtime(src):
        subprocess.run(["gcc", "-O2", "-fPIC", "-std=gnu11", "-ffp-contract=off", "-shared", "-o", _CLIB, src, "-lm"],
                       check=True)
    return _CLIB


def _c():
    global _clib
    if _clib is None:
        if not os.path.exists(_CLIB):
            build_c_oracle()
        lib = ctypes.CDLL(_CLIB)
        lib.pbqo_philox_raw.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_void_p]
        lib.pbqo_normals.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_void_p]
        lib.pbqo_normals.restype = ctypes.c_uint64
        lib.pbqo_log1p_pair.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p]
        _clib = lib
    return _clib


# ------------------------------------------------------------------ sketch --
def oracle_gaussian(rows, cols, seed=0):
    """numpy's own draw, exactly what the reference calls (linalg.py:92-93)."""
    rng = np.random.Generator(np.random.Philox(key=int(seed)))
    return rng.standard_normal((rows, cols))


def c_gaussian(rows, cols, seed=0, row_offset=0):
    """The C restatement (sketch_oracle.c): rows [row_offset, row_offset+rows)."""
    seed = int(seed)
    out = np.empty((rows, cols))
    _c().pbqo_normals(seed & (2**64 - 1), seed >> 64, row_offset * cols, rows * cols, out.ctypes.data)
    return out


def c_log1p_pair(x):
    """(restated glibc log1p — the device's glibc_log1p — , the C library's
    log1p) of every x: the pin of the sketch's exponential-tail arithmetic."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    a, b = np.empty_like(x), np.empty_like(x)
    _c().pbqo_log1p_pair(x.ctypes.data, x.size, a.ctypes.data, b.ctypes.data)
    return a, b


def c_philox_raw(seed, start, n):
    seed = int(seed)
    out = np.empty(n, dtype=np.uint64)
    _c().pbqo_philox_raw(seed & (2**64 - 1), seed >> 64, start, n, out.ctypes.data)
    return out


# ---------------------------------------------------------------------- QR --
def _fix_signs(q, r):
    k = min(r.shape)
    signs = np.sign(np.diagonal(r)[:k])
    signs[signs == 0] = 1.0
    q[:, :k] *= signs
    r[:k, :] *= signs[:, None]
    return q, r


def oracle_qr(m):
    """(Q, R) with diag(R) >= 0 and an exact-zero lower triangle (linalg.py:106-115)."""
    q, r = np.linalg.qr(np.asarray(m, dtype=np.float64), mode="reduced")
    q, r = _fix_signs(q.copy(), r.copy())
    return q, np.triu(r)


def rank_flag(r):
    """0 ok, 1 rank deficient, 2 identically zero — the two warnings of orth."""
    diag = np.abs(np.diagonal(r))
    if diag.size and diag[0] > 0 and np.any(diag < RANK_DEFICIENCY_RTOL * diag[0]):
        return 1
    if diag.size and diag[0] == 0:
        return 2
    return 0


def oracle_orth(m, diag_log=None):
    q, r = oracle_qr(m)
    if diag_log is not None:  # test hook: |diag R| of every orth call, in call order
        diag_log.append(np.abs(np.diagonal(r)).copy())
    return q, rank_flag(r)


def householder_qr_restated(m):
    """LAPACK dgeqr2 + dorg2r restated with numpy vector ops (small inputs)."""
    a = np.array(m, dtype=np.float64)
    mm, n = a.shape
    k = min(mm, n)
    taus = np.zeros(k)
    for j in range(k):
        alpha = a[j, j]
        x = a[j + 1:, j]
        xnorm = np.linalg.norm(x)
        if xnorm == 0.0:
            taus[j] = 0.0
            continue
        beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
        taus[j] = (beta - alpha) / beta
        a[j + 1:, j] = x / (alpha - beta)
        a[j, j] = beta
        v = np.concatenate(([1.0], a[j + 1:, j]))
        w = v @ a[j:, j + 1:]
        a[j:, j + 1:] -= taus[j] * np.outer(v, w)
    r = np.triu(a[:k, :])
    q = np.zeros((mm, k))
    q[:k, :k] = np.eye(k)
    for j in range(k - 1, -1, -1):
        v = np.concatenate(([1.0], a[j + 1:, j]))
        w = v @ q[j:, j:]
        q[j:, j:] -= taus[j] * np.outer(v, w)
    return _fix_signs(q, r)


# ---------------------------------------------------------------- pipeline --
def oracle_pbp_qlp(a, d, q=0, seed=0, reorthonormalize=True, phi=None):
    """algorithms.py:209-260 restated; returns a dict of the factors plus the
    per-orth rank flags (in call order) and the pass count."""
    a = np.asarray(a, dtype=np.float64)
    n1, n2 = a.shape
    if phi is None:
        phi = oracle_gaussian(n1, d, seed)
    flags = []
    diags = []  # |diag R| of each orth call (rank-test margins)
    passes = 0
    orth = lambda m: oracle_orth(m, diags)  # noqa: E731

    def apply(block):
        nonlocal passes
        passes += 1
        return a @ block

    def apply_t(block):
        nonlocal passes
        passes += 1
        return a.T @ block

    c = apply_t(phi)
    if reorthonormalize:
        pbar, f = orth(c)
        flags.append(f)
        for _ in range(q):
            pbar, f = orth(apply(pbar))
            flags.append(f)
            pbar, f = orth(apply_t(pbar))
            flags.append(f)
    else:
        for _ in range(q):
            c = apply_t(apply(c))
        pbar, f = orth(c)
        flags.append(f)
    dmat = apply(pbar)
    qfac, rfac = oracle_qr(dmat)
    w, rt = oracle_qr(rfac.T)
    l = np.tril(rt.T)
    p = pbar @ w
    return {"q": qfac, "l": l, "p": p, "r": rfac, "phi": phi, "rank_flags": flags, "passes": passes,
            "orth_r_diag": diags}


# ------------------------------------------------------------------ checks --
def column_relative_error(x, ref):
    """max_j ‖x_j − ref_j‖ / ‖ref_j‖ after aligning column signs (BASELINE §5)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    s = np.sign(np.sum(x * ref, axis=0))
    s[s == 0] = 1.0
    num = np.linalg.norm(x * s - ref, axis=0)
    den = np.linalg.norm(ref, axis=0)
    den[den == 0] = 1.0
    return num / den


def conditioning_tolerance(l_ref, strict=1e-10, factor=64.0):
    """Per-column tolerance max(strict, factor·u·κ_j), κ_j = L_00/L_jj
    (SURVEY.md §8 a9)."""
    diag = np.abs(np.diagonal(np.asarray(l_ref)))
    with np.errstate(divide="ignore"):
        kappa = np.where(diag > 0, diag[0] / diag, np.inf)
    return np.maximum(strict, factor * 2.0**-53 * kappa)


def oracle_r_svd(a, d, q=0, seed=0, reorthonormalize=True):
    """algorithms.py:263-292 restated (sketch Ω is n2×d; transpose_first=False
    power iterations; svd_full = np.linalg.svd, linalg.py:131-139)."""
    a = np.asarray(a, dtype=np.float64)
    omega = oracle_gaussian(a.shape[1], d, seed)
    flags = []
    f = a @ omega
    if reorthonormalize:
        ubar, fl = oracle_orth(f)
        flags.append(fl)
        for _ in range(q):
            ubar, fl = oracle_orth(a.T @ ubar)
            flags.append(fl)
            ubar, fl = oracle_orth(a @ ubar)
            flags.append(fl)
    else:
        for _ in range(q):
            f = a @ (a.T @ f)
        ubar, fl = oracle_orth(f)
        flags.append(fl)
    g = (a.T @ ubar).T
    uc, s, vh = np.linalg.svd(g, full_matrices=False)
    return {"u": ubar @ uc, "s": s, "v": vh.T, "omega": omega, "rank_flags": flags}


def oracle_spectral_norm(m):
    """linalg.py:194-207: dense σ₁ up to 2000 in the larger dimension, else
    power iteration on the Gram operator (linalg.py:168-191) from the seeded
    start gaussian_matrix(n, 1, seed=0x5EED), rtol 1e-10, ≤ 5000 steps."""
    m = np.asarray(m, dtype=np.float64)
    if max(m.shape) <= 2000:
        return float(np.linalg.svd(m, compute_uv=False)[0])
    v = oracle_gaussian(m.shape[1], 1, seed=0x5EED).ravel()
    v /= np.linalg.norm(v)
    estimate = 0.0
    for _ in range(5000):
        w = m @ v
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0
        v = m.T @ w
        nv = np.linalg.norm(v)
        if nv == 0.0:
            return 0.0
        v /= nv
        new = nv / nw
        if abs(new - estimate) <= 1e-10 * max(new, 1e-300):
            return float(new)
        estimate = new
    raise RuntimeError("power iteration did not converge")


def oracle_error_curve(a, d_values, q=0, seed=0, reorthonormalize=True):
    """analysis.py:213-247 for alg = "pbp_qlp"."""
    out = []
    for d in d_values:
        f = oracle_pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize)
        res = a - f["q"] @ f["l"] @ f["p"].T
        out.append({"d": d, "spectral_error": oracle_spectral_norm(res), "frobenius_error": float(np.linalg.norm(res))})
    return out


def reconstruction_error(a, qf, l, p):
    a = np.asarray(a, dtype=np.float64)
    return np.linalg.norm(a - qf @ l @ p.T) / np.linalg.norm(a)


# -------------------------------------------------------- pivoted QR / UTV --
def oracle_column_pivoted_qr(m):
    """linalg.py:118-129: scipy.linalg.qr(m, "economic", pivoting=True), signs
    fixed so diag(r) >= 0, r = triu(r)."""
    import scipy.linalg

    m = np.asarray(m, dtype=np.float64)
    q, r, perm = scipy.linalg.qr(m, mode="economic", pivoting=True)
    q, r = _fix_signs(q, r)
    return q, np.triu(r), perm


def cpqr_pivots_restated(m, return_gaps=False):
    """Pivot order of LAPACK dlaqp2 (dgeqp3's unblocked kernel), restated:
    p = first max of the partial norms vn1 over the free positions; swap;
    Householder reflector (dlarfg) applied to the trailing columns (dlarf);
    vn1[j] downdated by √(1 − (|a_kj|/vn1[j])²) unless
    (1 − (|a_kj|/vn1[j])²)·(vn1[j]/vn2[j])² ≤ √ε (ε = 2⁻⁵³), which
    recomputes it from rows k+1.. and resets vn2[j].

    With ``return_gaps`` also returns, per step, the relative margin
    (best − runner-up)/best of the pivot choice: where it is at rounding
    level the pivot order is decided by rounding, in LAPACK as anywhere."""
    a = np.array(m, dtype=np.float64, order="F", copy=True)
    rows, n = a.shape
    perm = np.arange(n)
    vn1 = np.sqrt((a * a).sum(axis=0))
    vn2 = vn1.copy()
    tol3z = np.sqrt(2.0**-53)
    gaps = np.full(min(rows, n), np.inf)
    for k in range(min(rows, n)):
        p = k + int(np.argmax(vn1[k:]))
        if n - k > 1 and vn1[p] > 0:
            gaps[k] = (vn1[p] - np.partition(vn1[k:], -2)[-2]) / vn1[p]
        if p != k:
            a[:, [k, p]] = a[:, [p, k]]
            perm[[k, p]] = perm[[p, k]]
            vn1[p], vn2[p] = vn1[k], vn2[k]
        tau = 0.0
        if k < rows - 1:
            alpha = a[k, k]
            xnorm = float(np.sqrt((a[k + 1:, k] ** 2).sum()))
            if xnorm != 0.0:
                beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
                tau = (beta - alpha) / beta
                a[k + 1:, k] /= alpha - beta
                a[k, k] = beta
        if k < n - 1:
            if tau != 0.0:
                v = np.concatenate(([1.0], a[k + 1:, k]))
                w = v @ a[k:, k + 1:]
                a[k:, k + 1:] -= tau * np.outer(v, w)
            for j in range(k + 1, n):
                if vn1[j] != 0.0:
                    t = 1.0 - (abs(a[k, j]) / vn1[j]) ** 2
                    t = max(t, 0.0)
                    t2 = t * (vn1[j] / vn2[j]) ** 2
                    if t2 <= tol3z:
                        vn1[j] = float(np.sqrt((a[k + 1:, j] ** 2).sum())) if k < rows - 1 else 0.0
                        vn2[j] = vn1[j]
                    else:
                        vn1[j] *= np.sqrt(t)
    return (perm, gaps) if return_gaps else perm


PINV_RTOL = 1e-12  # algorithms.py:56


def oracle_cor_utv(a, d, q=0, seed=0, pass_efficient=False, reorthonormalize=True):
    """algorithms.py:306-363 restated (Ω n2×d; _power_iterations with
    transpose_first=False; _transposed_pinv_apply :295-303)."""
    a = np.asarray(a, dtype=np.float64)
    omega = oracle_gaussian(a.shape[1], d, seed)
    flags = []
    passes = 1
    f1 = a @ omega
    if reorthonormalize:
        ubar_in = f1
        ubar, fl = oracle_orth(f1)
        flags.append(fl)
        for _ in range(q):
            ubar, fl = oracle_orth(a.T @ ubar)
            flags.append(fl)
            ubar_in = a @ ubar
            ubar, fl = oracle_orth(ubar_in)
            flags.append(fl)
            passes += 2
        f2 = a.T @ ubar
        gram = None
    else:
        for _ in range(q):
            f1 = a @ (a.T @ f1)
            passes += 2
        ubar_in = f1
        ubar, fl = oracle_orth(f1)
        flags.append(fl)
        f2 = a.T @ f1
        gram = ubar.T @ f1
    passes += 1
    vbar, fl = oracle_orth(f2)
    flags.append(fl)
    truncated = False
    pinv_kappa = 1.0  # κ₂ of the pseudoinverted gram over its kept singular values (1: no pinv)
    if pass_efficient:
        core = f2.T @ vbar
        if gram is not None:
            u, s, vh = np.linalg.svd(gram, full_matrices=False)
            if s[0] == 0.0:
                core, truncated = np.zeros_like(core), True
            else:
                keep = s > PINV_RTOL * s[0]
                inv = np.zeros_like(s)
                inv[keep] = 1.0 / s[keep]
                core, truncated = (u * inv) @ (vh @ core), bool(not keep.all())
                pinv_kappa = float(s[0] / s[keep][-1])
    else:
        core = ubar.T @ (a @ vbar)
        passes += 1
    qc, t, perm = oracle_column_pivoted_qr(core)
    # |diag R| of the inputs to the last orth of each basis: the forward error
    # of Ū's / V̄'s column j is ~ u·R_00/R_jj (what parity tolerances scale by)
    rd1 = np.abs(np.diag(oracle_qr(ubar_in)[1]))
    rd2 = np.abs(np.diag(oracle_qr(f2)[1]))
    return {"u": ubar @ qc, "t": t, "v": vbar[:, perm], "perm": perm, "omega": omega, "passes": passes,
            "pinv_truncated": truncated, "rank_flags": flags, "core": core, "rdiag_ubar": rd1, "rdiag_vbar": rd2,
            "pinv_kappa": pinv_kappa}
