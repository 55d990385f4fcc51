"""Accuracy study: whole-matrix Cholesky-QR2 (explicit triangular inverses,
as the device computes it) in place of Householder QR inside PbP-QLP.

For full column rank, the thin QR with diag(R) > 0 is unique, so CholQR2
targets exactly the reference's (Q, R) (linalg.py:106-115 after _fix_signs).
This prints, per test family, max(err_j / tol_j) of the end-to-end factors
under the parity tolerance of tests/test_gpu_configs.py, and the κ₁(R₁)
estimate of every QR call (the device's fallback trigger).

    python tools/proto_cholqr2_full.py [--big]
"""
import math
import sys

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle.pbp_qlp_oracle import (column_relative_error, conditioning_tolerance,  # noqa: E402
                                   oracle_gaussian, oracle_pbp_qlp, oracle_qr)

LOG = []


def tri_inv(r):
    return sla.solve_triangular(r, np.eye(r.shape[0]), lower=False)


def cholqr2(a, kmax):
    g = a.T @ a
    try:
        r1 = np.linalg.cholesky(g).T
    except np.linalg.LinAlgError:
        LOG.append(("chol-fail", a.shape, np.inf))
        return oracle_qr(a)
    r1i = tri_inv(r1)
    k1 = np.linalg.norm(r1, 1) * np.linalg.norm(r1i, 1)
    if not np.isfinite(k1) or k1 > kmax:
        LOG.append(("fallback", a.shape, k1))
        return oracle_qr(a)
    q1 = a @ r1i
    g2 = q1.T @ q1
    r2 = np.linalg.cholesky(g2).T
    q = q1 @ tri_inv(r2)
    r = r2 @ r1
    LOG.append(("cholqr2", a.shape, k1))
    return q, np.triu(r)


def pipeline(a, d, q, seed, qr):
    phi = oracle_gaussian(a.shape[0], d, seed)
    c = a.T @ phi
    pbar, _ = qr(c)
    for _ in range(q):
        pbar, _ = qr(a @ pbar)
        pbar, _ = qr(a.T @ pbar)
    qf, rf = qr(a @ pbar)
    w, rt = qr(rf.T)
    return qf, np.tril(rt.T), pbar @ w


def study(name, a, d, q, seed, kmax):
    LOG.clear()
    ref = oracle_pbp_qlp(a, d, q=q, seed=seed)
    gq, gl, gp = pipeline(a, d, q, seed, lambda m: cholqr2(m, kmax))
    tol = conditioning_tolerance(ref["l"])
    rq = (column_relative_error(gq, ref["q"]) / tol).max()
    rp = (column_relative_error(gp, ref["p"]) / tol).max()
    lref = np.abs(np.diag(ref["l"]))
    rl = (np.abs(np.abs(np.diag(gl)) - lref) / lref / conditioning_tolerance(ref["l"], factor=16.0)).max()
    calls = ", ".join(f"{k}{s[0]}x{s[1]}:{v:.1e}" for k, s, v in LOG)
    print(f"{name:28s} Q {rq:8.2e}  P {rp:8.2e}  L {rl:8.2e}  | {calls}", flush=True)


def cfg5_analog(n1, n2, k, seed):
    rng = np.random.default_rng(seed)
    gu = rng.standard_normal((n1, k))
    gv = rng.standard_normal((n2, k))
    sigma = np.exp(-np.arange(k) / 40.0)
    return (gu * sigma) @ gv.T / math.sqrt(n1) + 1e-8 * rng.standard_normal((n1, n2))


def main():
    kmax = float(next((x.split("=")[1] for x in sys.argv if x.startswith("--kmax=")), 1e6))
    big = "--big" in sys.argv
    from paper_2103_07245_b200 import workloads

    study("cfg1", workloads.make_cfg1(0), 40, 0, 0, kmax)
    study("cfg2", workloads.make_cfg2(0), 100, 0, 0, kmax)
    rng = np.random.default_rng(23)
    a = rng.standard_normal((700, 40)) @ rng.standard_normal((40, 500)) + 1e-2 * rng.standard_normal((700, 500))
    study("many_power_iters q=5", a, 48, 5, 8, kmax)
    study("full rank 300x200 d=200", np.random.default_rng(21).standard_normal((300, 200)), 200, 1, 4, kmax)
    n1, n2, k = (16384, 4096, 2048) if big else (4096, 1024, 512)
    a5 = cfg5_analog(n1, n2, k, 5)
    for d, q in [(64, 0), (256, 2), (512, 0)] + ([(1024, 2)] if big else []):
        study(f"cfg5 analog d={d} q={q}", a5, d, q, 3, kmax)
    if big:
        import torch

        a3 = workloads.make_cfg3(0, "cpu").numpy()
        study("cfg3 full", a3, 256, 1, 0, kmax)


if __name__ == "__main__":
    main()
