"""Probe one r_svd fuzz case: per-index error of device vs reference vs alt."""
import sys
import numpy as np
import torch
from oracle.pbp_qlp_oracle import oracle_r_svd
from paper_2103_07245_b200.rsvd import r_svd

for seed in map(int, sys.argv[1:]):
    rng = np.random.default_rng(8000 + seed)
    n1, n2 = int(rng.integers(30, 1500)), int(rng.integers(30, 1500))
    kmin = min(n1, n2)
    d = int(rng.integers(1, min(kmin, 260) + 1))
    q = int(rng.integers(0, 3))
    reorth = bool(rng.random() < 0.8)
    r = int(min(kmin, d + rng.integers(0, 30)))
    u, _ = np.linalg.qr(rng.standard_normal((n1, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n2, r)))
    decay = float(rng.choice([5.0, 30.0, 1e9]))
    a = (u * np.exp(-np.arange(r) / decay)) @ v.T + 1e-8 * rng.standard_normal((n1, n2))
    sd = int(rng.integers(0, 2**31))
    got = r_svd(a, d, q=q, seed=sd, reorthonormalize=reorth)
    ref = oracle_r_svd(a, d, q=q, seed=sd, reorthonormalize=reorth)
    perm = np.random.default_rng(seed).permutation(n1)
    alt = oracle_r_svd(a[perm], d, q=q, seed=sd, reorthonormalize=reorth)
    s, sr, sa = np.asarray(got.s), np.asarray(ref["s"]), np.asarray(alt["s"])
    st = np.linalg.svd(a, compute_uv=False)[:d]
    rel = lambda x, y: np.abs(x - y) / y
    print("seed", seed, a.shape, d, q, reorth, "decay", decay, "r", r)
    e, ea = rel(s, sr), rel(sa, sr)
    idx = np.argsort(-e / np.maximum(np.maximum.accumulate(ea), 1e-16))[:6]
    for j in sorted(idx):
        print(f"  j={j:3d} s/s0={sr[j]/sr[0]:.2e} dev-ref={e[j]:.2e} alt-ref={ea[j]:.2e} "
              f"dev-true={rel(s, st)[j]:.2e} ref-true={rel(sr, st)[j]:.2e} alt-true={rel(sa, st)[j]:.2e}")
    print("  max over j: dev-true", rel(s, st).max(), "ref-true", rel(sr, st).max(), "alt-true", rel(sa, st).max())
