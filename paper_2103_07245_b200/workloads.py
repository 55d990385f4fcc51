"""Synthetic inputs for the BASELINE.json configurations.

BASELINE names no public dataset; every config is a seeded synthetic matrix
with the stated shape and spectrum.  Small configs (1–2) are drawn with numpy
exactly as the recipe says (Haar factors from the reference's sign-fixed QR,
linalg.py:142); large configs (3–5) are drawn on the GPU with a seeded torch
generator (the recipe allows "a seeded torch CUDA generator for configs 4–5")
and copied to the host once, so the same bytes feed the GPU path and the CPU
oracle.  Building A is input preparation, not the PbP-QLP path, so it may use
torch/cuBLAS.
"""
import math

import numpy as np
import torch

CONFIGS = {
    "cfg1": dict(n1=1000, n2=1000, d=40, q=0),
    "cfg2": dict(n1=4000, n2=4000, d=100, q=0),
    "cfg3": dict(n1=20000, n2=10000, d=256, q=1),
    "cfg4": dict(n1=200000, n2=8192, d=512, q=1),
    "cfg5": dict(n1=65536, n2=16384, d=256, q=0),
}


def _haar(n, rng):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def make_cfg1(seed=0):
    rng = np.random.Generator(np.random.Philox(key=seed))
    u, v = _haar(1000, rng), _haar(1000, rng)
    sigma = np.concatenate([np.ones(20), np.full(980, 1e-3)])
    return (u * sigma) @ v.T + 1e-6 * rng.standard_normal((1000, 1000))


def make_cfg2(seed=0):
    rng = np.random.Generator(np.random.Philox(key=seed))
    u, v = _haar(4000, rng), _haar(4000, rng)
    sigma = np.arange(1, 4001, dtype=np.float64) ** -2.0
    return (u * sigma) @ v.T


def _gen(seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def make_cfg3(seed=0, device="cuda"):
    """A = G1·G2ᵀ/√200 + 1e-3·N, 20000×10000, on ``device`` (torch float64)."""
    g = _gen(seed, device)
    g1 = torch.randn(20000, 200, dtype=torch.float64, device=device, generator=g)
    g2 = torch.randn(10000, 200, dtype=torch.float64, device=device, generator=g)
    a = torch.randn(20000, 10000, dtype=torch.float64, device=device, generator=g)
    a.mul_(1e-3).addmm_(g1, g2.T, alpha=1.0 / math.sqrt(200.0))
    return a


def make_cfg4(seed=0, device="cuda", rows=None, row_offset=0):
    """A = (G_U·diag σ)·G_Vᵀ/√n1, σ_i = 10^(-i/128); 200000×8192 (optionally a row block)."""
    n1, n2, k = 200000, 8192, 1024
    rows = n1 - row_offset if rows is None else rows
    g = _gen(seed, device)
    gv = torch.randn(n2, k, dtype=torch.float64, device=device, generator=g)
    sigma = 10.0 ** (-torch.arange(k, dtype=torch.float64, device=device) / 128.0)
    g.manual_seed(seed + 1 + row_offset)
    gu = torch.randn(rows, k, dtype=torch.float64, device=device, generator=g)
    return (gu * sigma) @ gv.T / math.sqrt(n1)


def make_cfg5(seed=0, device="cuda"):
    """65536×16384, σ_i = e^(-i/40) over inner dim 2048, + 1e-8·N."""
    n1, n2, k = 65536, 16384, 2048
    g = _gen(seed, device)
    gu = torch.randn(n1, k, dtype=torch.float64, device=device, generator=g)
    gv = torch.randn(n2, k, dtype=torch.float64, device=device, generator=g)
    sigma = torch.exp(-torch.arange(k, dtype=torch.float64, device=device) / 40.0)
    a = torch.randn(n1, n2, dtype=torch.float64, device=device, generator=g)
    a.mul_(1e-8).addmm_(gu * sigma, gv.T, alpha=1.0 / math.sqrt(n1))
    return a


def make(name, seed=0, device="cuda"):
    if name == "cfg1":
        return torch.from_numpy(make_cfg1(seed)).to(device)
    if name == "cfg2":
        return torch.from_numpy(make_cfg2(seed)).to(device)
    return {"cfg3": make_cfg3, "cfg4": make_cfg4, "cfg5": make_cfg5}[name](seed, device)
