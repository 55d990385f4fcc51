"""Forward error of the FP64 GEMMs against an extended-precision reference
(numpy longdouble, 64-bit significand), for libpbq's DMMA GEMM, OpenBLAS
(numpy), and torch/cuBLAS DGEMM, on AᵀX shapes with long reductions.

  python tools/gemm_accuracy.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07245_b200 import device as D  # noqa: E402


def exact_tn(a, x):
    al, xl = a.astype(np.longdouble), x.astype(np.longdouble)
    return al.T @ xl


def main():
    dev = torch.device("cuda", 0)
    ctx = D.context(dev)
    rng = np.random.default_rng(0)
    for K, M, N in [(65536, 64, 16), (16384, 128, 16), (4096, 256, 32)]:
        a = rng.standard_normal((K, M))
        x = rng.standard_normal((K, N))
        ex = exact_tn(a, x)
        scale = (np.abs(a).T @ np.abs(x)).astype(np.longdouble)
        def err(c):
            return float(np.max(np.abs(c.astype(np.longdouble) - ex) / scale)), float(np.median(np.abs(c.astype(np.longdouble) - ex) / scale))
        c_blas = a.T @ x
        A, X = D.as_kernel_operand(torch.from_numpy(a).to(dev)), D.as_kernel_operand(torch.from_numpy(x).to(dev))
        c_pbq = D.gemm(ctx, A, X, trans_a=True).cpu().numpy()
        c_cub = (torch.from_numpy(a).to(dev).T @ torch.from_numpy(x).to(dev)).cpu().numpy()
        c_nn = D.gemm(ctx, D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)), X,
                      trans_a=False).cpu().numpy()
        print(f"K={K} M={M} N={N}  (max, median) |err|/(|a|ᵀ|x|) in units of u=2^-53:")
        for name, c in (("openblas", c_blas), ("libpbq TN", c_pbq), ("libpbq NN", c_nn), ("cublas", c_cub)):
            mx, md = err(c)
            print(f"   {name:10s} max {mx / 2**-53:9.2f} u   median {md / 2**-53:8.3f} u")


def big(shapes=((65536, 16384, 512), (20000, 10000, 256))):
    """Full-size AᵀX (many output tiles: each tile's K range is accumulated by
    one or two CTAs) — error measured on a 1024×16 corner of C against the
    extended-precision sum."""
    dev = torch.device("cuda", 0)
    ctx = D.context(dev)
    rng = np.random.default_rng(1)
    for K, M, N in shapes:
        a = rng.standard_normal((K, M))
        x = rng.standard_normal((K, N))
        sub_m, sub_n = 1024, 16
        ex = a[:, :sub_m].astype(np.longdouble).T @ x[:, :sub_n].astype(np.longdouble)
        scale = (np.abs(a[:, :sub_m]).T @ np.abs(x[:, :sub_n])).astype(np.longdouble)
        c_blas = (a[:, :sub_m].T @ x)[:, :sub_n]
        A, X = D.as_kernel_operand(torch.from_numpy(a).to(dev)), D.as_kernel_operand(torch.from_numpy(x).to(dev))
        c_pbq = D.gemm(ctx, A, X, trans_a=True)[:sub_m, :sub_n].cpu().numpy()
        print(f"K={K} M={M} N={N} (full-size C, {sub_m}x{sub_n} corner checked):")
        for name, c in (("openblas", c_blas), ("libpbq TN", c_pbq)):
            e = np.abs(c.astype(np.longdouble) - ex) / scale
            print(f"   {name:10s} max {float(e.max()) / 2**-53:9.2f} u   median {float(np.median(e)) / 2**-53:8.3f} u",
                  flush=True)
        del A, X
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
    big()
