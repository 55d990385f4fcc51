"""Which stage of the GPU pipeline departs from the reference, at full
config-5 size (d = 512, q = 0)?  Each GPU stage gets the CPU's exact input
for that stage, and its output is compared with the CPU's; the noise scale is
the same stage on the CPU with a permuted evaluation order.

   python tools/stage_probe.py [--d 512]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pbp_qlp_oracle import column_relative_error as cre, oracle_gaussian, oracle_qr  # noqa: E402
from paper_2103_07245_b200 import device as D, workloads  # noqa: E402


def perm_qr(m, seed=5):
    rng = np.random.default_rng(seed)
    p = rng.permutation(m.shape[0])
    q, r = oracle_qr(m[p])
    out = np.empty_like(q)
    out[p] = q
    return out, r


def dev_qr(ctx, m, method):
    ctx.set_qr_method(method)
    try:
        t = D.as_kernel_operand(torch.from_numpy(np.ascontiguousarray(m)).to("cuda"))
        r = D.empty_matrix(m.shape[1], m.shape[1], t.device)
        D.householder_qr_(ctx, t, r)
        return t.cpu().numpy(), r.cpu().numpy()
    finally:
        ctx.set_qr_method(ctx.QR_AUTO)


def rep(name, err):
    print(f"  {name:38s} max {err.max():.2e}  median {np.median(err):.2e}  col0 {err[0]:.2e}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=512)
    args = ap.parse_args()
    d = args.d
    ctx = D.context(torch.device("cuda", 0))
    a_dev = workloads.make_cfg5(0, "cuda")
    a = a_dev.cpu().numpy()
    n1, n2 = a.shape
    phi = oracle_gaussian(n1, d, 0)
    # stage 1: C = Aᵀ Φ
    c_cpu = a.T @ phi
    c_gpu = D.gemm(ctx, a_dev, D.as_kernel_operand(torch.from_numpy(phi).cuda()), trans_a=True).cpu().numpy()
    p1 = np.random.default_rng(1).permutation(n1)
    c_alt = a[p1].T @ phi[p1]
    print(f"stage C = AᵀΦ ({n2}x{d})")
    rep("gpu vs cpu", cre(c_gpu, c_cpu))
    rep("cpu permuted-sum vs cpu", cre(c_alt, c_cpu))
    # stage 2: P̄ = orth(C) from the CPU's C
    pb_cpu, _ = oracle_qr(c_cpu)
    pb_alt, _ = perm_qr(c_cpu)
    print("stage P̄ = orth(C_cpu)")
    rep("gpu auto (CholQR2) vs LAPACK", cre(dev_qr(ctx, c_cpu, ctx.QR_AUTO)[0], pb_cpu))
    rep("gpu householder vs LAPACK", cre(dev_qr(ctx, c_cpu, ctx.QR_HOUSEHOLDER)[0], pb_cpu))
    rep("LAPACK row-permuted vs LAPACK", cre(pb_alt, pb_cpu))
    # stage 3: D = A P̄ from the CPU's P̄
    d_cpu = a @ pb_cpu
    d_gpu = D.gemm(ctx, a_dev, D.as_kernel_operand(torch.from_numpy(pb_cpu).cuda()), trans_a=False).cpu().numpy()
    p2 = np.random.default_rng(2).permutation(n2)
    d_alt = a[:, p2] @ pb_cpu[p2]
    print(f"stage D = A·P̄ ({n1}x{d})")
    rep("gpu vs cpu", cre(d_gpu, d_cpu))
    rep("cpu permuted-sum vs cpu", cre(d_alt, d_cpu))
    # stage 4: (Q, R) = qr(D) from the CPU's D
    q_cpu, r_cpu = oracle_qr(d_cpu)
    q_alt, _ = perm_qr(d_cpu)
    print("stage Q = qr(D_cpu)")
    rep("gpu auto vs LAPACK", cre(dev_qr(ctx, d_cpu, ctx.QR_AUTO)[0], q_cpu))
    rep("gpu householder vs LAPACK", cre(dev_qr(ctx, d_cpu, ctx.QR_HOUSEHOLDER)[0], q_cpu))
    rep("LAPACK row-permuted vs LAPACK", cre(q_alt, q_cpu))
    # stage 5: second stage from the CPU's R
    w_cpu, rt_cpu = oracle_qr(r_cpu.T)
    wg, lg = D.second_stage(ctx, D.as_kernel_operand(torch.from_numpy(r_cpu).cuda()))
    w_alt, _ = perm_qr(r_cpu.T)
    print("stage W = qr(Rᵀ)")
    rep("gpu vs LAPACK", cre(wg.cpu().numpy(), w_cpu))
    rep("LAPACK row-permuted vs LAPACK", cre(w_alt, w_cpu))


if __name__ == "__main__":
    main()
