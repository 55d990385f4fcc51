"""Intrinsic rounding sensitivity of the reference's PbP-QLP factors, per
column, at full BASELINE size (run on the GPU box):

  python tools/noise_floor.py --workload cfg5 --d 512 --q 0 [--out gpurun_out/nf.npz]

Three factorizations of the SAME A and Φ:
  ref  the oracle (bitwise the reference's call sequence, numpy/OpenBLAS);
  alt  the same call sequence with every product's summation split in two
       halves of its reduction dimension (a legitimate reordering: each
       product is still a backward-stable FP64 dgemm);
  alt2 the call sequence with every QR applied to a row-permuted copy
       (LAPACK's own rounding perturbed; exact factors unchanged);
  alt3 every product summed in a random order and every QR row-permuted
       (a different, equally valid FP64 evaluation of the whole sequence);
  gpu  this package's pbp_qlp on the device (default QR method);
  hh   the same with the blocked Householder QR kernel forced.
Per column j it records the sign-normalised column errors of Q and P and
|ΔL_jj|/L_jj of alt-vs-ref and gpu-vs-ref, with κ_j = L_00/L_jj and the
relative gap to the neighbouring L values — the data behind the parity
tolerance of tests/test_gpu_configs.py."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.pbp_qlp_oracle import column_relative_error, oracle_gaussian, oracle_pbp_qlp, oracle_qr  # noqa: E402


def reordered_pbp_qlp(a, d, q, phi):
    """oracle_pbp_qlp with the reduction of every product split in two."""
    n1, n2 = a.shape
    h1, h2 = n1 // 2, n2 // 2

    def apply(x):  # a @ x, reduction over n2
        return a[:, :h2] @ x[:h2] + a[:, h2:] @ x[h2:]

    def apply_t(x):  # a.T @ x, reduction over n1
        return a[:h1].T @ x[:h1] + a[h1:].T @ x[h1:]

    pbar, _ = oracle_qr(apply_t(phi))
    for _ in range(q):
        pbar, _ = oracle_qr(apply(pbar))
        pbar, _ = oracle_qr(apply_t(pbar))
    qf, r = oracle_qr(apply(pbar))
    w, rt = oracle_qr(r.T)
    return {"q": qf, "l": np.tril(rt.T), "p": pbar @ w}


def permuted_qr_pbp_qlp(a, d, q, phi, seed=12345):
    """oracle_pbp_qlp whose every QR factors a row-permuted copy (Q = P·Q_perm):
    the exact factors are unchanged, LAPACK's rounding is not — the
    reference's own QR noise, which `alt` (same QR inputs up to GEMM
    rounding) cannot show."""
    rng = np.random.default_rng(seed)

    def qr(m):
        perm = rng.permutation(m.shape[0])
        qp, r = oracle_qr(m[perm])
        out = np.empty_like(qp)
        out[perm] = qp
        return out, r

    pbar, _ = qr(a.T @ phi)
    for _ in range(q):
        pbar, _ = qr(a @ pbar)
        pbar, _ = qr(a.T @ pbar)
    qf, r = qr(a @ pbar)
    w, rt = oracle_qr(r.T)
    return {"q": qf, "l": np.tril(rt.T), "p": pbar @ w}


def shuffled_pbp_qlp(a, d, q, phi, seed=777):
    """Every product summed in a random order (rows and columns of A
    permuted, results un-permuted) and every QR on a row-permuted copy: a
    different but equally valid FP64 evaluation order of the whole call
    sequence, like any reimplementation (a GPU's blocked DMMA sums) has."""
    rng = np.random.default_rng(seed)
    n1, n2 = a.shape
    p1, p2 = rng.permutation(n1), rng.permutation(n2)
    ap = a[p1][:, p2]

    def apply_t(x):  # aᵀx, summed over rows in p1 order
        out = np.empty((n2, x.shape[1]))
        out[p2] = ap.T @ x[p1]
        return out

    def apply(y):  # a·y, summed over columns in p2 order
        out = np.empty((n1, y.shape[1]))
        out[p1] = ap @ y[p2]
        return out

    def qr(m):
        perm = rng.permutation(m.shape[0])
        qp, r = oracle_qr(m[perm])
        out = np.empty_like(qp)
        out[perm] = qp
        return out, r

    pbar, _ = qr(apply_t(phi))
    for _ in range(q):
        pbar, _ = qr(apply(pbar))
        pbar, _ = qr(apply_t(pbar))
    qf, r = qr(apply(pbar))
    w, rt = oracle_qr(r.T)
    return {"q": qf, "l": np.tril(rt.T), "p": pbar @ w}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--d", type=int, nargs="+", default=[512])
    ap.add_argument("--q", type=int, nargs="+", default=[0])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/noise_floor")
    args = ap.parse_args()
    import torch

    from paper_2103_07245_b200 import pbp_qlp, workloads

    a_dev = workloads.make(args.workload, args.seed, "cuda")
    a = a_dev.cpu().numpy()
    for d in args.d:
        phi = oracle_gaussian(a.shape[0], d, args.seed)
        for q in args.q:
            t0 = time.time()
            ref = oracle_pbp_qlp(a, d, q=q, seed=args.seed, phi=phi)
            alt = reordered_pbp_qlp(a, d, q, phi)
            alt2 = permuted_qr_pbp_qlp(a, d, q, phi)
            alt3 = shuffled_pbp_qlp(a, d, q, phi)
            got = pbp_qlp(a_dev, d, q=q, seed=args.seed)
            gq, gl, gp = (x.cpu().numpy() for x in (got.q_basis, got.l, got.p_basis))
            from paper_2103_07245_b200 import device as D

            ctx = D.context(a_dev.device)
            ctx.set_qr_method(ctx.QR_HOUSEHOLDER)
            try:
                hh = pbp_qlp(a_dev, d, q=q, seed=args.seed)
            finally:
                ctx.set_qr_method(ctx.QR_AUTO)
            hq, hl, hp = (x.cpu().numpy() for x in (hh.q_basis, hh.l, hh.p_basis))
            lref = np.abs(np.diag(ref["l"]))
            kappa = lref[0] / lref
            gap = np.full(d, np.inf)
            rel = np.abs(np.diff(lref)) / lref[1:]
            gap[1:] = rel
            gap[:-1] = np.minimum(gap[:-1], rel)
            rec = {
                "kappa": kappa, "l": lref, "relgap": gap,
                "alt_q": column_relative_error(alt["q"], ref["q"]), "alt_p": column_relative_error(alt["p"], ref["p"]),
                "alt_l": np.abs(np.abs(np.diag(alt["l"])) - lref) / lref,
                "gpu_q": column_relative_error(gq, ref["q"]), "gpu_p": column_relative_error(gp, ref["p"]),
                "gpu_l": np.abs(np.abs(np.diag(gl)) - lref) / lref,
                "alt2_q": column_relative_error(alt2["q"], ref["q"]),
                "alt2_p": column_relative_error(alt2["p"], ref["p"]),
                "alt2_l": np.abs(np.abs(np.diag(alt2["l"])) - lref) / lref,
                "alt3_q": column_relative_error(alt3["q"], ref["q"]),
                "alt3_p": column_relative_error(alt3["p"], ref["p"]),
                "alt3_l": np.abs(np.abs(np.diag(alt3["l"])) - lref) / lref,
                "hh_q": column_relative_error(hq, ref["q"]), "hh_p": column_relative_error(hp, ref["p"]),
                "hh_l": np.abs(np.abs(np.diag(hl)) - lref) / lref,
            }
            os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
            np.savez(f"{args.out}_{args.workload}_d{d}_q{q}.npz", **rec)
            u = 2.0 ** -53
            for k in ("q", "p", "l"):
                parts = []
                for v in ("gpu", "hh", "alt", "alt2", "alt3"):
                    e = rec[f"{v}_{k}"]
                    parts.append(f"{v} max {e.max():.2e} (col {e.argmax()}, /(u·κ) {np.max(e / (u * kappa)):.1f})")
                print(f"{args.workload} d={d} q={q} {k.upper()}: " + "; ".join(parts), flush=True)
            print(f"  ({time.time() - t0:.0f} s)", flush=True)
            del got, hh
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
