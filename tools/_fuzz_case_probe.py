import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from tests.test_gpu_fuzz import _case
from paper_2103_07245_b200 import device as D, pbp_qlp
from paper_2103_07245_b200.algorithms import clear_plan_cache
dev = torch.device("cuda", 0)
ctx = D.context(dev)
for sd in (369, 366):
    a, d, q, s, r = _case(sd)
    A = torch.from_numpy(a).to(dev)
    for name, m in (("auto", 0), ("chain", 3), ("hh", 1)):
        ctx.set_qr_method(m)
        stats = torch.zeros(4, dtype=torch.int32, device=dev)
        ctx.cholqr_stats(stats)
        f = pbp_qlp(A, d, q=q, seed=s, reorthonormalize=r)
        ctx.cholqr_stats(None)
        gq, gl, gp = (x.cpu().numpy() for x in (f.q_basis, f.l, f.p_basis))
        e = np.linalg.norm(a - gq @ gl @ gp.T) / np.linalg.norm(a)
        print(sd, name, "QtQ", np.abs(gq.T @ gq - np.eye(d)).max(), "PtP", np.abs(gp.T @ gp - np.eye(d)).max(), "recon", e, "stats", stats.tolist(), flush=True)
    ctx.set_qr_method(0)
    # the orth of the sample alone
    c = a.T @ (a @ (a.T @ (a @ (a.T @ __import__("oracle.pbp_qlp_oracle", fromlist=["x"]).oracle_gaussian(a.shape[0], d, s)))))
    for name, m in (("auto", 0), ("hh", 1)):
        ctx.set_qr_method(m)
        t = D.as_kernel_operand(torch.from_numpy(c).to(dev))
        rr = D.empty_matrix(d, d, dev)
        D.householder_qr_(ctx, t, rr)
        qq = t.cpu().numpy()
        print("  orth(sample)", name, c.shape, "QtQ", np.abs(qq.T @ qq - np.eye(d)).max(), flush=True)
    ctx.set_qr_method(0)
