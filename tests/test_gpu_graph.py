"""The whole PbP-QLP pipeline as one CUDA graph (PbpQlpPlan.capture / replay):
every kernel of a factorization — sketch, passes, QR chains, second stage —
recorded once and replayed with new seeds (the sketch reads its key from
device memory, pbq_problem.seed_dev).  A replay must give the same bits as
the stream-ordered run with the same seed, and the oracle's factors."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n1,n2,d,q", [(600, 400, 48, 1), (1000, 1000, 40, 0), (2000, 1500, 130, 2)])
def test_graph_replay_matches_stream_run(cuda, n1, n2, d, q):
    from paper_2103_07245_b200 import PbpQlpPlan
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(n1 + d)
    a_np = rng.standard_normal((n1, 50)) @ rng.standard_normal((50, n2)) + 1e-3 * rng.standard_normal((n1, n2))
    a = D.as_kernel_operand(torch.from_numpy(a_np).to(cuda))
    plan = PbpQlpPlan(n1, n2, d, q, device=cuda)
    ref = {}
    for seed in (3, 2**70 + 5):
        plan.run(a, seed=seed)
        plan.finish()
        ref[seed] = [t.clone() for t in (plan.Q, plan.L, plan.P, plan.R, plan.PHI)]
    plan.capture(a)
    assert plan.graph_launches > 10
    for seed in (3, 2**70 + 5, 3):
        plan.replay(seed)
        plan.finish()
        for got, want in zip((plan.Q, plan.L, plan.P, plan.R, plan.PHI), ref[seed]):
            assert torch.equal(got, want)
    # stream-ordered runs after the capture read their own seed again
    plan.run(a, seed=2**70 + 5)
    plan.finish()
    assert torch.equal(plan.PHI, ref[2**70 + 5][4])


def test_graph_replay_matches_oracle(cuda):
    from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp
    from paper_2103_07245_b200 import PbpQlpPlan
    from paper_2103_07245_b200 import device as D

    rng = np.random.default_rng(5)
    a_np = rng.standard_normal((1500, 60)) @ rng.standard_normal((60, 700)) / 8 + 1e-3 * rng.standard_normal((1500, 700))
    a = D.as_kernel_operand(torch.from_numpy(a_np).to(cuda))
    plan = PbpQlpPlan(1500, 700, 48, 1, device=cuda)
    plan.capture(a)
    plan.replay(9)
    plan.finish()
    ref = oracle_pbp_qlp(a_np, 48, q=1, seed=9)
    tol = conditioning_tolerance(ref["l"], strict=1e-10)
    assert np.all(column_relative_error(plan.Q.cpu().numpy(), ref["q"]) <= tol)
    assert np.all(column_relative_error(plan.P.cpu().numpy(), ref["p"]) <= tol)


def test_clear_error_after_failed_capture(cuda):
    """A stream capture invalidated by an uncapturable operation leaves its
    error as the thread's CUDA last-error; pbq_clear_error resets it so the
    next library call (stream-ordered) runs (bench.py's N > 1 capture
    fallback relies on this).  Run in a subprocess: a failed capture also
    leaves torch's generator bookkeeping mid-capture for the rest of the
    process."""
    import os
    import subprocess
    import sys

    code = (
        "import torch, sys\n"
        "sys.path.insert(0, %r)\n"
        "from paper_2103_07245_b200 import device as D\n"
        "dev = torch.device('cuda', 0); ctx = D.context(dev)\n"
        "g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(dev)\n"
        "out = torch.empty(64, 8, dtype=torch.float64, device=dev)\n"
        "try:\n"
        "    with torch.cuda.graph(g, stream=s):\n"
        "        D.gaussian(ctx, 64, 8, 1, dev, out=out)\n"
        "        torch.cuda.synchronize()\n"
        "    raise SystemExit('capture did not fail')\n"
        "except RuntimeError:\n"
        "    pass\n"
        "torch.cuda.synchronize()\n"
        "ctx.clear_error()\n"
        "phi = D.gaussian(ctx, 64, 8, 1, dev)\n"
        "torch.cuda.synchronize()\n"
        "assert torch.isfinite(phi).all()\n"
        "print('RECOVERED')\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0 and "RECOVERED" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]
