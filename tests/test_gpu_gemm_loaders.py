"""The three shared-memory loaders of the FP64 DMMA GEMM give the same products.

libpbq stages the GEMM's k-blocks with the Tensor Memory Accelerator by
default: one 3-D copy per operand and k-block when the row length is a
multiple of 16 doubles, else one 2-D copy per 16-column group.
PBQ_TMA_NO3D=1 forces the 2-D copies and PBQ_GEMM_LOADER=cpasync the
per-thread cp.async ring (the variant measured against in DESIGN.md §3).  The
switch is read once per process, so each loader runs in its own subprocess;
the products must agree with numpy within the FP64 summation-order bound and
the nonfinite scan must fire under every loader.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2103_07245_b200 import device as D
dev = torch.device("cuda", 0)
ctx = D.context(dev)
out = {{}}
for (M, N, K, trans) in {shapes!r}:
    rng = np.random.default_rng(M * 7 + N * 3 + K + trans)
    a = rng.standard_normal((K, M) if trans else (M, K))
    b = rng.standard_normal((K, N))
    A = D.empty_matrix(a.shape[0], a.shape[1], dev); A.copy_(torch.from_numpy(a))
    B = D.empty_matrix(b.shape[0], b.shape[1], dev); B.copy_(torch.from_numpy(b))
    out[f"{{M}}x{{N}}x{{K}}x{{int(trans)}}"] = D.gemm(ctx, A, B, trans_a=trans).cpu().numpy().tolist()
a = np.ones((640, 96)); a[333, 17] = np.nan
A = D.empty_matrix(640, 96, dev); A.copy_(torch.from_numpy(a))
B = D.empty_matrix(640, 64, dev); B.fill_(1.0)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
D.gemm(ctx, A, B, trans_a=True, nonfinite=flag)
out["nonfinite"] = int(flag.item())
print(json.dumps(out))
"""

SHAPES = [(256, 256, 4096, True), (10000, 256, 2000, True), (2000, 256, 10000, False), (333, 100, 777, True),
          (777, 65, 1000, False), (4096, 512, 512, False), (130, 40, 1000, True)]


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, shapes=SHAPES)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    return json.loads(res.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("env", [{}, {"PBQ_TMA_NO3D": "1"}, {"PBQ_GEMM_LOADER": "cpasync"}],
                         ids=["tma3d", "tma2d", "cpasync"])
def test_gemm_loader_matches_fp64(cuda, env):
    got = _run(env)
    assert got["nonfinite"] == 1
    for (M, N, K, trans) in SHAPES:
        rng = np.random.default_rng(M * 7 + N * 3 + K + trans)
        a = rng.standard_normal((K, M) if trans else (M, K))
        b = rng.standard_normal((K, N))
        op = a.T if trans else a
        ref = op @ b
        bound = 4 * K * 2.0**-53 * (np.abs(op) @ np.abs(b))
        c = np.array(got[f"{M}x{N}x{K}x{int(trans)}"])
        assert np.all(np.abs(c - ref) <= bound + 1e-300), (M, N, K, trans)
