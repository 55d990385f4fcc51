"""The diagonal 32×32 Cholesky + inverse of the factor kernel runs on two
warps (cq_chol_inv32_2warp: R part and R⁻ᵀ part on separate warps, handed
over through named barriers); PBQ_CHOL_1WARP=1 selects the single-warp
variant.  Both perform the same operations on every element, so the QR
results must be bitwise identical (the switch is read once per process: the
single-warp run happens in a subprocess)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2103_07245_b200 import device as D
dev = torch.device("cuda", 0)
ctx = D.context(dev)
out = []
for (m, n, seed) in {shapes!r}:
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((m, n)) * np.logspace(0, -3, n)
    t = D.empty_matrix(m, n, dev); t.copy_(torch.from_numpy(x))
    r = D.empty_matrix(n, n, dev)
    D.householder_qr_(ctx, t, r, want_q=True)
    out += [t.cpu().numpy(), r.cpu().numpy()]
np.savez({path!r}, *out)
"""
SHAPES = [(4000, 256, 1), (3000, 100, 2), (9000, 512, 3), (500, 40, 4)]


def _run(env_extra, path):
    env = dict(os.environ)
    env.update(env_extra)
    res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, shapes=SHAPES, path=str(path))], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    z = np.load(path)
    return [z[f"arr_{i}"] for i in range(len(z.files))]


def test_two_warp_and_one_warp_cholesky_agree_bitwise(cuda, tmp_path):
    two = _run({}, tmp_path / "two.npz")
    one = _run({"PBQ_CHOL_1WARP": "1"}, tmp_path / "one.npz")
    for a, b in zip(two, one):
        assert np.array_equal(a, b)
