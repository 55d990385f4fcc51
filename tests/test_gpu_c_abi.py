"""The C ABI used from a non-Python host: examples/c_host.c (plain C against
include/pbq.h + the CUDA runtime) is compiled with gcc, run on a seeded
problem, and its factors must equal the Python drop-in's bit for bit (same
kernels, same inputs) and match the oracle (reference algorithms.py:209-260)."""
import os
import subprocess

import numpy as np
import pytest

from oracle.pbp_qlp_oracle import column_relative_error, conditioning_tolerance, oracle_pbp_qlp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "c_host")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    lib = os.path.join(ROOT, "paper_2103_07245_b200")
    cmd = ["gcc", "-std=c11", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
           os.path.join(ROOT, "examples", "c_host.c"), "-o", exe, "-L", lib, "-lpbq", "-L",
           os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{lib}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_host_matches_python_and_oracle(cuda, tmp_path):
    from paper_2103_07245_b200 import pbp_qlp

    exe = _build(tmp_path)
    rng = np.random.default_rng(31)
    n1, n2, d, q, seed = 700, 450, 40, 1, 12345
    a = rng.standard_normal((n1, 60)) @ rng.standard_normal((60, n2)) / 8 + 1e-3 * rng.standard_normal((n1, n2))
    a_path, out_path = tmp_path / "a.bin", tmp_path / "out.bin"
    a.tofile(a_path)
    res = subprocess.run([exe, str(a_path), str(n1), str(n2), str(d), str(q), str(seed), str(out_path)],
                         capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    raw = np.fromfile(out_path, dtype=np.uint8)
    status = raw[:4].view(np.int32)[0]
    flags = raw[4:4 + 4 * (2 * q + 1)].view(np.int32)
    vals = raw[4 + 4 * (2 * q + 1):].view(np.float64)
    sizes = [n1 * d, d * d, n2 * d, d * d, n1 * d]
    parts, off = [], 0
    for s in sizes:
        parts.append(vals[off:off + s])
        off += s
    qf, l, p, r, phi = (parts[0].reshape(n1, d), parts[1].reshape(d, d), parts[2].reshape(n2, d),
                        parts[3].reshape(d, d), parts[4].reshape(n1, d))
    assert status == 0 and not flags.any()
    f = pbp_qlp(a, d, q=q, seed=seed)
    for x, y in ((qf, f.q_basis), (l, f.l), (p, f.p_basis), (r, f.first_stage_r), (phi, f.sketch.test_matrix)):
        assert np.array_equal(x, y)
    ref = oracle_pbp_qlp(a, d, q=q, seed=seed)
    tol = conditioning_tolerance(ref["l"])
    assert np.all(column_relative_error(qf, ref["q"]) <= tol)
    assert np.all(column_relative_error(p, ref["p"]) <= tol)
    assert np.array_equal(phi, ref["phi"])
