import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"
# the stock reference installed by tools/install_reference.sh (git-ignored;
# travels to the GPU box, where /root/reference does not exist)
REFERENCE_INSTALL = os.path.join(ROOT, "baseline", "_ref")


def reference_path():
    """Directory to put on sys.path to import the reference ``pbpqlp``, or None."""
    for cand in (REFERENCE_SRC, REFERENCE_INSTALL):
        if os.path.isfile(os.path.join(cand, "pbpqlp", "__init__.py")):
            return cand
    return None


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libpbq.so")
    config.addinivalue_line("markers", "slow: full-size BASELINE configurations")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_07245_b200 import _lib

    _lib.load()  # fail loudly if the extension is missing on a GPU box
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def reference_pkg():
    """The reference package: /root/reference in the build container, the
    stock install under baseline/_ref on the GPU box."""
    path = reference_path()
    if path is None:
        pytest.skip("reference not present (run tools/install_reference.sh)")
    if path not in sys.path:
        sys.path.insert(0, path)
    import pbpqlp

    return pbpqlp


@pytest.fixture(params=["auto", "chain", "householder"])
def qr_method(request, cuda):
    """Run a test under each QR method: the default guarded Cholesky-QR2
    (the single-launch kernel of cholqr_small_f64.cuh where it applies, else
    the chain of cholqr_f64.cuh), the chain forced, and the blocked
    Householder kernel (qr_f64.cuh)."""
    from paper_2103_07245_b200 import device as D

    ctx = D.context(cuda)
    ctx.set_qr_method({"auto": ctx.QR_AUTO, "chain": ctx.QR_CHOLQR_CHAIN, "householder": ctx.QR_HOUSEHOLDER}[request.param])
    yield request.param
    ctx.set_qr_method(ctx.QR_AUTO)


@pytest.fixture(autouse=True)
def _dirty_device_memory(request):
    """Every GPU test starts with NaN-filled memory in torch's caching
    allocator, so a workspace the library forgets to initialise is caught
    (freshly mapped device memory is zero and would hide it)."""
    if request.node.get_closest_marker("gpu") is None:
        yield
        return
    import torch

    if torch.cuda.is_available():
        junk = torch.full((64 << 20,), float("nan"), dtype=torch.float64, device="cuda:0")  # 512 MB
        del junk
    yield
