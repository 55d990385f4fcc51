"""The drop-in boundary: the C ABI declared in include/pbq.h is exported by
libpbq.so, the library loads without a GPU, and the Python host layer keeps
the reference's argument contract (/root/reference/pkg/src/pbpqlp/
validation.py:17-61, algorithms.py:187-190, 239-241) — checked on CPU."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pbq.h")
MANIFEST = json.load(open(os.path.join(ROOT, "tests", "golden", "manifest.json")))


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pbq_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2103_07245_b200 import _lib, build

    build.build()  # no-op when up to date; nvcc cross-compiles without a GPU
    return _lib.load()


def test_header_symbols_exported(lib):
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/pbq.h but not exported"
    from paper_2103_07245_b200 import _lib

    assert sorted(_lib.EXPORTED) == declared


def test_ctx_create_fails_cleanly_without_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    assert lib.pbq_ctx_create(0, ctypes.byref(h)) != 0
    assert not h.value


def test_no_cpu_fallback_without_gpu():
    import torch

    from paper_2103_07245_b200 import DeviceError, pbp_qlp

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(DeviceError):
        pbp_qlp(np.eye(8), 2)


_nan = np.ones((6, 5))
_nan[2, 3] = np.nan
ERROR_CASES = {
    "d_zero": (([[1.0, 2.0], [3.0, 4.0]], 0), {}),
    "d_too_big": (([[1.0, 2.0], [3.0, 4.0]], 3), {}),
    "d_float": (([[1.0, 2.0], [3.0, 4.0]], 2.0), {}),
    "d_bool": (([[1.0, 2.0], [3.0, 4.0]], True), {}),
    "q_negative": (([[1.0, 2.0], [3.0, 4.0]], 1), {"q": -1}),
    "q_float": (([[1.0, 2.0], [3.0, 4.0]], 1), {"q": 1.5}),
    "q_bool": (([[1.0, 2.0], [3.0, 4.0]], 1), {"q": True}),
    "a_1d": (([1.0, 2.0, 3.0], 1), {}),
    "a_3d": ((np.ones((2, 2, 2)), 1), {}),
    "a_empty": ((np.ones((0, 3)), 1), {}),
    "a_string": (("abc", 1), {}),
    "a_nan_and_bad_d": ((_nan, 9), {}),
}


@pytest.mark.parametrize("label", sorted(ERROR_CASES))
def test_error_contract_matches_reference(label):
    """Same exception class as the reference for every invalid argument that
    is rejected before the device is touched."""
    import paper_2103_07245_b200 as P

    args, kwargs = ERROR_CASES[label]
    expected = MANIFEST["errors"][label]
    with pytest.raises(getattr(P, expected)):
        P.pbp_qlp(*args, **kwargs)


def test_exception_hierarchy():
    import paper_2103_07245_b200 as P

    assert issubclass(P.DimensionError, P.ParameterError)
    assert issubclass(P.ParameterError, ValueError)
    assert issubclass(P.MatrixInputError, ValueError)
    assert issubclass(P.RankDeficiencyWarning, UserWarning)


def test_flop_model_matches_baseline():
    """F(n1, n2, d, q) of SURVEY.md §8d / BASELINE.md §4."""
    from paper_2103_07245_b200 import pbp_qlp_flops

    table = {(1000, 1000, 40, 0): 1.760e8, (4000, 4000, 100, 0): 6.800e9, (20000, 10000, 256, 1): 4.266e11,
             (200000, 8192, 512, 1): 7.151e12, (65536, 16384, 64, 0): 2.764e11, (65536, 16384, 1024, 2): 1.425e13}
    for key, f in table.items():
        assert abs(pbp_qlp_flops(*key) / f - 1) < 2e-3, key


def test_integration_shim_maps_errors_to_reference_classes(reference_pkg):
    """integration.install rebinds every reference module that imported
    pbp_qlp; invalid arguments then raise the reference's own classes."""
    import sys

    from paper_2103_07245_b200 import integration

    saved = integration.install(reference_pkg)
    try:
        assert {name for _, name in saved} == {"pbp_qlp", "r_svd", "cor_utv", "column_pivoted_qr"}
        for modname, name in saved:
            assert getattr(sys.modules[modname], name).__wrapped_gpu__
        with pytest.raises(reference_pkg.ParameterError):
            reference_pkg.pbp_qlp(np.eye(4), 9)
        with pytest.raises(reference_pkg.ParameterError):
            reference_pkg.r_svd(np.eye(4), 9)
        with pytest.raises(reference_pkg.DimensionError):
            reference_pkg.pbp_qlp(np.eye(4), 2, q=-1)
        with pytest.raises(reference_pkg.MatrixInputError):
            reference_pkg.pbp_qlp(np.ones(3), 1)
    finally:
        integration.uninstall(saved)
    assert not getattr(reference_pkg.pbp_qlp, "__wrapped_gpu__", False)
    assert not getattr(reference_pkg.r_svd, "__wrapped_gpu__", False)


def test_multi_gpu_launcher_validates_before_touching_a_device():
    """pbp_qlp_multi_gpu keeps pbp_qlp's argument contract (algorithms.py:239-241)
    and fails loudly without CUDA (no CPU path)."""
    import numpy as np
    import torch

    from paper_2103_07245_b200 import DeviceError, MatrixInputError, ParameterError, pbp_qlp_multi_gpu
    from paper_2103_07245_b200.multigpu import usable_world

    a = np.ones((30, 20))
    with pytest.raises(ParameterError):
        pbp_qlp_multi_gpu(a, 21)
    bad = a.copy()
    bad[3, 4] = np.inf
    with pytest.raises(MatrixInputError):
        pbp_qlp_multi_gpu(bad, 0)
    with pytest.raises(ParameterError):
        pbp_qlp_multi_gpu(a, 5, backend="mpi")
    if not torch.cuda.is_available():
        with pytest.raises(DeviceError):
            pbp_qlp_multi_gpu(a, 5)
    assert [usable_world(200000, 512, n) for n in (1, 2, 4, 8)] == [1, 2, 4, 8]
    assert usable_world(1000, 512, 8) == 1


def test_multi_gpu_pool_fails_loudly_without_cuda():
    import torch

    from paper_2103_07245_b200 import DeviceError, MultiGpuPool, ParameterError

    with pytest.raises(ParameterError):
        MultiGpuPool([0, 1], backend="mpi")
    if not torch.cuda.is_available():
        with pytest.raises(DeviceError):
            MultiGpuPool([0, 1])
