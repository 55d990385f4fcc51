"""pytest plugin (``-p tests.reference_suite_plugin``) that routes the
REFERENCE's own test suite through the GPU drop-in.

At ``pytest_configure`` — before any reference test module is imported and
binds ``from pbpqlp import pbp_qlp`` — it calls
``integration.install(pbpqlp)``, which rebinds pbp_qlp, r_svd, cor_utv and
column_pivoted_qr in every reference module that imported them
(INTEGRATION.md).  Each rebound entry point is wrapped once more to count its
calls; the count is printed at the end of the session so that the caller
(tests/test_gpu_reference_suite.py) can prove the GPU path ran.
"""
import functools

CALLS = {}


def _counted(name, fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*args, **kwargs)

    wrapper.__wrapped_gpu__ = True
    return wrapper


def pytest_configure(config):
    import importlib

    import pbpqlp

    from paper_2103_07245_b200 import _lib, integration

    _lib.load()  # the CUDA library must be there: no silent CPU run
    integration.install(pbpqlp)
    for suffix in integration._BINDERS:
        mod = importlib.import_module(pbpqlp.__name__ + suffix) if suffix else pbpqlp
        for name in ("pbp_qlp", "r_svd", "cor_utv", "column_pivoted_qr"):
            fn = getattr(mod, name, None)
            if fn is not None and getattr(fn, "__wrapped_gpu__", False):
                setattr(mod, name, _counted(name, fn))


def pytest_sessionfinish(session, exitstatus):
    import torch

    from paper_2103_07245_b200 import device as D

    launches = D.context(torch.device("cuda", 0)).launch_count if torch.cuda.is_available() else 0
    calls = ",".join(f"{k}={v}" for k, v in sorted(CALLS.items()))
    print(f"\nGPU-DROPIN calls: {calls or 'none'}; libpbq launches: {launches}")
