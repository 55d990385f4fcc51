"""Drop-in wiring for the reference package.

``install(pbpqlp)`` rebinds the reference's PbP-QLP entry point (and the
siblings ``r_svd``, algorithms.py:263-292, ``cor_utv``, :306-363, and its
core ``column_pivoted_qr``, linalg.py:118-129) — in every
module that imported it by name (algorithms.py:209, __init__.py:18,
analysis.py:16-25 → factorize :153-154, estimators.py:17 → PbpQlp
:98-105, bounds.py:42 → eval_highprob_bounds :589, cli.py:43 → :448, :733)
— to a wrapper around :func:`paper_2103_07245_b200.pbp_qlp` that

* returns the reference's own ``QlpFactors`` / ``SketchRecord`` dataclasses
  holding numpy arrays (so every downstream consumer keeps working),
* raises the reference's exception classes (ParameterError, DimensionError,
  MatrixInputError), and
* re-emits rank-deficiency warnings as the reference's RankDeficiencyWarning.

The GPU does every FLOP; this module only adapts types.
"""
import warnings

from . import algorithms as _alg
from . import exceptions as _exc

# modules of the reference that bind the patched names at import time
_BINDERS = ("", ".linalg", ".algorithms", ".analysis", ".estimators", ".bounds", ".cli")


def _translated(pbpqlp, fn):
    """Run ``fn`` mapping this package's exceptions / warnings to the reference's."""
    ref_exc = pbpqlp.exceptions
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always", _exc.RankDeficiencyWarning)
        try:
            out = fn()
        except _exc.DimensionError as e:
            raise ref_exc.DimensionError(str(e)) from None
        except _exc.ParameterError as e:
            raise ref_exc.ParameterError(str(e)) from None
        except _exc.MatrixInputError as e:
            raise ref_exc.MatrixInputError(str(e)) from None
    for w in rec:
        if issubclass(w.category, _exc.RankDeficiencyWarning):
            warnings.warn(str(w.message), ref_exc.RankDeficiencyWarning, stacklevel=3)
        else:
            warnings.warn_explicit(w.message, w.category, w.filename, w.lineno)
    return out


def make_rsvd_dropin(pbpqlp):
    """Reference-typed ``r_svd(a, d, q=0, seed=0, reorthonormalize=True)``
    (algorithms.py:263-292) running on the GPU path."""
    from . import rsvd as _rsvd

    ref_alg = pbpqlp.algorithms

    def r_svd(a, d, q=0, seed=0, reorthonormalize=True):
        f = _translated(pbpqlp, lambda: _rsvd.r_svd(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize))
        sk = f.sketch
        sketch = ref_alg.SketchRecord(sk.test_matrix, int(seed), sk.d, sk.q, sk.passes_over_a)
        return ref_alg.RsvdFactors(f.u, f.s, f.v, sketch)

    r_svd.__doc__ = ref_alg.r_svd.__doc__
    r_svd.__wrapped_gpu__ = True
    return r_svd


def make_utv_dropin(pbpqlp):
    """Reference-typed ``cor_utv(a, d, q=0, seed=0, pass_efficient=False,
    reorthonormalize=True)`` (algorithms.py:306-363) on the GPU path."""
    from . import utv as _utv

    ref_alg = pbpqlp.algorithms

    def cor_utv(a, d, q=0, seed=0, pass_efficient=False, reorthonormalize=True):
        f = _translated(pbpqlp, lambda: _utv.cor_utv(a, d, q=q, seed=seed, pass_efficient=pass_efficient,
                                                     reorthonormalize=reorthonormalize))
        sk = f.sketch
        sketch = ref_alg.SketchRecord(sk.test_matrix, int(seed), sk.d, sk.q, sk.passes_over_a)
        return ref_alg.UtvFactors(f.u, f.t, f.v, f.pass_efficient, sketch, f.pinv_truncated)

    cor_utv.__doc__ = ref_alg.cor_utv.__doc__
    cor_utv.__wrapped_gpu__ = True
    return cor_utv


def make_cpqr_dropin(pbpqlp):
    """Reference-typed ``column_pivoted_qr(m)`` (linalg.py:118-129) on the GPU."""
    from . import linalg as _linalg

    ref_lin = pbpqlp.linalg

    def column_pivoted_qr(m):
        f = _translated(pbpqlp, lambda: _linalg.column_pivoted_qr(m))
        return ref_lin.QrFactors(f.q, f.r, f.perm)

    column_pivoted_qr.__doc__ = ref_lin.column_pivoted_qr.__doc__
    column_pivoted_qr.__wrapped_gpu__ = True
    return column_pivoted_qr


def make_dropin(pbpqlp, devices=None, backend="nccl"):
    """Return a reference-typed ``pbp_qlp(a, d, q=0, seed=0, reorthonormalize=True)``.
    ``devices`` (a list of CUDA indices, more than one): the calls are row-sharded
    over those GPUs by a ``MultiGpuPool`` (one worker process per GPU, started by
    the first call, stopped by ``uninstall`` or at exit)."""
    ref_alg = pbpqlp.algorithms
    ref_exc = pbpqlp.exceptions
    multi = devices is not None and len(devices) > 1
    holder = {"pool": None}  # the worker pool, started by the first call and kept until uninstall / exit

    def _pool():
        import atexit

        from .multigpu import MultiGpuPool

        pool = holder["pool"]
        if pool is None or pool.broken:
            pool = holder["pool"] = MultiGpuPool(devices, backend)
            atexit.register(pool.close)
        return pool

    def pbp_qlp(a, d, q=0, seed=0, reorthonormalize=True):
        with warnings.catch_warnings(record=True) as rec:
            warnings.simplefilter("always", _exc.RankDeficiencyWarning)
            try:
                if multi:
                    f = _pool().pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize)
                else:
                    f = _alg.pbp_qlp(a, d, q=q, seed=seed, reorthonormalize=reorthonormalize)
            except _exc.DimensionError as e:
                raise ref_exc.DimensionError(str(e)) from None
            except _exc.ParameterError as e:
                raise ref_exc.ParameterError(str(e)) from None
            except _exc.MatrixInputError as e:
                raise ref_exc.MatrixInputError(str(e)) from None
        for w in rec:
            if issubclass(w.category, _exc.RankDeficiencyWarning):
                warnings.warn(str(w.message), ref_exc.RankDeficiencyWarning, stacklevel=2)
            else:
                warnings.warn_explicit(w.message, w.category, w.filename, w.lineno)
        sk = f.sketch
        sketch = ref_alg.SketchRecord(sk.test_matrix, int(seed), sk.d, sk.q, sk.passes_over_a)
        return ref_alg.QlpFactors(f.q_basis, f.l, f.p_basis, f.first_stage_r, sketch)

    pbp_qlp.__doc__ = ref_alg.pbp_qlp.__doc__
    pbp_qlp.__wrapped_gpu__ = True
    pbp_qlp.__pool_holder__ = holder
    return pbp_qlp


def install(pbpqlp, devices=None, backend="nccl"):
    """Patch every module of the imported reference package ``pbpqlp`` that
    bound ``pbp_qlp``; returns the previous bindings (for ``uninstall``).
    ``devices=[0, 1, …]`` routes ``pbp_qlp`` through the multi-GPU launcher."""
    import importlib

    dropins = {"pbp_qlp": make_dropin(pbpqlp, devices, backend), "r_svd": make_rsvd_dropin(pbpqlp),
               "cor_utv": make_utv_dropin(pbpqlp), "column_pivoted_qr": make_cpqr_dropin(pbpqlp)}
    saved = {}
    for suffix in _BINDERS:
        mod = importlib.import_module(pbpqlp.__name__ + suffix) if suffix else pbpqlp
        for name, fn in dropins.items():
            if hasattr(mod, name):
                saved[(mod.__name__, name)] = getattr(mod, name)
                setattr(mod, name, fn)
    return saved


def uninstall(saved):
    import sys

    for (modname, name), fn in saved.items():
        current = getattr(sys.modules[modname], name, None)
        holder = getattr(current, "__pool_holder__", None)
        if holder and holder.get("pool") is not None:  # stop the multi-GPU workers of the drop-in
            holder["pool"].close()
            holder["pool"] = None
        setattr(sys.modules[modname], name, fn)
