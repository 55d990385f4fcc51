#!/usr/bin/env python3
"""Golden fixtures for the sibling path cor_utv (algorithms.py:306-363) and
its core, column_pivoted_qr (linalg.py:118-129), produced by running the
REFERENCE package (importable only in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_utv.py
"""
import hashlib
import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import pbpqlp  # noqa: E402  (the reference)

from tests.golden.recipes import CPQR_CASES, UTV_CASES, make_input  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    utv = {}
    for name, case in UTV_CASES.items():
        a = make_input(case["recipe"])
        with warnings.catch_warnings(record=True) as rec:
            warnings.simplefilter("always")
            f = pbpqlp.cor_utv(a, case["d"], q=case["q"], seed=case["seed"], pass_efficient=case["pass_efficient"],
                               reorthonormalize=case["reorth"])
        n_warn = sum(1 for w in rec if issubclass(w.category, pbpqlp.RankDeficiencyWarning))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), u=f.u, t=f.t, v=f.v)
        utv[name] = {**{k: v for k, v in case.items() if k != "recipe"}, "recipe": case["recipe"],
                     "a_sha256": sha(a), "passes_over_a": f.sketch.passes_over_a,
                     "pinv_truncated": bool(f.pinv_truncated), "rank_warnings": n_warn}
        print(name, a.shape, "passes", f.sketch.passes_over_a, "trunc", f.pinv_truncated, "warnings", n_warn)
    cpqr = {}
    for name, recipe in CPQR_CASES.items():
        m = make_input(recipe)
        f = pbpqlp.column_pivoted_qr(m)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), q=f.q, r=f.r, perm=f.perm)
        cpqr[name] = {"recipe": recipe, "m_sha256": sha(m), "perm": [int(x) for x in f.perm]}
        print(name, m.shape, list(f.perm)[:8])
    with open(os.path.join(HERE, "manifest_utv.json"), "w") as fh:
        json.dump({"utv": utv, "cpqr": cpqr, "generator": "pbpqlp " + pbpqlp.__version__ + ", numpy " + np.__version__},
                  fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
