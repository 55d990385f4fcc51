#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package (/root/reference/pkg/src/pbpqlp, importable only in the build
container) on small seeded inputs.

Each case stores the input recipe (regenerated bit-for-bit by the tests with
numpy), a checksum of the input matrix, and the reference's outputs
(Q, L, P, R, Φ, passes, per-orth warnings).  The GPU tests compare against
these fixtures on the box, where the reference itself is absent.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
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

from tests.golden.recipes import CASES, make_input  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    manifest = {}
    for name, case in CASES.items():
        rec_ = case["recipe"]
        if rec_["kind"] == "stored":  # inputs from a reference generator, e.g. gen_hansen('baart', 200)
            import ast

            fn, args = rec_["source"].split("(", 1)
            gen_args = ast.literal_eval("(" + args.rstrip()[:-1] + ",)")
            np.save(os.path.join(HERE, rec_["file"]), getattr(pbpqlp, fn)(*gen_args))
        a = make_input(rec_)
        with warnings.catch_warnings(record=True) as rec:
            warnings.simplefilter("always")
            f = pbpqlp.pbp_qlp(a, case["d"], q=case["q"], seed=case["seed"], reorthonormalize=case["reorth"])
        n_warn = sum(1 for w in rec if issubclass(w.category, pbpqlp.RankDeficiencyWarning))
        # rank-test margins of the reference's own orth calls (the oracle is
        # bitwise the reference here): smallest |R_ii|/|R_00| per call
        from oracle.pbp_qlp_oracle import oracle_pbp_qlp

        o = oracle_pbp_qlp(a, case["d"], q=case["q"], seed=case["seed"], reorthonormalize=case["reorth"])
        assert np.array_equal(o["q"], f.q_basis), "oracle is not the reference"
        min_ratio = [float(dg.min() / dg[0]) if dg[0] > 0 else 0.0 for dg in o["orth_r_diag"]]
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            q=f.q_basis, l=f.l, p=f.p_basis, r=f.first_stage_r, phi=f.sketch.test_matrix,
        )
        manifest[name] = {
            **{k: v for k, v in case.items() if k != "recipe"},
            "recipe": case["recipe"],
            "a_sha256": sha(a),
            "passes_over_a": f.sketch.passes_over_a,
            "rank_warnings": n_warn,
            "rank_flags": [int(x) for x in o["rank_flags"]],
            "orth_min_ratio": min_ratio,
        }
        print(name, a.shape, "warnings", n_warn)
    # sketch-only fixtures: gaussian_matrix(rows, cols, seed)
    sketches = {}
    for rows, cols, seed in [(7, 13, 2**100 + 7), (64, 40, 0), (33, 5, 123456789)]:
        g = pbpqlp.gaussian_matrix(rows, cols, seed)
        key = f"gauss_{rows}x{cols}_{seed}"
        np.save(os.path.join(HERE, key + ".npy"), g)
        sketches[key] = {"rows": rows, "cols": cols, "seed": seed, "sha256": sha(g)}
    # error contract: the exception class the reference raises for bad arguments
    errors = {}
    for label, args in ERROR_CASES.items():
        try:
            pbpqlp.pbp_qlp(*args[0], **args[1])
            errors[label] = None
        except Exception as exc:  # noqa: BLE001
            errors[label] = type(exc).__name__
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump({"cases": manifest, "sketches": sketches, "errors": errors,
                   "generator": "pbpqlp " + pbpqlp.__version__ + ", numpy " + np.__version__}, fh, indent=1,
                  sort_keys=True)


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
    "a_nan": ((_nan, 2), {}),
    "a_nan_and_bad_d": ((_nan, 9), {}),
    "a_inf": ((np.full((4, 4), np.inf), 2), {}),
}


if __name__ == "__main__":
    main()
