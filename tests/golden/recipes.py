"""Seeded input recipes for the golden fixtures (numpy, bit-reproducible on any
machine with the same numpy)."""
import numpy as np

CASES = {
    # name: recipe + pbp_qlp arguments
    "tiny_q1": {"recipe": {"kind": "gauss", "shape": [60, 40], "seed": 1}, "d": 10, "q": 1, "seed": 5, "reorth": True},
    "lowrank_q0": {"recipe": {"kind": "lowrank", "shape": [300, 200], "rank": 12, "noise": 1e-4, "seed": 2},
                   "d": 20, "q": 0, "seed": 0, "reorth": True},
    "lowrank_q2": {"recipe": {"kind": "lowrank", "shape": [300, 200], "rank": 12, "noise": 1e-4, "seed": 2},
                   "d": 20, "q": 2, "seed": 3, "reorth": True},
    "noreorth_q1": {"recipe": {"kind": "lowrank", "shape": [200, 150], "rank": 30, "noise": 1e-2, "seed": 4},
                    "d": 16, "q": 1, "seed": 9, "reorth": False},
    "wide": {"recipe": {"kind": "gauss", "shape": [40, 90], "seed": 6}, "d": 7, "q": 1, "seed": 8, "reorth": True},
    "odd_shapes": {"recipe": {"kind": "gauss", "shape": [61, 37], "seed": 7}, "d": 33, "q": 0, "seed": 2**70 + 1,
                   "reorth": True},
    "d_one": {"recipe": {"kind": "gauss", "shape": [50, 30], "seed": 8}, "d": 1, "q": 2, "seed": 4, "reorth": True},
    "rank_deficient": {"recipe": {"kind": "lowrank", "shape": [120, 80], "rank": 3, "noise": 0.0, "seed": 9},
                       "d": 8, "q": 1, "seed": 1, "reorth": True},
    "cfg1": {"recipe": {"kind": "cfg1", "seed": 0}, "d": 40, "q": 0, "seed": 0, "reorth": True},
    # the reference's own rank-test edge case (test_analysis.py:209-215):
    # Hansen's baart(200) at the norm-ratio default d = 20, every orth warns;
    # several |R_ii|/|R_00| sit within 10x of the 1e-14 threshold
    "baart200_q0": {"recipe": {"kind": "stored", "file": "baart200_a.npy", "source": "gen_hansen('baart', 200)"},
                    "d": 20, "q": 0, "seed": 1, "reorth": True},
    "baart200_q2": {"recipe": {"kind": "stored", "file": "baart200_a.npy", "source": "gen_hansen('baart', 200)"},
                    "d": 20, "q": 2, "seed": 1, "reorth": True},
}


def _haar(n, rng):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def make_input(recipe):
    kind = recipe["kind"]
    if kind == "stored":
        # an input produced by a reference generator (make_golden.py), stored
        # as-is because the generator is not part of this package
        import os

        return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), recipe["file"]))
    if kind == "eye":
        return np.eye(recipe["n"])
    if kind == "gauss":
        rng = np.random.Generator(np.random.Philox(key=recipe["seed"]))
        return rng.standard_normal(tuple(recipe["shape"]))
    if kind == "lowrank":
        rng = np.random.Generator(np.random.Philox(key=recipe["seed"]))
        m, n = recipe["shape"]
        k = recipe["rank"]
        a = rng.standard_normal((m, k)) @ rng.standard_normal((k, n)) / np.sqrt(k)
        if recipe["noise"]:
            a = a + recipe["noise"] * rng.standard_normal((m, n))
        return a
    if kind == "cfg1":
        # BASELINE config 1: Haar U, V; σ = 1 (×20), 1e-3 (×980); + 1e-6·N(0,1)
        rng = np.random.Generator(np.random.Philox(key=recipe["seed"]))
        u, v = _haar(1000, rng), _haar(1000, rng)
        sigma = np.concatenate([np.ones(20), np.full(980, 1e-3)])
        return (u * sigma) @ v.T + 1e-6 * rng.standard_normal((1000, 1000))
    if kind == "planted":
        # exactly the given singular values, sign-fixed QR factors of Gaussians
        rng = np.random.Generator(np.random.Philox(key=recipe["seed"]))
        m, n = recipe["shape"]
        vals = np.asarray(recipe["values"], dtype=np.float64)
        u = _thin_q(rng.standard_normal((m, len(vals))))
        v = _thin_q(rng.standard_normal((n, len(vals))))
        return (u * vals) @ v.T
    if kind == "graded":
        # Gaussian columns scaled by logspace(0, -decades, n), columns shuffled
        rng = np.random.Generator(np.random.Philox(key=recipe["seed"]))
        m, n = recipe["shape"]
        g = rng.standard_normal((m, n)) * np.logspace(0, -recipe["decades"], n)
        return g[:, rng.permutation(n)]
    if kind == "int_ties":
        # small-integer entries, every column the same multiset up to sign:
        # the column norms tie exactly (pivot 0 must be column 0)
        rng = np.random.Generator(np.random.Philox(key=recipe["seed"]))
        m, n = recipe["shape"]
        base = rng.integers(-3, 4, size=m).astype(np.float64)
        cols = [rng.permutation(base) * rng.choice([-1.0, 1.0], size=m) for _ in range(n)]
        return np.stack(cols, axis=1)
    raise ValueError(kind)


def _thin_q(g):
    q, r = np.linalg.qr(g)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


# cor_utv cases (algorithms.py:306-363): recipe + arguments
UTV_CASES = {
    "utv_exact": {"recipe": {"kind": "planted", "shape": [50, 40], "values": list(np.linspace(1, 0.1, 10)), "seed": 11},
                  "d": 10, "q": 0, "seed": 2, "pass_efficient": False, "reorth": True},
    "utv_pe_reorth": {"recipe": {"kind": "planted", "shape": [100, 80], "values": list(np.linspace(1, 0.1, 10)),
                                 "seed": 12}, "d": 20, "q": 0, "seed": 3, "pass_efficient": True, "reorth": True},
    "utv_pe_noreorth": {"recipe": {"kind": "planted", "shape": [100, 80], "values": list(np.linspace(1, 0.1, 10)),
                                   "seed": 12}, "d": 20, "q": 0, "seed": 3, "pass_efficient": True, "reorth": False},
    "utv_q2": {"recipe": {"kind": "lowrank", "shape": [300, 200], "rank": 12, "noise": 1e-4, "seed": 2},
               "d": 20, "q": 2, "seed": 3, "pass_efficient": False, "reorth": True},
    "utv_noreorth_q1": {"recipe": {"kind": "lowrank", "shape": [200, 150], "rank": 30, "noise": 1e-2, "seed": 4},
                        "d": 16, "q": 1, "seed": 9, "pass_efficient": False, "reorth": False},
    "utv_truncated": {"recipe": {"kind": "planted", "shape": [30, 20], "values": [1.0, 1e-14, 1e-15], "seed": 13},
                      "d": 6, "q": 0, "seed": 1, "pass_efficient": True, "reorth": False},
    "utv_d_gt_n1": {"recipe": {"kind": "gauss", "shape": [40, 90], "seed": 6}, "d": 60, "q": 1, "seed": 8,
                    "pass_efficient": False, "reorth": True},
    "utv_identity": {"recipe": {"kind": "eye", "n": 4}, "d": 4, "q": 0, "seed": 0, "pass_efficient": False,
                     "reorth": True},
}

# column_pivoted_qr cases (linalg.py:118-129)
CPQR_CASES = {
    "cpqr_gauss_40x15": {"kind": "gauss", "shape": [40, 15], "seed": 2},
    "cpqr_graded_30x10": {"kind": "graded", "shape": [30, 10], "decades": 8, "seed": 4},
    "cpqr_wide_12x30": {"kind": "gauss", "shape": [12, 30], "seed": 5},
    "cpqr_square_96": {"kind": "graded", "shape": [96, 96], "decades": 6, "seed": 7},
    "cpqr_lowrank_64x48": {"kind": "lowrank", "shape": [64, 48], "rank": 20, "noise": 1e-6, "seed": 8},
    "cpqr_ties_9x6": {"kind": "int_ties", "shape": [9, 6], "seed": 3},
    "cpqr_single_col": {"kind": "gauss", "shape": [7, 1], "seed": 1},
    "cpqr_single_row": {"kind": "gauss", "shape": [1, 7], "seed": 1},
}
