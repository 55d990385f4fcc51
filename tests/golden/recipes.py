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
}


def _haar(n, rng):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def make_input(recipe):
    kind = recipe["kind"]
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
    raise ValueError(kind)
