"""The reference harness's ``runtime`` experiment on the GPU paths (SURVEY.md
§8 f4): the same protocol and DSV table, so GPU rows sit beside the CPU rows
the reference writes.

Restates /root/reference/pkg/src/pbpqlp/cli.py:

* ``_cmd_runtime`` (:373-443): for each n, d, q, alg — build the matrix once,
  one discarded warm-up ``factorize``, then ``trials`` timed calls with seeds
  ``seed+1+t`` (``time.perf_counter_ns``); rows carry the median and mean ns;
* the DSV writer ``_write_table`` / ``_cell`` (:301-320): a ``# <tool>
  <version> runtime key=value ...`` echo line, a tab-separated header, then
  one tab-separated row per point (ints as ints, floats by ``repr``);
* ``--d`` as absolute sizes or ``frac:<list>`` (:142-171), the memory cap
  check (:276-283, 24 bytes per entry, default order 2500), exit codes
  (:69-73: 2 usage, 3 input, 4 resource).

The timed call is the public function a user makes (numpy in, numpy out), so
each trial includes the host→device copy of A and the device→host copy of
the factors, like the e2e number of bench.py.  Matrices come from the
reference's synthetic families (matgen.py): ``lowrank``, ``stairs``,
``fast`` and ``slow``, drawn from the same seeded Philox stream with the
same sign-fixed QR factors, so the inputs equal the reference's (for
``lowrank`` with n > 2000 the noise normalisation uses this package's
spectral norm, equal to rounding).  ``hansen`` and ``image`` are outside
this package.

    python -m paper_2103_07245_b200.runtime --n 1000,2000 --d frac:0.05,0.1 --alg pbp_qlp,r_svd,cor_utv
"""
import argparse
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

from . import __version__
from . import exceptions as _exc
from .validation import check_count, check_index_range

EXIT_OK, EXIT_USAGE, EXIT_INPUT, EXIT_RESOURCE = 0, 2, 3, 4  # cli.py:69-73
MEMORY_FACTOR = 3 * 8  # cli.py:81
DEFAULT_MEM_CAP = MEMORY_FACTOR * 2500 * 2500  # cli.py:84
OUT_DIR_ENV = "PBPQLP_OUT_DIR"  # cli.py:76
RANDOMIZED_ALGORITHMS = ("r_svd", "cor_utv", "pbp_qlp")  # analysis.py:54
HEADER = ("experiment", "alg", "n1", "n2", "d", "q", "seed", "trials", "median_ns", "mean_ns")  # cli.py:429-440
TOOL = "paper_2103_07245_b200"


class ResourceLimitError(RuntimeError):
    """Workload above the memory cap (exceptions.py:46, a RuntimeError)."""


# ------------------------------------------------------------- matrices --
_RAMP_FLOOR = 1e-25  # matgen.py:38


def _rng(seed):
    return np.random.Generator(np.random.Philox(key=int(seed)))


def _orth_host(g):
    """The reference's orth (householder_qr + _fix_signs, linalg.py:96-165)
    for input synthesis on the host."""
    q, r = np.linalg.qr(g)
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def _planted(reference, rng):
    """matgen.py:45-53."""
    n = reference.shape[0]
    r = max(int(np.count_nonzero(reference)), 1)
    u = _orth_host(rng.standard_normal((n, r)))
    v = _orth_host(rng.standard_normal((n, r)))
    return (u * reference[:r]) @ v.T


def _spectral_norm_host(m):
    if max(m.shape) <= 2000:  # linalg.py:194-207, dense branch
        return float(np.linalg.svd(m, compute_uv=False)[0])
    from .analysis import spectral_norm

    return spectral_norm(m)


def _parse_params(text, family):
    params = {}
    for item in text.split(","):
        item = item.strip()
        if not item:
            continue
        if "=" not in item:
            raise _exc.ParameterError(f"{family}: expected key=value, got {item!r}")
        key, value = item.split("=", 1)
        params[key.strip()] = value.strip()
    extra = set(params) - {"k", "mu", "step_len", "step_ratio"}
    if extra:
        raise _exc.ParameterError(f"{family}: unknown parameters {sorted(extra)}")
    return params


def build_matrix(spec, n, seed):
    """``SpectrumSpec.parse(spec, n, seed).build()`` (matgen.py:181-238) for
    the synthetic families."""
    family, _, rest = str(spec).strip().partition(":")
    family = family.lower()
    if family in ("hansen", "image"):
        raise _exc.ParameterError(f"matrix family {family!r} is outside this package (synthetic families only)")
    if family not in ("lowrank", "stairs", "fast", "slow"):
        raise _exc.ParameterError(f"unknown matrix family {family!r}; choose from lowrank, stairs, fast, slow")
    p = _parse_params(rest, family)
    rng = _rng(seed)
    if family == "lowrank":  # matgen.py:56-85
        n = check_count(n, "n", minimum=2)
        k = check_count(int(p.get("k", 20)), "k", minimum=1, maximum=n - 1)
        mu = float(p.get("mu", 0.005))
        if not (mu >= 0.0 and np.isfinite(mu)):
            raise _exc.ParameterError(f"mu must be >= 0, got {mu}")
        reference = np.zeros(n)
        reference[:k] = 1.0 - np.arange(k) * (1.0 - _RAMP_FLOOR) / (n - 1)
        a = _planted(reference, rng)
        if mu > 0.0:
            noise = rng.standard_normal((n, n))
            a = a + (mu * reference[k - 1] / _spectral_norm_host(noise)) * noise
        return a
    n = check_count(n, "n", minimum=1)
    if family == "stairs":  # matgen.py:88-100
        step_len = check_count(int(p.get("step_len", 15)), "step_len", minimum=1)
        ratio = float(p.get("step_ratio", 0.5))
        if not 0.0 < ratio < 1.0:
            raise _exc.ParameterError(f"step_ratio must lie in (0, 1), got {ratio}")
        return _planted(ratio ** (np.arange(n) // step_len).astype(float), rng)
    i = np.arange(1, n + 1, dtype=float)  # matgen.py:103-119
    return _planted(np.exp(-i / 6.0) if family == "fast" else i**-2.0, rng)


# --------------------------------------------------------------- tables --
def parse_d_spec(text):
    """``--d``: absolute sizes ``20,30`` or ``frac:0.04,0.2`` (cli.py:142-163)."""
    text = str(text).strip()
    if text.lower().startswith("frac:"):
        fractions = []
        for piece in text[len("frac:"):].split(","):
            piece = piece.strip()
            if not piece:
                continue
            try:
                value = float(piece)
            except ValueError:
                raise _exc.ParameterError(f"d: expected comma-separated fractions after 'frac:', got {text!r}") from None
            if not 0.0 < value <= 1.0:
                raise _exc.ParameterError(f"d: fractions must lie in (0, 1], got {value}")
            fractions.append(value)
        if not fractions:
            raise _exc.ParameterError(f"d: expected at least one fraction, got {text!r}")
        return ("frac", fractions)
    return ("abs", int_list(text, "d"))


def resolve_d_list(d_spec, limit):
    """cli.py:166-171."""
    kind, values = d_spec
    if kind == "abs":
        return [check_index_range(v, "d", 1, limit) for v in values]
    return [min(limit, max(1, int(round(f * limit)))) for f in values]


def int_list(text, name):
    out = []
    for piece in str(text).split(","):
        piece = piece.strip()
        if not piece:
            continue
        try:
            out.append(int(piece))
        except ValueError:
            raise _exc.ParameterError(f"{name}: expected comma-separated integers, got {text!r}") from None
    if not out:
        raise _exc.ParameterError(f"{name}: expected at least one value, got {text!r}")
    return out


def cell(value):
    """cli.py:301-308."""
    if isinstance(value, bool):
        return str(int(value))
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    if isinstance(value, (float, np.floating)):
        return repr(float(value))
    return str(value)


def write_table(path, command, config_pairs, header, rows):
    """cli.py:311-320 (the echo line names this package and the device)."""
    config_echo = " ".join(f"{key}={value}" for key, value in config_pairs)
    lines = [f"# {TOOL} {__version__} {command} {config_echo}".rstrip(), "\t".join(header)]
    for row in rows:
        if len(row) != len(header):
            raise AssertionError("row width disagrees with header")
        lines.append("\t".join(cell(v) for v in row))
    path = Path(path)
    path.write_text("\n".join(lines) + "\n", encoding="utf-8")
    return path


def check_workload(n1, n2, cap):
    """cli.py:276-283."""
    required = MEMORY_FACTOR * int(n1) * int(n2)
    if required > cap:
        raise ResourceLimitError(
            f"refusing a {n1} x {n2} dense workload: it needs about {required} bytes "
            f"({MEMORY_FACTOR} bytes per entry including working copies), which exceeds "
            f"the memory cap of {cap} bytes; raise --mem-cap to proceed"
        )


def output_path(out, command):
    """cli.py:290-298."""
    path = Path(out) if out else Path(os.environ.get(OUT_DIR_ENV, ".")) / f"{command.replace('-', '_')}.dsv"
    if path.parent != Path(""):
        path.parent.mkdir(parents=True, exist_ok=True)
    return path


# ------------------------------------------------------------ experiment --
def runtime(n_list, d_spec=("frac", [0.2]), q_list=(0,), algs=RANDOMIZED_ALGORITHMS, matrix="lowrank", seed=0,
            trials=5, mem_cap=DEFAULT_MEM_CAP, reorth=True):
    """Rows of the runtime table (cli.py:373-420) timed on the GPU paths."""
    from .analysis import factorize

    for alg in algs:
        if alg not in RANDOMIZED_ALGORITHMS:
            raise _exc.ParameterError(f"runtime: algorithm {alg!r} not in {RANDOMIZED_ALGORITHMS}")
    trials = check_count(trials, "trials", minimum=1)
    rows = []
    for n in n_list:
        check_count(n, "n", minimum=2)
        check_workload(n, n, mem_cap)
        a = build_matrix(matrix, n, seed)
        for d in resolve_d_list(d_spec, min(a.shape)):
            for q in q_list:
                for alg in algs:
                    factorize(a, alg, d, q=q, seed=seed, reorthonormalize=reorth)  # warm-up (discarded)
                    samples = []
                    for t in range(trials):
                        start = time.perf_counter_ns()
                        factorize(a, alg, d, q=q, seed=seed + 1 + t, reorthonormalize=reorth)
                        samples.append(time.perf_counter_ns() - start)
                    rows.append(("runtime", alg, a.shape[0], a.shape[1], d, q, seed, trials,
                                 float(statistics.median(samples)), float(statistics.fmean(samples))))
    return rows


def _echo_d(d_spec):
    kind, values = d_spec
    text = ",".join(str(v) for v in values)
    return "frac:" + text if kind == "frac" else text


def _build_parser():
    ap = argparse.ArgumentParser(prog="python -m paper_2103_07245_b200.runtime",
                                 description="The reference harness's runtime experiment on the B200 paths.")
    ap.add_argument("--matrix", default="lowrank", help="matrix spec, family[:params]")
    ap.add_argument("--n", required=True, help="matrix orders, comma list")
    ap.add_argument("--d", default="frac:0.2", help="sampling sizes: comma list or frac:<list>")
    ap.add_argument("--q", default="0", help="power-iteration exponents, comma list")
    ap.add_argument("--alg", default=",".join(RANDOMIZED_ALGORITHMS), help="algorithm ids, comma list")
    ap.add_argument("--seed", default="0")
    ap.add_argument("--trials", default="5")
    ap.add_argument("--out", default=None, help="output table path")
    ap.add_argument("--format", default="dsv", help="output format (dsv)")
    ap.add_argument("--mem-cap", dest="mem_cap", default=str(DEFAULT_MEM_CAP), help="memory cap in bytes")
    ap.add_argument("--no-reorth", dest="no_reorth", action="store_true")
    return ap


def main(argv=None):
    try:
        args = _build_parser().parse_args(argv)
        if str(args.format).strip().lower() != "dsv":
            raise _exc.ParameterError(f"format: only 'dsv' is supported, got {args.format!r}")
        n_list = int_list(args.n, "n")
        d_spec = parse_d_spec(args.d)
        q_list = int_list(args.q, "q")
        algs = [a.strip() for a in args.alg.split(",") if a.strip()]
        seed = int_list(args.seed, "seed")[0]
        trials = int_list(args.trials, "trials")[0]
        cap = int_list(args.mem_cap, "mem_cap")[0]
        reorth = not args.no_reorth
        rows = runtime(n_list, d_spec, q_list, algs, args.matrix, seed, trials, cap, reorth)
        path = output_path(args.out, "runtime")
        import torch

        config = [("matrix", args.matrix), ("n", ",".join(map(str, n_list))), ("d", _echo_d(d_spec)),
                  ("q", ",".join(map(str, q_list))), ("alg", ",".join(algs)), ("seed", seed), ("trials", trials),
                  ("reorth", int(reorth)), ("device", torch.cuda.get_device_name(0).replace(" ", "_"))]
        write_table(path, "runtime", config, HEADER, rows)
        print(f"wrote {path} ({len(rows)} rows)")
        return EXIT_OK
    except ResourceLimitError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RESOURCE
    except (_exc.MatrixInputError, _exc.ConvergenceError, _exc.DeviceError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INPUT
    except _exc.ParameterError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INPUT


if __name__ == "__main__":
    sys.exit(main())
