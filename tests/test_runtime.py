"""The runtime harness (cli.py:373-443) restated for the GPU
paths: table format, argument parsing and matrix families against the
reference (CPU), and one small end-to-end run (GPU)."""
import numpy as np
import pytest

from paper_2103_07245_b200 import runtime as R


def test_d_spec_and_lists():
    assert R.parse_d_spec("frac:0.05, 0.2") == ("frac", [0.05, 0.2])
    assert R.parse_d_spec("20,30") == ("abs", [20, 30])
    assert R.resolve_d_list(("frac", [0.05, 0.2, 1.0]), 300) == [15, 60, 300]
    from paper_2103_07245_b200 import ParameterError

    for bad in ("frac:", "frac:0", "frac:1.5", "frac:x", "a,b"):
        with pytest.raises(ParameterError):
            R.parse_d_spec(bad)
    with pytest.raises(ParameterError):
        R.resolve_d_list(("abs", [400]), 300)


def test_table_format(tmp_path):
    rows = [("runtime", "pbp_qlp", 100, 100, 20, 0, 0, 3, 1234.5, 1300.25)]
    p = R.write_table(tmp_path / "t.dsv", "runtime", [("matrix", "lowrank"), ("n", "100")], R.HEADER, rows)
    lines = p.read_text().splitlines()
    assert lines[0].startswith("# paper_2103_07245_b200 ") and lines[0].endswith("runtime matrix=lowrank n=100")
    assert lines[1].split("\t") == list(R.HEADER)
    assert lines[2] == "runtime\tpbp_qlp\t100\t100\t20\t0\t0\t3\t1234.5\t1300.25"


def test_table_cells_match_reference(reference_pkg, tmp_path):
    """Same header and cell formatting as the reference's _write_table."""
    from pbpqlp import cli

    rows = [("runtime", "r_svd", 7, 9, 3, 1, 2, 5, float(np.float64(1.0) / 3), 2.5e9)]
    cfg = [("matrix", "fast"), ("n", "7")]
    mine = R.write_table(tmp_path / "a.dsv", "runtime", cfg, R.HEADER, rows).read_text().splitlines()
    ref = cli._write_table(tmp_path / "b.dsv", "runtime", cfg,
                           ("experiment", "alg", "n1", "n2", "d", "q", "seed", "trials", "median_ns", "mean_ns"),
                           rows).read_text().splitlines()
    assert mine[1:] == ref[1:]
    assert mine[0].split(" ", 3)[3] == ref[0].split(" ", 3)[3]  # the config echo


@pytest.mark.parametrize("spec,n", [("lowrank", 60), ("lowrank:k=5,mu=0.01", 40), ("stairs:step_len=4,step_ratio=0.3", 30),
                                    ("fast", 25), ("slow", 20), ("lowrank:mu=0", 50)])
def test_matrix_families_match_reference(reference_pkg, spec, n):
    from pbpqlp.matgen import SpectrumSpec

    a = R.build_matrix(spec, n, 7)
    ref = SpectrumSpec.parse(spec, n=n, seed=7).build()
    np.testing.assert_array_equal(a, ref)


def test_cli_errors_and_exit_codes(tmp_path):
    assert R.main(["--n", "100", "--format", "csv", "--out", str(tmp_path / "x")]) == R.EXIT_USAGE
    assert R.main(["--n", "100", "--alg", "svd", "--out", str(tmp_path / "x")]) == R.EXIT_USAGE
    assert R.main(["--n", "3000", "--out", str(tmp_path / "x")]) == R.EXIT_RESOURCE
    assert R.main(["--n", "100", "--matrix", "hansen:baart", "--out", str(tmp_path / "x")]) == R.EXIT_USAGE
    assert R.main(["--n", "100", "--matrix", "lowrank:zz=1", "--out", str(tmp_path / "x")]) == R.EXIT_USAGE


@pytest.mark.gpu
def test_runtime_end_to_end(cuda, tmp_path):
    out = tmp_path / "rt.dsv"
    assert R.main(["--n", "300,500", "--d", "frac:0.1", "--q", "0,1", "--trials", "2", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0].startswith("# paper_2103_07245_b200") and "device=" in lines[0]
    assert lines[1].split("\t") == list(R.HEADER)
    rows = [l.split("\t") for l in lines[2:]]
    assert len(rows) == 2 * 2 * 3  # n × q × alg
    for r in rows:
        assert r[0] == "runtime" and r[1] in R.RANDOMIZED_ALGORITHMS and int(r[7]) == 2
        assert int(r[4]) == round(0.1 * int(r[2]))
        assert float(r[8]) > 0 and float(r[9]) > 0
