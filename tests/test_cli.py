"""bench_cli: sgm10 unit values, generator files, exit codes
and bench tables. The solve/bench tests run the GPU solver."""
import csv
import io
import json
import os

import numpy as np
import pytest

import paper_2311_07710_b200 as rb
from paper_2311_07710_b200 import cli


def test_sgm10_unit_values():  # SPEC AC8
    assert cli.sgm10([0, 0]) == pytest.approx(0.0, abs=1e-12)
    assert cli.sgm10([90, 90]) == pytest.approx(90.0, abs=1e-12)
    assert cli.sgm10([0, 990]) == pytest.approx(90.0, abs=1e-12)
    with pytest.raises(ValueError):
        cli.sgm10([])


def test_sgm10_properties():
    v = [3.0, 17.0, 250.0, 1e5]
    assert cli.sgm10(v) == pytest.approx(cli.sgm10(v[::-1]))  # permutation-invariant
    assert cli.sgm10([3.0, 18.0, 250.0, 1e5]) > cli.sgm10(v)   # monotone
    assert cli.sgm10([5e5, 10.0], limit=cli.ITER_LIMIT) == pytest.approx(cli.sgm10([2e5, 10.0]))


def test_generate_files_deterministic(tmp_path):
    a, b = tmp_path / "a.qps", tmp_path / "b.qps"
    assert cli.main(["generate", "random_qp", "0.2", "7", str(a)]) == 0
    assert cli.main(["generate", "random_qp", "0.2", "7", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()  # same seed -> byte-identical
    meta = json.loads((tmp_path / "a.json").read_text())
    p = rb.read_qps(str(a))
    assert meta["n"] == p.num_vars() and meta["m_ineq"] + meta["m_eq"] == p.num_rows()
    assert cli.main(["generate", "no_such_class", "1", "1", str(tmp_path / "c.qps")]) == 3


def test_solve_missing_file_exit_3(tmp_path, capsys):
    assert cli.main(["solve", str(tmp_path / "missing.qps")]) == 3
    assert "missing.qps" in capsys.readouterr().err


def test_bench_empty_dir_is_an_error(tmp_path):
    assert cli.main(["bench", str(tmp_path)]) == 3


def test_restart_flag_parsing():
    assert cli._restart("fixed=64") == (rb.RestartPolicy.kFixed, 64)
    assert cli._restart("halving")[0] == rb.RestartPolicy.kAdaptiveHalving
    with pytest.raises(Exception):
        cli._restart("sometimes")


def one_d_qps(path):
    # SPEC AC1: min x^2 - 2x  s.t.  x <= 0.5   (Q = 2, c = -2, A = 1, b = 0.5)
    p = rb.QuadraticProgram(q=rb.SparseMatrix(1, 1, [(0, 0, 2.0)]), c=np.array([-2.0]),
                            a_ineq=rb.SparseMatrix(1, 1, [(0, 0, 1.0)]), b_ineq=np.array([0.5]),
                            a_eq=rb.SparseMatrix(0, 1), b_eq=np.zeros(0), name="ONE_D")
    path.write_text(rb.write_qps(p))


@pytest.mark.gpu
def test_cli_solve_one_d(tmp_path):
    f = tmp_path / "one_d.qps"
    one_d_qps(f)
    out, log = tmp_path / "sol.json", tmp_path / "log.csv"
    assert cli.main(["solve", str(f), "--tol", "1e-9", "--out", str(out), "--log", str(log)]) == 0
    sol = json.loads(out.read_text())
    assert sol["status"] == "optimal" and sol["objective"] == pytest.approx(-0.75, abs=1e-6)
    assert sol["x"][0] == pytest.approx(0.5, abs=1e-6)
    rows = list(csv.reader(io.StringIO(log.read_text())))
    assert rows[0] == ["iter", "r_primal", "r_dual", "r_gap", "eta", "omega", "restarted"] and len(rows) > 1
    assert cli.main(["solve", str(f), "--max-iters", "0"]) == 2


@pytest.mark.gpu
def test_cli_bench_table(tmp_path):
    one_d_qps(tmp_path / "a_one_d.qps")
    assert cli.main(["generate", "random_qp", "0.1", "3", str(tmp_path / "b_rand.qps")]) == 0
    (tmp_path / "c_broken.qps").write_text("NAME broken\nROWS\n N obj\nCOLUMNS\n x obj notanumber\nENDATA\n")
    t1, t2 = tmp_path / "t1.csv", tmp_path / "t2.csv"
    assert cli.main(["bench", str(tmp_path), "--tol", "1e-6", "--out", str(t1)]) == 0
    assert cli.main(["bench", str(tmp_path), "--tol", "1e-6", "--out", str(t2)]) == 0
    r1 = list(csv.reader(io.StringIO(t1.read_text())))
    r2 = list(csv.reader(io.StringIO(t2.read_text())))
    assert [r[0] for r in r1[1:4]] == ["a_one_d", "b_rand", "c_broken"]
    assert r1[3][2] == "parse_failure"
    footer = {r[0]: r for r in r1 if r[0].startswith("#")}
    assert footer["#solved"][2] == "2"
    # deterministic apart from the seconds column
    strip = lambda rows: [r[:4] + r[5:] for r in rows if r[0] != "#sgm10_seconds"]
    assert strip(r1) == strip(r2)
