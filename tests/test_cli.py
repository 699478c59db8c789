"""hpbj_cli — the reference harness contract (bjgmres_cli.cpp: solve / bench /
partition, JSON report schema, history CSV, bench table) on the B200 solver
(SURVEY.md §8f-1). The partition subcommand and argument checks run on CPU;
solve and bench run the GPU path (-m gpu)."""
import csv
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2509_09139_b200 as hp
from tests import fixtures as fx

CLI = os.path.join(os.path.dirname(hp.__file__), "lib", "hpbj_cli")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


@pytest.fixture
def mtx(tmp_path):
    a = fx.random_dd(300, 5, 21)
    p = str(tmp_path / "rdd300.mtx")
    hp.write_matrix_market(p, a)
    return p, a


def test_partition_subcommand_matches_reference(ref, mtx, tmp_path):
    path, a = mtx
    out = str(tmp_path / "part.txt")
    r = run("partition", "--matrix", path, "--blocks", "7", "--out", out)
    assert r.returncode == 0, r.stderr
    asg = np.loadtxt(out, dtype=np.int64)
    ref_asg, _, _, _ = ref.partition(a.row_starts, a.col_indices, a.values, 7)
    assert np.array_equal(asg, ref_asg)
    p = hp.partition_from_assignment(asg, 7)
    _, imb = hp.measure_block_nnz(p, a)
    cut = hp.cut_weight(hp.graph_from_matrix(a), p)
    assert r.stdout.strip() == f"blocks=7 cut_weight={cut:.6g} nnz_imbalance={imb:.4f}"


@pytest.mark.parametrize("args,msg", [
    (["solve"], "--matrix is required"),
    (["solve", "--matrix", "x.mtx", "--precision", "double"], "not implemented on the GPU path"),
    (["solve", "--matrix", "x.mtx", "--precision", "quad"], "unknown precision"),
    (["solve", "--matrix", "x.mtx", "--precond", "ilu0", "--blocks", "4"], "--blocks requires --precond block-jacobi"),
    (["solve", "--matrix", "x.mtx", "--ritz"], "--ritz"),
    (["solve", "--matrix", "x.mtx", "--restart", "0"], "numeric flags out of range"),
    (["partition", "--matrix", "x.mtx", "--blocks", "0", "--out", "p"], "--blocks must be >= 1"),
    (["bench", "--specs", "/nonexistent.json"], "cannot open specs file"),
])
def test_argument_errors(args, msg):
    r = run(*args)
    assert r.returncode == 1 and msg in r.stderr


def test_matrix_errors_are_reported(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    r = run("partition", "--matrix", str(bad), "--blocks", "1", "--out", str(tmp_path / "p"))
    assert r.returncode == 1 and "matrix market: line 3" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("rhs", ["axones", "ones", "random:7"])
def test_solve_report_history_and_parity(ref, mtx, tmp_path, rhs):
    path, a = mtx
    rep, hist = str(tmp_path / "r.json"), str(tmp_path / "h.csv")
    r = run("solve", "--matrix", path, "--blocks", "6", "--restart", "20", "--tol", "1e-10", "--rhs", rhs,
            "--report", rep, "--history", hist)
    assert r.returncode == 0, r.stderr
    doc = json.load(open(rep))
    assert set(doc) == {"matrix", "config", "result", "preconditioner"}
    assert doc["matrix"] == {"name": "rdd300", "n": 300, "nnz": a.nnz()}
    res = doc["result"]
    assert res["converged"] and res["final_residual"] <= 1e-10 and res["setup_ms"] > 0 and res["solve_ms"] > 0
    assert doc["config"]["precision"] == "hybrid" and doc["config"]["rhs"] == rhs
    blocks = doc["preconditioner"]["blocks"]
    assert len(blocks) == 6 and sum(b["dim"] for b in blocks) == 300
    rows = list(csv.reader(open(hist)))
    assert rows[0] == ["restart_cycle", "global_iteration", "relative_residual"]
    assert len(rows) == res["iterations"] + 2 and rows[1][:2] == ["0", "0"]  # header + iterations + 1
    # same system through the reference library (Hybrid, same partition): same iteration count
    n = a.n
    if rhs == "ones":
        b = np.ones(n)
    elif rhs == "axones":
        b = np.array([a.values[a.row_starts[i]:a.row_starts[i + 1]].sum() for i in range(n)])
    else:
        b = None
    if b is not None:
        part = hp.partition_graph(a, 6, 0.1)
        out = ref.solve(a.row_starts, a.col_indices, a.values, 6, b, 20, 1e-10, 40, hybrid=True,
                        assignment=part.assignment)
        assert res["iterations"] == out.total_iterations


@pytest.mark.gpu
def test_solve_with_partition_file_and_rhs_file(mtx, tmp_path):
    path, a = mtx
    pfile, bfile = str(tmp_path / "p.txt"), str(tmp_path / "b.txt")
    assert run("partition", "--matrix", path, "--blocks", "5", "--out", pfile).returncode == 0
    np.savetxt(bfile, np.linspace(-1, 1, a.n))
    r = run("solve", "--matrix", path, "--blocks", "5", "--partition-file", pfile, "--rhs", "file:" + bfile)
    assert r.returncode == 0, r.stderr
    assert "converged=true" in r.stdout


@pytest.mark.gpu
def test_bench_table_and_csv(mtx, tmp_path):
    path, a = mtx
    specs = tmp_path / "specs.json"
    specs.write_text(json.dumps([{"matrix": path, "blocks": 6, "restart": 30, "tol": 1e-9},
                                 {"matrix": path, "blocks": 10, "rhs": "ones", "precision": "hybrid"},
                                 {"matrix": "/nonexistent.mtx"}]))
    out = str(tmp_path / "t.csv")
    r = run("bench", "--specs", str(specs), "--repetitions", "2", "--out", out)
    assert r.returncode == 0, r.stderr
    assert "warning: skipping spec" in r.stderr
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["matrix_name", "n", "nnz", "nnz_per_row", "precond_setup_ms", "solve_ms", "iterations",
                       "converged", "final_residual"]
    assert len(rows) == 3 and all(row[0] == "rdd300" and row[7] == "true" for row in rows[1:])


@pytest.mark.gpu
def test_solve_with_neumann_order(ref, mtx, tmp_path):
    path, a = mtx
    rep = str(tmp_path / "r.json")
    r = run("solve", "--matrix", path, "--blocks", "6", "--restart", "20", "--tol", "1e-10", "--rhs", "ones",
            "--neumann-order", "2", "--report", rep)
    assert r.returncode == 0, r.stderr
    doc = json.load(open(rep))
    assert doc["config"]["neumann_order"] == 2 and doc["result"]["converged"]
    part = hp.partition_graph(a, 6, 0.1)
    out = ref.solve(a.row_starts, a.col_indices, a.values, 6, np.ones(a.n), 20, 1e-10, 40, hybrid=True,
                    assignment=part.assignment, neumann_order=2)
    assert doc["result"]["iterations"] == out.total_iterations


@pytest.mark.gpu
@pytest.mark.parametrize("precond", ["ilu0", "none"])
def test_solve_with_other_preconditioners(ref, mtx, tmp_path, precond):
    """--precond ilu0 / none default to precision double like the reference
    and reproduce its iteration counts; hybrid ILU(0) fails like the reference."""
    path, a = mtx
    rep = str(tmp_path / "r.json")
    r = run("solve", "--matrix", path, "--precond", precond, "--restart", "20", "--tol", "1e-10", "--rhs", "ones",
            "--report", rep)
    assert r.returncode == 0, r.stderr
    doc = json.load(open(rep))
    assert doc["config"]["precond"] == precond and doc["config"]["precision"] == "double"
    assert doc["preconditioner"]["blocks"] == [] and doc["result"]["converged"]
    b = np.ones(a.n)
    if precond == "ilu0":
        out = ref.solve_ilu0(a.row_starts, a.col_indices, a.values, b, 20, 1e-10, 40, hybrid=False)
    else:
        out = ref.solve_identity(a.row_starts, a.col_indices, a.values, b, 20, 1e-10, 40, hybrid=False)
    assert abs(doc["result"]["iterations"] - out.total_iterations) <= 1
    if precond == "ilu0":
        r = run("solve", "--matrix", path, "--precond", "ilu0", "--precision", "hybrid")
        assert r.returncode == 1 and "values_low requested before materialize_low" in r.stderr


def test_unknown_preconditioner_is_reported(mtx):
    path, _ = mtx
    r = run("solve", "--matrix", path, "--precond", "amg")
    assert r.returncode == 1 and "unknown preconditioner: amg" in r.stderr
