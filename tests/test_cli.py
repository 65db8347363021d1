"""The `search` subcommand of the reference CLI on the engine
(paper_0804_1448_b200/knn_b200_cli), ported from the reference's
tests/test_cli.cpp:58-106: exact text on the three-point fixture, atomic
--out, exit 2 + line number on malformed CSV, exit 3 + one-line "error:" on
contract violations, non-zero on unknown flags.  The error cases fail before
any device work and run on CPU; the searches need a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_0804_1448_b200", "knn_b200_cli")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_0804_1448_b200")], check=True)
    return CLI


def run(cli, *args):
    r = subprocess.run([cli, *args], capture_output=True, text=True, timeout=120)
    return r.returncode, r.stdout, r.stderr


def write(path, text):
    with open(path, "w") as f:
        f.write(text)
    return str(path)


@pytest.mark.gpu
def test_search_happy_path_three_point_fixture(cli, tmp_path):
    refs = write(tmp_path / "refs.csv", "0,0\n1,0\n2,0\n")
    query = write(tmp_path / "query.csv", "0.1,0\n")
    code, out, _ = run(cli, "search", "--ref", refs, "--query", query, "--k", "3", "--metric",
                       "euclidean")
    assert code == 0
    assert out == ("query_index,rank,ref_index,distance\n"
                   "0,0,0,0.1\n"
                   "0,1,1,0.9\n"
                   "0,2,2,1.9\n")
    code2, out2, _ = run(cli, "search", "--ref", refs, "--query", query, "--k", "3", "--method",
                         "kdtree")
    assert code2 == 0 and out2 == out


@pytest.mark.gpu
def test_search_writes_out_atomically_and_identically(cli, tmp_path):
    refs = write(tmp_path / "refs.csv", "0,0\n1,0\n2,0\n")
    query = write(tmp_path / "query.csv", "0.1,0\n")
    out = str(tmp_path / "result.csv")
    code, _, _ = run(cli, "search", "--ref", refs, "--query", query, "--k", "2", "--out", out)
    assert code == 0
    assert not os.path.exists(out + ".tmp")
    first = open(out).read()
    code, _, _ = run(cli, "search", "--ref", refs, "--query", query, "--k", "2", "--out", out)
    assert code == 0 and open(out).read() == first


@pytest.mark.gpu
def test_search_metrics_and_comments(cli, tmp_path):
    refs = write(tmp_path / "refs.csv", "# points\n0,0\n\n3,4\n1,1\n")
    query = write(tmp_path / "query.csv", "0,0\n")
    mat = write(tmp_path / "m.csv", "2,0\n0,2\n")
    expect = {"euclidean": [0, 2 ** 0.5, 5], "manhattan": [0, 2, 7], "chebyshev": [0, 1, 4],
              "mahalanobis:" + mat: [0, 2, 50 ** 0.5]}
    for metric, dists in expect.items():
        code, out, err = run(cli, "search", "--ref", refs, "--query", query, "--k", "3",
                             "--metric", metric)
        assert code == 0, err
        rows = out.strip().split("\n")[1:]
        assert [r.split(",")[2] for r in rows] == ["0", "2", "1"]
        got = [float(r.split(",")[3]) for r in rows]
        assert got == pytest.approx(dists, rel=1e-6, abs=1e-7), metric


def test_malformed_csv_exits_2_and_names_the_line(cli, tmp_path):
    bad = write(tmp_path / "bad.csv", "0,0\n1\n")
    query = write(tmp_path / "query.csv", "0.1,0\n")
    code, _, err = run(cli, "search", "--ref", bad, "--query", query, "--k", "1")
    assert code == 2
    assert "line 2" in err


def test_contract_violations_exit_3(cli, tmp_path):
    refs = write(tmp_path / "refs.csv", "0,0\n1,0\n")
    query = write(tmp_path / "query.csv", "0.1,0\n")
    code, _, err = run(cli, "search", "--ref", refs, "--query", query, "--k", "5")
    assert code == 3
    assert "error:" in err
    assert err.find("\n") == len(err) - 1  # single line


def test_unknown_flags_are_an_error(cli):
    code, _, _ = run(cli, "search", "--frobnicate", "3")
    assert code != 0


@pytest.mark.gpu
def test_bench_grid_report(cli, tmp_path):
    """knn-cli bench (bench.cpp:75-166, 207-232) for the bf method: the report
    schema, one row per (n, d) cell, n*n distance evaluations, JSON twin."""
    import json
    out, js = str(tmp_path / "grid.csv"), str(tmp_path / "grid.json")
    code, _, err = run(cli, "bench", "--n-values", "300,500", "--d-values", "8,16,32", "--k",
                       "5", "--reps", "2", "--seed", "42", "--out", out, "--json", js)
    assert code == 0, err
    lines = open(out).read().strip().split("\n")
    assert lines[0] == "method,n,d,k,seconds,dist_evals,seed"
    rows = [r.split(",") for r in lines[1:]]
    assert [(r[0], int(r[1]), int(r[2])) for r in rows] == [
        ("bf", n, d) for n in (300, 500) for d in (8, 16, 32)]
    for r in rows:
        n = int(r[1])
        assert int(r[3]) == 5 and float(r[4]) > 0 and int(r[5]) == n * n and r[6] == "42"
    doc = json.load(open(js))
    assert len(doc["rows"]) == 6 and all(not row["skipped"] for row in doc["rows"])


def test_bench_grid_contract_errors(cli):
    code, _, err = run(cli, "bench", "--methods", "bf,kdt", "--reps", "1")
    assert code == 3 and "not available" in err
    code, _, err = run(cli, "bench", "--k", "5000", "--reps", "1")
    assert code == 3 and "exceeds cell size" in err
