"""Command-line front end (cli.py; the reference's chordalkit/cli.py): host-side
behaviour here -- generators against the reference's outputs, exit codes for
unusable input; GPU verdicts in the `gpu`-marked tests below."""

import hashlib
import json
import os

import pytest

from paper_1508_06329_b200.cli import main, make_graph
from paper_1508_06329_b200.textio import write_graph_text

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cli_gen.json")


@pytest.mark.parametrize("case", json.load(open(GOLDEN))["cases"],
                         ids=lambda c: f"{c['cls']}-{c['n']}-{c['param']}-{c['seed']}")
def test_gen_matches_reference(case):
    text = write_graph_text(make_graph(case["cls"], case["n"], case["seed"], case["param"]))
    assert hashlib.sha256(text.encode()).hexdigest() == case["sha256"]


def test_gen_writes_file(tmp_path, capsys):
    out = tmp_path / "g.txt"
    assert main(["gen", "chordal", "30", "--seed", "4", "--out", str(out)]) == 0
    assert capsys.readouterr().out.startswith("n=30 m=")
    assert out.read_text() == write_graph_text(make_graph("chordal", 30, 4))


def test_malformed_input_and_missing_file_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.txt"
    bad.write_text("p 2 1\nbogus\n")
    assert main(["check", str(bad)]) == 2
    assert "error:" in capsys.readouterr().err
    assert main(["check", "/nonexistent/graph.txt"]) == 2
    assert main(["order", str(bad)]) == 2


def test_verify_oracle_properties_are_out_of_scope(tmp_path, capsys):
    g = tmp_path / "c4.txt"
    g.write_text("p 4 4\ne 1 2\ne 1 4\ne 2 3\ne 3 4\n")
    o = tmp_path / "o.txt"
    o.write_text("1 2 4 3\n")
    assert main(["verify", str(g), str(o), "lb"]) == 2
    assert "only 'peo'" in capsys.readouterr().err


# ---- GPU: the reference's test_cli.py goldens ----------------------------------

C4 = "p 4 4\ne 1 2\ne 1 4\ne 2 3\ne 3 4\n"
K4 = "p 4 6\ne 1 2\ne 1 3\ne 1 4\ne 2 3\ne 2 4\ne 3 4\n"
P3 = "p 3 2\ne 1 2\ne 2 3\n"


def _p(tmp_path, name, text):
    f = tmp_path / name
    f.write_text(text)
    return str(f)


@pytest.mark.gpu
def test_check_goldens(tmp_path, capsys):
    assert main(["check", _p(tmp_path, "c4.txt", C4)]) == 1
    out = capsys.readouterr().out
    assert "chordal: no" in out and "witness: v=3 p=4 z=2" in out and "algorithm ms:" in out
    for algo in ("seq-labels", "seq-partition", "parallel"):
        assert main(["check", _p(tmp_path, "k4.txt", K4), "--algo", algo]) == 0
        assert "peo: 1 2 3 4" in capsys.readouterr().out
    assert main(["check", _p(tmp_path, "c4.txt", C4), "--algo", "parallel", "--seed", "5"]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("algo,text,expected", [("lexbfs-labels", C4, "1 2 4 3\n"), ("lexbfs-partition", C4, "1 2 4 3\n"),
                                                ("parallel-lexbfs", C4, "1 2 4 3\n"), ("mcs", K4, "1 2 3 4\n"),
                                                ("bfs", P3, "1 2 3\n")])
def test_order_goldens(tmp_path, capsys, algo, text, expected):
    assert main(["order", _p(tmp_path, "g.txt", text), "--algo", algo]) == 0
    assert capsys.readouterr().out == expected


@pytest.mark.gpu
def test_verify_and_bench(tmp_path, capsys):
    assert main(["verify", _p(tmp_path, "c4.txt", C4), _p(tmp_path, "o.txt", "1 2 4 3\n"), "peo"]) == 1
    assert "counterexample: v=3 p=4 z=2" in capsys.readouterr().out
    assert main(["verify", _p(tmp_path, "k4.txt", K4), _p(tmp_path, "o.txt", "1 2 3 4\n"), "peo"]) == 0
    capsys.readouterr()
    out = tmp_path / "b.csv"
    assert main(["bench", "--classes", "clique", "chordal", "tree", "--sizes", "60", "--reps", "1",
                 "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "class,n,m,algo,rep,seed,phase,ms" and len(lines) == 1 + 3 * 2 * 2
