"""GPU subcommands of the CLI (the reference's harness, bench.py:238-391)."""
import pytest

pytestmark = pytest.mark.gpu


def test_cli_sort_dtsort_and_plain_verified(tmp_path, capsys):
    from paper_2401_00710_b200.cli import main

    f = tmp_path / "d.isrt"
    assert main(["gen", "--dist", "exp", "--param", "2", "--n", "300000", "--bits", "64", "--out", str(f)]) == 0
    for algo in ("dtsort", "plain"):
        o = tmp_path / f"{algo}.isrt"
        assert main(["sort", "--algo", algo, "--in", str(f), "--verify", "--instrument", "--out", str(o)]) == 0
        out = capsys.readouterr().out
        assert "verified=ok" in out and "moves=" in out
        assert main(["verify", "--in", str(o), "--algo", algo]) == 0


def test_cli_bench_grid_small(tmp_path, capsys):
    from paper_2401_00710_b200.cli import CSV_HEADER, main

    csv = tmp_path / "g.csv"
    assert main(["bench", "--preset", "grid32", "--n", "20000", "--repeat", "2", "--csv", str(csv)]) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 1 + 20 * 3
    assert all(",true," in ln for ln in lines[1:])


def test_cli_transpose_and_theory(capsys):
    from paper_2401_00710_b200.cli import main

    assert main(["transpose-demo", "--vertices", "5000", "--edges", "200000", "--skew", "1.1"]) == 0
    out = capsys.readouterr().out
    assert "transposed 200000 edges over 5000 vertices" in out and "stability check: ok" in out
    assert main(["theory-check", "--sizes", "100000", "1000000"]) == 0
    assert "accounting bounds hold" in capsys.readouterr().out
