"""GPU subcommands of the CLI (the reference's harness, bench.py:238-391)."""
import numpy as np
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


def test_cli_verify_and_baseline_sort(tmp_path, capsys):
    from harness.refgen import DistSpec, generate
    from paper_2401_00710_b200.cli import main, reference_sort
    from paper_2401_00710_b200.isrt import read_dataset, write_dataset

    f = tmp_path / "d.isrt"
    assert main(["gen", "--dist", "zipf", "--param", "1.2", "--n", "20000", "--out", str(f)]) == 0
    capsys.readouterr()
    recs, _ = read_dataset(f)
    write_dataset(tmp_path / "s.isrt", reference_sort(recs))
    for algo in ("baseline", "dtsort", "plain"):
        assert main(["verify", "--in", str(tmp_path / "s.isrt"), "--algo", algo]) == 0
        assert "verified: stable sort output of 20000 records" in capsys.readouterr().out
    assert main(["verify", "--in", str(f)]) == 1  # unsorted input is rejected
    assert main(["sort", "--algo", "baseline", "--in", str(f), "--verify", "--out", str(tmp_path / "b.isrt")]) == 0
    assert "verified=ok" in capsys.readouterr().out
    # a file whose equal keys are out of input order is not a stable sort
    bad = reference_sort(recs)
    k = bad.keys
    i = int(np.nonzero(k[1:] == k[:-1])[0][0])
    p = bad.payloads.copy()
    p[i], p[i + 1] = p[i + 1], p[i]
    write_dataset(tmp_path / "u.isrt", type(bad)(k, p))
    assert main(["verify", "--in", str(tmp_path / "u.isrt")]) == 1
    # 4-byte payloads round-trip through the device path
    write_dataset(tmp_path / "p4.isrt", recs, payload_width=4)
    assert main(["sort", "--in", str(tmp_path / "p4.isrt"), "--verify", "--out", str(tmp_path / "p4s.isrt")]) == 0
    back, pw = read_dataset(tmp_path / "p4s.isrt")
    want = reference_sort(recs)
    assert pw == 4 and np.array_equal(back.keys, want.keys) and np.array_equal(back.payloads, want.payloads)
