"""Dataset layer: the harness port of the
reference's generators (harness/refgen.py) and the ISRT writer
(paper_2401_00710_b200/isrt.py) byte-identical to the reference (golden
SHA-256 from tests/golden/make_datasets_golden.py), reader validation
messages, and the CLI's `gen`.  The device subcommands are in
test_gpu_cli.py."""
import hashlib
import json
import pathlib

import numpy as np
import pytest

from paper_2401_00710_b200.core import RecordArray
from harness.refgen import DistSpec, generate, generate_edges
from paper_2401_00710_b200.isrt import read_dataset, read_header, write_dataset

G = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "datasets_golden.json").read_text())


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("c", G["generate"], ids=lambda c: f"{c['family']}{c['param']}-{c['bits']}-{c['n']}")
def test_generate_matches_reference(c):
    r = generate(DistSpec(c["family"], c["param"], c["n"], c["bits"], c["seed"]))
    assert sha(r.keys) == c["keys"] and sha(r.payloads) == c["pays"]


def test_generate_edges_matches_reference():
    e = G["edges"]
    src, dst = generate_edges(e["vertices"], e["edges"], e["skew"], e["seed"])
    assert sha(src) == e["src"] and sha(dst) == e["dst"]


@pytest.mark.parametrize("f", G["files"], ids=lambda f: f"pw{f['payload_width']}")
def test_written_file_matches_reference(tmp_path, f):
    r = generate(DistSpec(f["family"], f["param"], f["n"], f["bits"], f["seed"]))
    rec = r if f["payload_width"] else RecordArray(r.keys)
    path = tmp_path / "x.isrt"
    write_dataset(path, rec, payload_width=f["payload_width"])
    assert hashlib.sha256(path.read_bytes()).hexdigest() == f["sha"]
    back, pw = read_dataset(path)
    assert pw == f["payload_width"] and np.array_equal(back.keys, r.keys)
    if pw:
        assert np.array_equal(back.payloads, r.payloads)


def test_reader_errors(tmp_path):
    p = tmp_path / "bad"
    p.write_bytes(b"abc")
    with pytest.raises(ValueError, match="truncated before header"):
        read_dataset(p)
    p.write_bytes(b"XXXX" + bytes(12))
    with pytest.raises(ValueError, match="bad magic"):
        read_dataset(p)
    r = generate(DistSpec("uniform", 10.0, 10))
    write_dataset(p, r)
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(ValueError, match="length mismatch"):
        read_dataset(p)
    with pytest.raises(ValueError, match="payload_width must be 0, 4, or 8"):
        write_dataset(p, r, payload_width=2)


def test_distspec_validation():
    with pytest.raises(ValueError, match="unknown family"):
        DistSpec("nope", 1.0, 10)
    with pytest.raises(ValueError, match="uniform needs an integer key count"):
        DistSpec("uniform", 0.5, 10)
    with pytest.raises(ValueError, match="bexp needs odds"):
        DistSpec("bexp", 0.5, 10)


def test_cli_gen_writes_the_reference_bytes(tmp_path, capsys):
    from paper_2401_00710_b200.cli import main

    f = tmp_path / "d.isrt"
    assert main(["gen", "--dist", "zipf", "--param", "1.2", "--n", "20000", "--out", str(f)]) == 0
    assert "wrote 20000 32-bit records (zipf 1.2)" in capsys.readouterr().out
    recs, pw = read_dataset(f)
    want = generate(DistSpec("zipf", 1.2, 20000))
    assert pw == 8 and np.array_equal(recs.keys, want.keys) and np.array_equal(recs.payloads, want.payloads)
    h = read_header(f)
    assert (h.key_bits, h.payload_width, h.count) == (32, 8, 20000)


def test_isrt_chunked_write_and_empty_file(tmp_path):
    import paper_2401_00710_b200.isrt as isrt

    isrt._CHUNK, old = 1000, isrt._CHUNK  # several chunks
    try:
        r = generate(DistSpec("exp", 2.0, 4321, 64, 3))
        for pw in (0, 4, 8):
            p = tmp_path / f"x{pw}.isrt"
            write_dataset(p, r if pw else RecordArray(r.keys), payload_width=pw)
            back, bpw = read_dataset(p)
            assert bpw == pw and np.array_equal(back.keys, r.keys)
            if pw:
                assert np.array_equal(back.payloads, r.payloads)
    finally:
        isrt._CHUNK = old
    e = tmp_path / "e.isrt"
    write_dataset(e, RecordArray(np.empty(0, np.uint32)))
    back, pw = read_dataset(e)
    assert len(back) == 0 and pw == 0
