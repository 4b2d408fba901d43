"""Pin the counter replay (paper_2401_00710_b200/replay.py, SURVEY.md §8(f)
row 1) against the reference's own InstrumentReports, recorded in
tests/golden/sort_golden.json by tests/golden/make_golden.py from the
reference package.  The GPU supplies (sorted keys, stable permutation) at
run time; here numpy's stable argsort stands in for it (test
infrastructure), so this checks the replay logic on the CPU."""
import json
import pathlib

import numpy as np
import pytest

import cases
from paper_2401_00710_b200.core import SortConfig
from paper_2401_00710_b200.replay import replay_report

G = pathlib.Path(__file__).resolve().parent / "golden"
GOLD = json.loads((G / "sort_golden.json").read_text())


def _report(keys, cfg, plain):
    perm = np.argsort(keys, kind="stable")
    rep = replay_report(keys, keys[perm], perm, SortConfig(instrument=True, **cfg), plain)
    return {
        "moves": rep.moves,
        "merge_out_copies": rep.merge_out_copies,
        "merge_in_array_moves": rep.merge_in_array_moves,
        "levels": rep.levels,
        "level_mass": rep.level_mass,
        "base_case_records": rep.base_case_records,
        "heavy_records_removed": rep.heavy_records_removed,
        "skipped_bits": rep.skipped_bits,
    }


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_replay_counters_match_reference(case):
    keys, _ = cases.make_input(case)
    for mode in ("dt", "plain"):
        want = case[f"{mode}_report"]
        got = _report(keys, dict(case["cfg"]), mode == "plain")
        assert {k: got[k] for k in want} == want, mode


def test_replay_known_answer_c1():
    kc = GOLD["known"]["c1"]
    c1 = np.random.default_rng(0).integers(0, 2**32, size=10**6, dtype=np.uint32)
    got = _report(c1, {}, False)
    assert {k: got[k] for k in kc["report"]} == kc["report"]
