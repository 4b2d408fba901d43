"""Pin the CPU oracle against fixtures generated from the reference package
itself (tests/golden/make_golden.py): outputs byte-for-byte, and — because
the oracle restates numpy's Philox sampler — the InstrumentReport counters
exactly."""
import json
import pathlib

import numpy as np
import pytest

import cases
from oracle import oracle as ora

G = pathlib.Path(__file__).resolve().parent / "golden"
GOLD = json.loads((G / "sort_golden.json").read_text())


def _cfg(case):
    return {k: v for k, v in case["cfg"].items()}


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_oracle_sort_matches_reference(case):
    keys, pays = cases.make_input(case)
    assert cases.sha(keys, pays) == case["input_sha"]
    for mode in ("dt", "plain"):
        k = keys.copy()
        p = None if pays is None else pays.copy()
        rep = ora.sort_inplace(k, p, mode, report=True, **_cfg(case))
        assert cases.sha(k, p) == case[f"{mode}_sha"], mode
        want = case[f"{mode}_report"]
        got = {key: rep[key] for key in want}
        assert got == want, mode


def test_oracle_small_cases_raw_arrays():
    data = np.load(G / "small_cases.npz")
    names = sorted({k.split("/")[0] for k in data.files})
    assert names
    for name in names:
        k_in = data[name + "/in_keys"]
        pays = np.arange(k_in.shape[0], dtype=np.uint64)
        k, p = ora.dt_sort(k_in, pays)
        assert np.array_equal(k, data[name + "/out_keys"])
        if name + "/out_pays" in data.files:
            assert np.array_equal(p, data[name + "/out_pays"])


def test_known_answer_c1_and_c2_shape():
    c1 = np.random.default_rng(0).integers(0, 2**32, size=10**6, dtype=np.uint32)
    kc = GOLD["known"]["c1"]
    assert cases.sha(c1) == kc["input_sha"]
    assert c1[:2].tolist() == kc["first_keys"] == [3653403231, 2735729615]
    k = c1.copy()
    rep = ora.sort_inplace(k, None, "dt", report=True)
    assert cases.sha(k) == kc["output_sha"]
    # SURVEY.md §8c digests computed from the reference
    assert kc["output_sha"] == "3ed7cae1f3151dac77ecb9a5e3ed6a482d7d49327323089e406046683fa350de"
    assert {key: rep[key] for key in kc["report"]} == kc["report"]
    c2k = np.random.default_rng(0).integers(0, 10**9, size=10**6, dtype=np.uint32)
    c2v = np.arange(10**6, dtype=np.uint32)
    k2, v2 = ora.dt_sort(c2k, c2v)
    kn = GOLD["known"]["c2_1e6"]
    assert cases.sha(c2k) == kn["input_sha"] == "73470bde16cb07150aac4bb1bce7cee70a3d20a23a5e7a4a83c75360b91b2403"
    assert cases.sha(k2) == kn["keys_sha"] == "6a297e05c43b6653838aed3f7d053dce0f0679117ea3979a216aa97740ba0399"
    assert cases.sha(v2) == kn["vals_u32_sha"] == "096bf2bd3d60623a8543a956f55133eb24349e0ca8f3a63feb8b88841d6a757b"


def test_oracle_dt_merge_exhaustive_grid():
    g = np.load(G / "merge_golden.npz")
    offs = g["offsets"]
    for i, (light, heavy) in enumerate(cases.merge_grid()):
        keys, pays = cases.build_zone(light, heavy)
        hk = np.array([k for k, _ in heavy], dtype=np.uint32)
        hl = np.array([ln for _, ln in heavy], dtype=np.int64)
        st = ora.dt_merge(keys, pays, len(light), hk, hl)
        assert np.array_equal(keys, g["keys"][offs[i]:offs[i + 1]])
        assert np.array_equal(pays, g["pays"][offs[i]:offs[i + 1]])
        assert list(st) == g["stats"][i].tolist()


def test_oracle_dt_merge_random_zones():
    rand = json.loads((G / "merge_random.json").read_text())
    rng = np.random.default_rng(2024)
    for trial, r in enumerate(rand):
        light_len = int(rng.integers(0, 300))
        m = int(rng.integers(0, 33))
        universe = int(rng.integers(4, 500))
        light = np.sort(rng.integers(0, universe, size=light_len) * 2)
        hk = np.sort(rng.choice(universe, size=min(m, universe), replace=False) * 2 + 1)
        heavy = [(int(k), int(rng.integers(0, 40))) for k in hk]
        assert heavy == [tuple(h) for h in r["heavy"]]
        keys, pays = cases.build_zone(light.tolist(), heavy, np.uint64 if r["wide"] else np.uint32)
        assert cases.sha(keys) == r["in_sha"]
        st = ora.dt_merge(keys, pays, light_len, [k for k, _ in heavy], [ln for _, ln in heavy])
        assert cases.sha(keys, pays) == r["out_sha"]
        assert list(st) == r["stats"]


def test_oracle_dt_merge_known_case_and_errors():
    keys = np.array([1, 3, 5, 4, 4], np.uint32)
    pays = np.arange(5, dtype=np.uint64)
    ora.dt_merge(keys, pays, 3, [4], [2])
    assert keys.tolist() == [1, 3, 4, 4, 5] and pays.tolist() == [0, 1, 3, 4, 2]
    for args, msg in [
        (([1, 2, 9, 9], 3, [9], [2]), "tile"),
        (([1, 2, 9], 2, [5, 9], [-1, 2]), "nonnegative"),
        (([1, 2, 9, 5], 2, [9, 5], [1, 1]), "increasing"),
        (([2, 1, 9], 2, [9], [1]), "sorted"),
        (([1, 9, 9], 2, [9], [1]), "light run"),
        (([1, 2, 9, 8], 2, [9], [2]), "foreign"),
    ]:
        k = np.asarray(args[0], np.uint32)
        with pytest.raises(ValueError, match=msg):
            ora.dt_merge(k, np.arange(k.shape[0], dtype=np.uint64), args[1], args[2], args[3],
                         scratch_len=64)


def test_oracle_philox_matches_numpy_draws():
    d = np.load(G / "philox_golden.npz")
    for i in range(4):
        k0, k1, high = (int(x) for x in d[f"p{i}"])
        assert np.array_equal(ora.philox_integers(k0, k1, high, 20_000), d[f"d{i}"])


def test_oracle_counting_sort_known_answer():
    # reference test_counting.py:46-51: [5,3,5,3,5,3], bucket k//4
    keys = np.array([5, 3, 5, 3, 5, 3], np.uint32)
    pays = np.arange(6, dtype=np.uint64)
    ok, op, offs = ora.counting_sort(keys, pays, keys // 4, 2)
    assert ok.tolist() == [3, 3, 3, 5, 5, 5]
    assert op.tolist() == [1, 3, 5, 0, 2, 4]
    assert offs.tolist() == [0, 3, 6]


def test_reference_sort_restatement_and_certificate():
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 1000, 50_000):
        k = rng.integers(0, 50, size=n).astype(np.uint32)
        v = np.arange(n, dtype=np.uint32)
        rk, rv = ora.reference_sort(k, v)
        order = np.argsort(k, kind="stable")
        assert np.array_equal(rk, k[order]) and np.array_equal(rv, v[order])
        assert ora.stable_certificate(k, rk, rv)
        if n > 2:
            bad = rv.copy()
            bad[[0, 1]] = bad[[1, 0]]
            assert not ora.stable_certificate(k, rk, bad)
