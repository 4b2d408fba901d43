"""Generate the golden fixtures from the REFERENCE package itself.

Runs only in the build container (it imports /root/reference/pkg/src);
the fixtures it writes are committed and travel to the GPU box.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes:
  sort_golden.json   per case: reference dt_sort / plain_msd_sort output
                     SHA-256 and InstrumentReport.structural() counters,
                     plus the C1 / C2-shape known-answer digests.
  small_cases.npz    raw input/output arrays of the n <= 1000 cases.
  merge_golden.npz   reference dt_merge outputs + MergeStats on the
                     exhaustive 70 x 64 grid and 400 random zones.
  philox_golden.npz  numpy Generator(Philox(key)).integers draws.
"""
from __future__ import annotations

import json
import os
import pathlib
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from dovetail.bench import reference_sort  # noqa: E402
from dovetail.core import RecordArray, SortConfig  # noqa: E402
from dovetail.dtmerge import dt_merge  # noqa: E402
from dovetail.dtsort import dt_sort, plain_msd_sort  # noqa: E402


def structural(rep) -> dict:
    return {
        "moves": rep.moves,
        "merge_out_copies": rep.merge_out_copies,
        "merge_in_array_moves": rep.merge_in_array_moves,
        "levels": rep.levels,
        "level_mass": list(rep.level_mass),
        "base_case_records": rep.base_case_records,
        "heavy_records_removed": list(rep.heavy_records_removed),
        "skipped_bits": rep.skipped_bits,
    }


def main() -> None:
    out = {"cases": [], "known": {}}
    small = {}
    for case in cases.sort_cases():
        keys, pays = cases.make_input(case)
        entry = dict(case)
        entry["input_sha"] = cases.sha(keys, pays)
        for mode, fn in (("dt", dt_sort), ("plain", plain_msd_sort)):
            rec = RecordArray(keys.copy(), None if pays is None else pays.copy())
            rep = fn(rec, SortConfig(instrument=True, **case["cfg"]))
            entry[f"{mode}_sha"] = cases.sha(rec.keys, rec.payloads)
            entry[f"{mode}_report"] = structural(rep)
            if mode == "dt" and case["n"] <= 1000:
                small[case["name"] + "/in_keys"] = keys
                small[case["name"] + "/out_keys"] = rec.keys
                if pays is not None:
                    small[case["name"] + "/out_pays"] = rec.payloads
        assert entry["dt_sha"] == entry["plain_sha"]
        ref = reference_sort(RecordArray(keys.copy(), None if pays is None else pays.copy()))
        assert cases.sha(ref.keys, ref.payloads) == entry["dt_sha"]
        out["cases"].append(entry)
        print(case["name"], entry["dt_report"]["levels"], flush=True)

    # C1 (BASELINE.json configs[0]) and the C2 shape at n=1e6
    c1 = np.random.default_rng(0).integers(0, 2**32, size=10**6, dtype=np.uint32)
    rec = RecordArray(c1.copy())
    rep = dt_sort(rec, SortConfig(seed=0, instrument=True))
    out["known"]["c1"] = {"input_sha": cases.sha(c1), "output_sha": cases.sha(rec.keys),
                          "report": structural(rep), "first_keys": c1[:2].tolist(),
                          "min": int(rec.keys[0]), "max": int(rec.keys[-1]),
                          "distinct": int(np.unique(rec.keys).size)}
    c2k = np.random.default_rng(0).integers(0, 10**9, size=10**6, dtype=np.uint32)
    c2v = np.arange(10**6, dtype=np.uint64)
    rec = RecordArray(c2k.copy(), c2v.copy())
    rep = dt_sort(rec, SortConfig(seed=0, instrument=True))
    out["known"]["c2_1e6"] = {"input_sha": cases.sha(c2k), "keys_sha": cases.sha(rec.keys),
                              "vals_u32_sha": cases.sha(rec.payloads.astype(np.uint32)),
                              "report": structural(rep)}
    (HERE / "sort_golden.json").write_text(json.dumps(out, indent=1))
    np.savez_compressed(HERE / "small_cases.npz", **small)

    # dt_merge: exhaustive grid + random zones (test_dtmerge.py:62-97 shapes)
    mk, mp, ms, moff = [], [], [], [0]
    for light, heavy in cases.merge_grid():
        keys, pays = cases.build_zone(light, heavy)
        hk = np.array([k for k, _ in heavy], dtype=np.uint32)
        hl = np.array([ln for _, ln in heavy], dtype=np.int64)
        small_side = min(len(light), int(hl.sum()))
        st = dt_merge(keys, pays, len(light), hk, hl, np.empty(small_side, np.uint32),
                      np.empty(small_side, np.uint64))
        mk.append(keys); mp.append(pays)
        ms.append([st.out_copies, st.in_array_moves, st.restore_copies])
        moff.append(moff[-1] + keys.shape[0])
    rng = np.random.default_rng(2024)
    rand = []
    for trial in range(400):
        light_len = int(rng.integers(0, 300))
        m = int(rng.integers(0, 33))
        universe = int(rng.integers(4, 500))
        light = np.sort(rng.integers(0, universe, size=light_len) * 2)
        hk = np.sort(rng.choice(universe, size=min(m, universe), replace=False) * 2 + 1)
        heavy = [(int(k), int(rng.integers(0, 40))) for k in hk]
        keys, pays = cases.build_zone(light.tolist(), heavy, np.uint64 if trial % 2 == 0 else np.uint32)
        hka = np.array([k for k, _ in heavy], dtype=keys.dtype)
        hl = np.array([ln for _, ln in heavy], dtype=np.int64)
        small_side = min(light_len, int(hl.sum()))
        zk_in = keys.copy()
        st = dt_merge(keys, pays, light_len, hka, hl, np.empty(small_side, keys.dtype),
                      np.empty(small_side, np.uint64))
        rand.append(dict(light_len=light_len, heavy=heavy, wide=trial % 2 == 0,
                         in_sha=cases.sha(zk_in), out_sha=cases.sha(keys, pays),
                         stats=[st.out_copies, st.in_array_moves, st.restore_copies]))
    np.savez_compressed(HERE / "merge_golden.npz", keys=np.concatenate(mk), pays=np.concatenate(mp),
                        stats=np.array(ms, np.int64), offsets=np.array(moff, np.int64))
    (HERE / "merge_random.json").write_text(json.dumps(rand))

    # numpy Philox bounded draws (pins the oracle's sampler RNG)
    draws = {}
    for i, (k0, k1, high) in enumerate([(0, 1 << 60, 1000), (7, 11, 10**7 + 3),
                                        (123, (1 << 60) | (5 << 48) | (77 << 8) | 3, 999_999_937),
                                        (5, 1 << 62, (1 << 40) + 7)]):
        g = np.random.Generator(np.random.Philox(key=np.array([k0, k1], dtype=np.uint64)))
        draws[f"d{i}"] = g.integers(0, high, size=20_000, dtype=np.uint64)
        draws[f"p{i}"] = np.array([k0, k1, high], dtype=np.uint64)
    np.savez_compressed(HERE / "philox_golden.npz", **draws)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
