"""InstrumentReport counters of the GPU sort against the reference's own
counter tests.

Each test restates the assertions of one reference test, re-pointed at this
package: pkg/tests/test_dtsort.py:106-197 and
pkg/tests/test_acceptance.py:161-192 (criteria 5 and 6).  The counters
follow the reference's structure when SortConfig(instrument=True): the
reference digit policy (core.py:154-164), its base-case threshold
(core.py:148-151), the root's gamma-granular leading-digit skip
(sampler.py:192-207) and its `moves` accounting (dtsort.py:64-108).
The report is the host replay of the reference recursion
(paper_2401_00710_b200/replay.py) over the GPU's stable (key, index) sort,
drawing the reference's own numpy Philox sample streams, so the counters
equal the reference's value for value (pinned on the 99 golden reports in
tests/test_replay_golden.py and through the GPU at the end of this file);
the GPU pipeline's own structure is checked in tests/test_gpu_structure.py.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rec(keys, pay=True):
    from paper_2401_00710_b200 import RecordArray

    keys = np.array(keys, copy=True)  # dt_sort sorts in place
    return RecordArray(keys, np.arange(keys.shape[0], dtype=np.uint64) if pay else None)


def predicted_levels(n, key_width, cfg, skipped_bits=0):
    """Reference bench.py:201-218: passes of a perfectly balanced run."""
    from paper_2401_00710_b200 import gamma_for

    remaining = key_width - skipped_bits
    n_prime = int(n)
    levels = 0
    while remaining > 0 and n_prime > 0:
        gamma = gamma_for(n_prime, remaining, cfg)
        if n_prime < cfg.effective_theta(gamma):
            break
        levels += 1
        remaining -= gamma
        n_prime >>= gamma
    return levels


def test_instrument_invariants_random_input():
    """test_dtsort.py:106-116"""
    from paper_2401_00710_b200 import SortConfig, dt_sort

    rng = np.random.default_rng(4)
    n = 120_000
    rec = _rec(rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32))
    rep = dt_sort(rec, SortConfig(instrument=True))
    assert rep.level_mass[0] == n
    assert rep.levels <= -(-32 // 8)
    assert rep.moves <= 3 * max(rep.levels, 1) * n
    for d in range(rep.levels):
        removed = rep.heavy_records_removed[d] if d < len(rep.heavy_records_removed) else 0
        assert rep.level_mass[d + 1] <= rep.level_mass[d] - removed
    assert rep.base_case_records <= n


def test_all_equal_heavy_shortcut():
    """test_dtsort.py:119-136"""
    from paper_2401_00710_b200 import SortConfig, dt_sort, plain_msd_sort

    n = 200_000
    rec = _rec(np.full(n, 123_456, np.uint32))
    rep = dt_sort(rec, SortConfig(instrument=True))
    assert np.all(rec.keys == 123_456)
    assert np.array_equal(rec.payloads, np.arange(n, dtype=np.uint64))
    assert rep.levels == 1
    assert rep.level_mass[1] == 0
    assert rep.heavy_records_removed[0] == n
    assert rep.moves == 2 * n
    assert rep.skipped_bits == 8

    rec = _rec(np.full(n, 123_456, np.uint32))
    prep = plain_msd_sort(rec, SortConfig(instrument=True))
    assert np.all(rec.keys == 123_456)
    assert prep.levels == 4
    assert prep.moves >= 4 * n


def test_all_zero_keys_skip_cap():
    """test_dtsort.py:139-143"""
    from paper_2401_00710_b200 import SortConfig, dt_sort

    rec = _rec(np.zeros(50_000, np.uint32))
    rep = dt_sort(rec, SortConfig(instrument=True))
    assert rep.skipped_bits == 24
    assert rep.levels == 1


def test_small_keys_skip_leading_digits():
    """test_dtsort.py:146-151"""
    from paper_2401_00710_b200 import SortConfig, dt_sort

    rng = np.random.default_rng(5)
    rec = _rec(rng.integers(0, 1 << 16, size=100_000).astype(np.uint32))
    rep = dt_sort(rec, SortConfig(instrument=True))
    assert rep.skipped_bits == 16
    assert np.all(np.diff(rec.keys.astype(np.int64)) >= 0)


def test_overflow_bucket_catches_rare_outliers():
    """test_dtsort.py:154-172"""
    from paper_2401_00710_b200 import SortConfig, dt_sort

    rng = np.random.default_rng(6)
    base = rng.integers(0, 1 << 12, size=150_000, dtype=np.uint32)
    outliers = np.array([1 << 20, (1 << 32) - 1, 1 << 28], np.uint32)
    saw_skip = False
    for seed in range(12):
        keys = base.copy()
        keys[rng.integers(0, len(keys), size=3)] = outliers
        order = np.argsort(keys, kind="stable")
        rec = _rec(keys)
        rep = dt_sort(rec, SortConfig(seed=seed, instrument=True))
        assert np.array_equal(rec.keys, keys[order])
        assert np.array_equal(rec.payloads, order.astype(np.uint64))
        if rep.skipped_bits:
            saw_skip = True
            assert rep.skipped_bits == 16
            assert rep.levels == 1
            break
    assert saw_skip


def test_merge_traffic_on_planted_heavy_keys():
    """test_dtsort.py:175-186"""
    from paper_2401_00710_b200 import SortConfig, dt_sort

    rng = np.random.default_rng(7)
    n = 100_000
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    keys[: n // 3] = 0x12345678
    rng.shuffle(keys)
    order = np.argsort(keys, kind="stable")
    rec = _rec(keys)
    rep = dt_sort(rec, SortConfig(instrument=True))
    assert np.array_equal(rec.keys, keys[order])
    assert np.array_equal(rec.payloads, order.astype(np.uint64))
    assert rep.merge_out_copies > 0
    assert rep.heavy_records_removed[0] >= n // 3


def test_theory_mode_threshold():
    """test_dtsort.py:189-197"""
    from paper_2401_00710_b200 import SortConfig, dt_sort

    rng = np.random.default_rng(8)
    cfg = SortConfig(theory_mode=True, base_case_exponent=2, gamma_lo=4, gamma_hi=4, instrument=True)
    keys = rng.integers(0, 1 << 32, size=40_000, dtype=np.uint64).astype(np.uint32)
    order = np.argsort(keys, kind="stable")
    rec = _rec(keys)
    rep = dt_sort(rec, cfg)
    assert np.array_equal(rec.keys, keys[order])
    assert rep.levels >= 2


@pytest.mark.parametrize("bits,level_cap", [(32, 4), (64, 8)])
def test_criterion_5_work_bound_shape(bits, level_cap):
    """test_acceptance.py:161-170"""
    from paper_2401_00710_b200 import SortConfig, dt_sort
    from harness.refgen import DistSpec, generate

    for n in (10**5, 10**6, 10**7):
        data = generate(DistSpec("uniform", float(2**bits), n, bits, 1))
        rep = dt_sort(data, SortConfig(seed=1, instrument=True))
        assert rep.levels <= level_cap, (bits, n, rep.levels)
        assert rep.moves <= 3 * rep.levels * n, (bits, n, rep.moves, rep.levels)
        assert rep.levels == predicted_levels(n, bits, SortConfig(), rep.skipped_bits), (bits, n, rep.levels)


@pytest.mark.parametrize("mu", [10, 32])
def test_criterion_6_duplicate_advantage(mu):
    """test_acceptance.py:173-192 (20 seeds instead of 100: the bound is
    per seed, and the reference asks for >= 99/100)"""
    from paper_2401_00710_b200 import SortConfig, dt_sort, plain_msd_sort
    from harness.refgen import DistSpec, generate

    n, trials = 10**6, 20
    mass_ok = moves_ok = 0
    for seed in range(trials):
        data = generate(DistSpec("uniform", float(mu), n, 32, seed))
        dt_work = data.copy()
        dt_rep = dt_sort(dt_work, SortConfig(seed=seed, instrument=True))
        plain_rep = plain_msd_sort(data, SortConfig(seed=seed, instrument=True))
        mass1 = dt_rep.level_mass[1] if len(dt_rep.level_mass) > 1 else 0
        mass_ok += mass1 <= 0.05 * n
        moves_ok += dt_rep.moves <= 0.6 * plain_rep.moves
    assert mass_ok == trials and moves_ok == trials, (mass_ok, moves_ok)


def _gold_cases():
    import json
    import pathlib

    g = pathlib.Path(__file__).resolve().parent / "golden" / "sort_golden.json"
    return json.loads(g.read_text())["cases"]


@pytest.mark.parametrize("case", _gold_cases(), ids=[c["name"] for c in _gold_cases()])
def test_gpu_instrument_equals_reference_report(case):
    """Through the public sorters on the GPU: keys/payloads equal the
    reference's bytes and the InstrumentReport equals the reference's
    (tests/golden/sort_golden.json, written from the reference package)."""
    import cases

    from paper_2401_00710_b200 import RecordArray, SortConfig, dt_sort, plain_msd_sort

    keys, pays = cases.make_input(case)
    for mode, fn in (("dt", dt_sort), ("plain", plain_msd_sort)):
        rec = RecordArray(keys.copy(), None if pays is None else pays.copy())
        rep = fn(rec, SortConfig(instrument=True, **case["cfg"]))
        assert cases.sha(rec.keys, rec.payloads) == case[f"{mode}_sha"], mode
        want = case[f"{mode}_report"]
        got = {k: getattr(rep, k) for k in want}
        assert got == want, mode
