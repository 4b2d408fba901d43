"""The GPU pipeline's OWN structure (``rep.gpu`` / ``sort_device(report=True)``),
not the host replay: these tests fail if the device sampler
(k_sample_plan: sampler.py:121-174 sample, :177-189 detect_heavy) or the
root overflow skip (sampler.py:192-207 plan_overflow) stop firing, even
though the output would stay correct (VERDICT r1 "what's weak" 1)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev_sort(keys, vals, mode=0):
    import torch

    from paper_2401_00710_b200 import SortConfig
    from paper_2401_00710_b200.dtsort import sort_device

    dt = {4: torch.int32, 8: torch.int64}
    k = torch.from_numpy(keys.view(np.int32 if keys.itemsize == 4 else np.int64).copy()).cuda()
    v = torch.from_numpy(vals.view(np.int32 if vals.itemsize == 4 else np.int64).copy()).cuda()
    assert k.dtype == dt[keys.itemsize]
    rep = sort_device(k, v, SortConfig(seed=0), mode, report=True)
    torch.cuda.synchronize()
    kk = k.cpu().numpy().view(keys.dtype)
    vv = v.cpu().numpy().view(vals.dtype)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(kk, keys[order]) and np.array_equal(vv, vals[order])
    return rep


def test_planted_heavy_key_gets_its_own_bucket_on_the_device():
    rng = np.random.default_rng(7)
    n = 2_000_000
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    keys[: n // 3] = 0x1234
    rng.shuffle(keys)
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint32))
    assert rep.kernel_launches["sample"] >= 1 and rep.kernel_records["sample"] >= 1
    # every record of the planted key leaves the recursion at level 0
    assert rep.heavy_records_removed[0] >= n // 3
    # ... so level 1 holds at most the light records
    assert rep.level_mass[1] <= n - n // 3


def test_heavy_detection_is_off_in_plain_mode():
    rng = np.random.default_rng(7)
    n = 2_000_000
    keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    keys[: n // 3] = 0x1234
    rng.shuffle(keys)
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint32), mode=1)
    assert rep.kernel_launches["sample"] == 0
    assert sum(rep.heavy_records_removed) == 0 and rep.skipped_bits == 0


def test_root_overflow_skip_on_small_keys_with_outliers():
    """Keys < 2^20 plus three outliers: the root skips the empty leading bits
    and routes the outliers to the overflow bucket (plan_overflow)."""
    rng = np.random.default_rng(5)
    n = 2_000_000
    keys = rng.integers(0, 1 << 20, size=n, dtype=np.uint32)
    keys[rng.integers(0, n, size=3)] = np.array([1 << 30, (1 << 32) - 1, 1 << 28], np.uint32)
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint32))
    assert rep.skipped_bits >= 8
    # two distribution levels cover the 20 remaining bits (9 + local sort)
    assert rep.levels <= 2


def test_u64_exponential_root_skip():
    rng = np.random.default_rng(9)
    n = 2_000_000
    keys = np.floor(rng.exponential(1e5, size=n)).astype(np.uint64)
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint64))
    # keys < 2^24 w.h.p.: at least 32 of the 64 bits are skipped at the root
    assert rep.skipped_bits >= 32


def test_zipf_heavy_mass_found_on_the_device():
    from paper_2401_00710_b200 import gen

    n = 4_000_000
    keys = gen.zipf_keys_host(1.5, n, 10**9, 3)
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint32))
    # rank 1 alone holds 1/zeta(1.5) ~ 38 % of the records
    assert rep.heavy_records_removed[0] >= 0.3 * n


def test_all_equal_keys_leave_in_one_pass():
    n = 1_000_000
    keys = np.full(n, 42, np.uint32)
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint32))
    assert rep.heavy_records_removed[0] == n and rep.levels == 1


def test_u64_records_reach_the_base_case_after_one_pass_at_3800_per_bucket():
    """8-byte columns: the base case takes spans of 4608 records (one SMEM span
    buffer), so 512 buckets of ~3800 u64/u64 records end after ONE distribution
    pass (with the former 2560-record spans every bucket went down a level)."""
    rng = np.random.default_rng(11)
    n = 512 * 3800
    keys = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint64))
    assert rep.levels == 1
    assert rep.records_distributed == n and rep.base_case_records == n


def test_small_duplicate_rich_segments_take_wide_digits():
    """A segment just above the base case is split on at least 6 bits per
    level: 40 000 records over 64 distinct values in the low 12 bits leave
    after one pass, not after a 2-bit-per-level tail of levels."""
    rng = np.random.default_rng(12)
    n = 40_000
    vals64 = rng.integers(0, 4096, size=64).astype(np.uint32)
    keys = vals64[rng.integers(0, 64, size=n)]
    rep = _dev_sort(keys, np.arange(n, dtype=np.uint32))
    assert rep.levels <= 2
