"""Host-side API contract (no GPU needed): validation messages and types
mirror the reference (core.py:50-59, :132-146; dtsort.py:82-83;
dtmerge.py:149-163; parallel.py:25-38)."""
import numpy as np
import pytest

from paper_2401_00710_b200 import (
    InstrumentReport, RecordArray, SortConfig, ceil_log2, dt_merge, dt_sort, gamma_for,
    num_workers, plain_msd_sort, rng_stream, set_num_workers,
)


def test_record_array_accepts_widths_and_torch():
    import torch

    for dt, width in ((np.uint32, 32), (np.uint64, 64)):
        rec = RecordArray(np.arange(5, dtype=dt))
        assert rec.key_width == width and len(rec) == 5 and rec.payloads is None
    rec = RecordArray(torch.arange(4, dtype=torch.int64).to(torch.uint64),
                      torch.zeros(4, dtype=torch.uint32))
    assert rec.key_width == 64 and rec.payload_width == 32


def test_record_array_rejects_bad_inputs():
    with pytest.raises(ValueError, match="keys must be uint32 or uint64, got int32"):
        RecordArray(np.arange(4, dtype=np.int32))
    with pytest.raises(ValueError, match="uint32 or uint64"):
        RecordArray(np.arange(4, dtype=np.float64))
    with pytest.raises(ValueError, match="one-dimensional"):
        RecordArray(np.zeros((2, 2), dtype=np.uint32))
    with pytest.raises(ValueError, match="payloads must be uint32 or uint64"):
        RecordArray(np.arange(4, dtype=np.uint32), np.arange(4, dtype=np.int64))
    with pytest.raises(ValueError, match="payloads must match keys in length"):
        RecordArray(np.arange(4, dtype=np.uint32), np.arange(3, dtype=np.uint64))


def test_record_array_copy_and_bytes():
    rec = RecordArray(np.arange(3, dtype=np.uint32), np.arange(3, dtype=np.uint64))
    dup = rec.copy()
    dup.keys[0] = 99
    assert rec.keys[0] == 0
    assert rec.tobytes() == rec.keys.tobytes() + rec.payloads.tobytes()


def test_sort_config_validation():
    cfg = SortConfig()
    assert cfg.gamma_lo == 8 and cfg.gamma_hi == 12 and cfg.effective_theta(8) == 1 << 14
    for kw, msg in [
        (dict(gamma_lo=0), "gamma_lo"),
        (dict(gamma_lo=9, gamma_hi=8), "gamma_lo"),
        (dict(gamma_hi=17), "gamma_hi"),
        (dict(seed=2**64), "seed"),
        (dict(parallel_grain=0), "parallel_grain"),
        (dict(base_case_threshold=100), "base_case_threshold"),
        (dict(theory_mode=True, base_case_exponent=0), "base_case_exponent"),
    ]:
        with pytest.raises(ValueError, match=msg):
            SortConfig(**kw)
    assert SortConfig(theory_mode=True, base_case_exponent=2).effective_theta(10) == 1 << 20


def test_helpers_match_reference_values():
    for n in range(1, 3000):
        k = ceil_log2(n)
        assert 2**k >= n and (k == 1 or 2 ** (k - 1) < n)
    cfg = SortConfig()
    assert gamma_for(10**9, 32, cfg) == 9
    assert gamma_for(10**6, 32, cfg) == 8
    assert gamma_for(2**40, 4, cfg) == 4
    a = rng_stream(7, 11).integers(0, 2**63, size=8)
    b = rng_stream(7, 11).integers(0, 2**63, size=8)
    assert np.array_equal(a, b)
    with pytest.raises(ValueError):
        rng_stream(-1, 0)


def test_type_error_and_empty_input_without_gpu():
    with pytest.raises(TypeError, match="records must be a RecordArray"):
        dt_sort(np.arange(5, dtype=np.uint32))
    with pytest.raises(TypeError):
        plain_msd_sort([1, 2, 3])
    rec = RecordArray(np.empty(0, np.uint32), np.empty(0, np.uint64))
    assert dt_sort(rec) is None
    rep = plain_msd_sort(rec, SortConfig(instrument=True))
    assert isinstance(rep, InstrumentReport)
    assert rep.moves == 0 and rep.levels == 0 and rep.level_mass == [0]


def test_config_callables_rejected():
    rec = RecordArray(np.empty(0, np.uint32))
    with pytest.raises(NotImplementedError):
        dt_sort(rec, SortConfig(sample_rule=lambda n, g, t: 17))
    with pytest.raises(NotImplementedError):
        dt_sort(rec, SortConfig(block_policy=lambda n, b, w: 1))


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rec = RecordArray(np.arange(10, dtype=np.uint32))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        dt_sort(rec)


def test_dt_merge_host_side_validation():
    def call(keys, light_len, hk, lens, scratch=64, pays="auto"):
        keys = np.asarray(keys, np.uint32)
        p = np.arange(keys.shape[0], dtype=np.uint64) if pays == "auto" else pays
        sp = np.empty(scratch, np.uint64) if p is not None else None
        return dt_merge(keys, p, light_len, np.asarray(hk, np.uint32), lens,
                        np.empty(scratch, np.uint32), sp)

    with pytest.raises(ValueError, match="equal length"):
        call([1, 2, 9], 2, [9], [1, 1])
    with pytest.raises(ValueError, match="scratch holds"):
        call([1, 2, 3, 9, 9, 9, 9], 3, [9], [4], scratch=2)
    keys = np.array([1, 2, 9, 9], np.uint32)
    with pytest.raises(ValueError, match="scratch payloads"):
        dt_merge(keys, np.arange(4, dtype=np.uint64), 2, np.array([9], np.uint32), [2],
                 np.empty(2, np.uint32), None)


def test_worker_knob():
    set_num_workers(3)
    assert num_workers() == 3
    with pytest.raises(ValueError):
        set_num_workers(0)
    set_num_workers(None)
    assert num_workers() >= 1
