"""GPU: sizes around the write-combining scatter's tile (9216 records with
4-byte columns, 5120 with 8-byte columns) and stripe (about 44 tiles)
boundaries, and around the local sort's span capacity (4608 records) —
bit-exact against the oracle."""
import numpy as np
import pytest

from oracle import oracle as ora

pytestmark = pytest.mark.gpu

T32, T64, LBS = 9216, 5120, 44
SIZES = sorted({T32 - 1, T32, T32 + 1, 2 * T32 - 1, 2 * T32 + 1, T32 * LBS - 1, T32 * LBS, T32 * LBS + 1,
                3 * T32 * LBS + 4097, T64 - 1, T64, T64 + 1, T64 * LBS + 5, 2 * T64 * LBS - 3,
                4607, 4608, 4609, 2 * 4608 + 1, 2559, 2560, 2561, 7167, 7168, 7169})


@pytest.mark.parametrize("kb,vb", [(4, 4), (8, 8), (4, 0)])
@pytest.mark.parametrize("n", SIZES)
def test_gpu_boundary_sizes(kb, vb, n):
    import torch

    from paper_2401_00710_b200 import RecordArray, dt_sort

    rng = np.random.default_rng(n + kb)
    kd = np.uint32 if kb == 4 else np.uint64
    hi = 1 << 26 if n > 100_000 else 1 << 20
    keys = rng.integers(0, hi, n).astype(kd)
    keys[rng.random(n) < 0.05] = 12345  # a heavy key
    vals = None if vb == 0 else rng.integers(0, 1 << 30, n).astype(np.uint32 if vb == 4 else np.uint64)
    wk, wv = ora.dt_sort(keys, vals)
    tk = torch.from_numpy(keys.copy()).cuda()
    tv = None if vals is None else torch.from_numpy(vals.copy()).cuda()
    dt_sort(RecordArray(tk, tv))
    assert np.array_equal(tk.cpu().numpy(), wk)
    if vals is not None:
        assert np.array_equal(tv.cpu().numpy(), wv)
