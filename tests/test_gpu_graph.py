"""GPU: the C5 graph-transpose path — k_gen_rmat against its host twin, the
CSR offsets kernel against numpy (bincount + cumsum, the reference's
bench.py:348-349), transpose() against a stable argsort, and the split path
for inputs above one dts_sort call (forced small with DTS_SPLIT_N) against
the oracle."""
import numpy as np
import pytest

from oracle import oracle as ora

pytestmark = pytest.mark.gpu


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("n,scale,base", [(1, 28, 0), (100_003, 28, 0), (65_536, 20, 12_345_678)])
def test_gen_rmat_matches_host_twin(n, scale, base):
    from paper_2401_00710_b200 import gen

    d, s = gen.rmat_edges(n, scale, seed=7, edge_base=base)
    hd, hs = gen.rmat_edges_host(n, scale, seed=7, edge_base=base)
    assert np.array_equal(_u32(d), hd) and np.array_equal(_u32(s), hs)


@pytest.mark.parametrize("case", ["dense", "sparse", "long_gaps", "empty", "one_vertex"])
def test_csr_offsets_matches_numpy(case):
    import torch

    from paper_2401_00710_b200.graph import csr_offsets

    rng = np.random.default_rng(5)
    if case == "dense":
        nv, keys = 1000, rng.integers(0, 1000, 100_000)
    elif case == "sparse":
        nv, keys = 1 << 20, rng.integers(0, 1 << 20, 5000)
    elif case == "long_gaps":
        nv, keys = 1 << 22, np.concatenate([np.full(10, 3), np.full(7, 2_000_000), np.full(3, (1 << 22) - 1)])
    elif case == "empty":
        nv, keys = 77, np.zeros(0, np.int64)
    else:
        nv, keys = 1, np.zeros(9, np.int64)
    keys = np.sort(keys).astype(np.uint32)
    want = np.concatenate(([0], np.cumsum(np.bincount(keys, minlength=nv)))).astype(np.int64)
    got = csr_offsets(torch.from_numpy(keys.view(np.int32)).cuda(), nv).cpu().numpy()
    assert np.array_equal(got, want)
    if keys.size:  # 64-bit keys too
        got8 = csr_offsets(torch.from_numpy(keys.astype(np.int64)).cuda(), nv).cpu().numpy()
        assert np.array_equal(got8, want)


def test_csr_offsets_rejects_bad_keys():
    import torch

    from paper_2401_00710_b200.graph import csr_offsets

    with pytest.raises(ValueError, match="ascending and below nverts"):
        csr_offsets(torch.tensor([3, 1], dtype=torch.int32, device="cuda"), 10)
    with pytest.raises(ValueError, match="ascending and below nverts"):
        csr_offsets(torch.tensor([1, 10], dtype=torch.int32, device="cuda"), 10)


def test_transpose_rmat_matches_stable_argsort():
    from paper_2401_00710_b200 import gen
    from paper_2401_00710_b200.graph import transpose

    scale, n = 18, 400_000
    d, s = gen.rmat_edges(n, scale, seed=2)
    row_ptr, srcs = transpose(s, d, 1 << scale)
    hd, hs = _u32(d), _u32(s)
    order = np.argsort(hd, kind="stable")
    assert np.array_equal(_u32(srcs), hs[order])
    want = np.concatenate(([0], np.cumsum(np.bincount(hd, minlength=1 << scale))))
    assert np.array_equal(row_ptr.cpu().numpy(), want)


@pytest.mark.parametrize("kb,vb", [(4, 4), (4, 0), (8, 8)])
def test_split_sort_matches_oracle(monkeypatch, kb, vb):
    """n above the per-call bound: sample splitters, dts_partition, sort the
    parts — bit-exact with the oracle (heavy keys make the parts uneven)."""
    import torch

    from paper_2401_00710_b200.dtsort import sort_device
    from paper_2401_00710_b200 import SortConfig

    monkeypatch.setenv("DTS_SPLIT_N", str(1 << 18))
    rng = np.random.default_rng(11)
    n = 700_001
    kd = np.uint32 if kb == 4 else np.uint64
    keys = rng.integers(0, 1 << 20, n).astype(kd)
    keys[rng.random(n) < 0.3] = 77  # a heavy key spanning parts
    vals = None if vb == 0 else np.arange(n, dtype=np.uint32 if vb == 4 else np.uint64)
    tk = torch.from_numpy(keys.view(np.int32 if kb == 4 else np.int64).copy()).cuda()
    tv = None if vals is None else torch.from_numpy(vals.view(np.int32 if vb == 4 else np.int64).copy()).cuda()
    rep = sort_device(tk, tv, SortConfig(), 0, report=True)
    wk, wv = ora.dt_sort(keys, vals)
    assert np.array_equal(tk.cpu().numpy().view(kd), wk)
    if vals is not None:
        assert np.array_equal(tv.cpu().numpy().view(vals.dtype), wv)
    assert rep.level_mass[0] == n and rep.gpu_launches > 6


def test_c5_shape_small_matches_oracle():
    """C5 at 2^22 edges / 2^20 vertices through the bench generator."""
    import torch

    from paper_2401_00710_b200 import gen, RecordArray, dt_sort

    d, s = gen.rmat_edges(1 << 22, 20, seed=0)
    hd, hs = ora.dt_sort(_u32(d).copy(), _u32(s).copy())
    dt_sort(RecordArray(d.view(torch.uint32), s.view(torch.uint32)))
    assert np.array_equal(_u32(d), hd) and np.array_equal(_u32(s), hs)
