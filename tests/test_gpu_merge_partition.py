"""GPU dt_merge (drop-in for dtmerge.py:132-238) against the reference's
golden outputs + MergeStats, and dts_partition against a host model."""
import json
import pathlib

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu
G = pathlib.Path(__file__).resolve().parent / "golden"


def test_gpu_dt_merge_exhaustive_grid_matches_reference():
    """All 4480 cases of test_dtmerge.py:62-82's grid."""
    from paper_2401_00710_b200 import dt_merge

    g = np.load(G / "merge_golden.npz")
    offs = g["offsets"]
    for i, (light, heavy) in enumerate(cases.merge_grid()):
        keys, pays = cases.build_zone(light, heavy)
        hk = np.array([k for k, _ in heavy], dtype=np.uint32)
        hl = np.array([ln for _, ln in heavy], dtype=np.int64)
        small = min(len(light), int(hl.sum()))
        st = dt_merge(keys, pays, len(light), hk, hl, np.empty(small, np.uint32),
                      np.empty(small, np.uint64))
        assert np.array_equal(keys, g["keys"][offs[i]:offs[i + 1]])
        assert np.array_equal(pays, g["pays"][offs[i]:offs[i + 1]])
        assert [st.out_copies, st.in_array_moves, st.restore_copies] == g["stats"][i].tolist()


def test_gpu_dt_merge_random_zones_match_reference():
    from paper_2401_00710_b200 import dt_merge

    rand = json.loads((G / "merge_random.json").read_text())
    rng = np.random.default_rng(2024)
    for trial, r in enumerate(rand):
        light_len = int(rng.integers(0, 300))
        m = int(rng.integers(0, 33))
        universe = int(rng.integers(4, 500))
        light = np.sort(rng.integers(0, universe, size=light_len) * 2)
        hk = np.sort(rng.choice(universe, size=min(m, universe), replace=False) * 2 + 1)
        heavy = [(int(k), int(rng.integers(0, 40))) for k in hk]
        dt = np.uint64 if r["wide"] else np.uint32
        keys, pays = cases.build_zone(light.tolist(), heavy, dt)
        hka = np.array([k for k, _ in heavy], dtype=dt)
        hl = np.array([ln for _, ln in heavy], dtype=np.int64)
        small = min(light_len, int(hl.sum()))
        st = dt_merge(keys, pays, light_len, hka, hl, np.empty(small, dt), np.empty(small, np.uint64))
        assert cases.sha(keys, pays) == r["out_sha"]
        assert [st.out_copies, st.in_array_moves, st.restore_copies] == r["stats"]


def test_gpu_dt_merge_errors_and_known_case():
    from paper_2401_00710_b200 import MergeStats, dt_merge

    keys = np.array([1, 3, 5, 4, 4], np.uint32)
    pays = np.arange(5, dtype=np.uint64)
    dt_merge(keys, pays, 3, np.array([4], np.uint32), [2], np.empty(2, np.uint32),
             np.empty(2, np.uint64))
    assert keys.tolist() == [1, 3, 4, 4, 5] and pays.tolist() == [0, 1, 3, 4, 2]
    keys = np.array([2, 2, 9], np.uint32)
    assert dt_merge(keys, None, 3, np.empty(0, np.uint32), [], np.empty(0, np.uint32)) == MergeStats()

    def call(keys, light_len, hk, lens, scratch=64):
        keys = np.asarray(keys, np.uint32)
        p = np.arange(keys.shape[0], dtype=np.uint64)
        return dt_merge(keys, p, light_len, np.asarray(hk, np.uint32), lens,
                        np.empty(scratch, np.uint32), np.empty(scratch, np.uint64))

    for args, msg in [
        (([1, 2, 9, 9], 3, [9], [2]), "tile"),
        (([1, 2, 9], 2, [5, 9], [-1, 2]), "nonnegative"),
        (([1, 2, 9, 5], 2, [9, 5], [1, 1]), "increasing"),
        (([2, 1, 9], 2, [9], [1]), "sorted"),
        (([1, 9, 9], 2, [9], [1]), "light run"),
        (([1, 2, 9, 8], 2, [9], [2]), "foreign"),
    ]:
        with pytest.raises(ValueError, match=msg):
            call(*args)


def test_gpu_dt_merge_large_zone():
    import torch

    from paper_2401_00710_b200 import dt_merge

    rng = np.random.default_rng(1)
    light = np.sort(rng.integers(0, 1 << 20, size=3_000_000).astype(np.uint64) * 2)
    hkeys = np.sort(rng.choice(1 << 20, size=500, replace=False).astype(np.uint64) * 2 + 1)
    lens = rng.integers(0, 5000, size=500)
    keys, pays = cases.build_zone(light, list(zip(hkeys.tolist(), lens.tolist())), np.uint64)
    order = np.argsort(keys, kind="stable")
    dk = torch.from_numpy(keys).cuda()
    dp = torch.from_numpy(pays).cuda()
    small = min(light.shape[0], int(lens.sum()))
    sk = torch.empty(small, dtype=torch.uint64, device="cuda")
    sp = torch.empty(small, dtype=torch.uint64, device="cuda")
    dt_merge(dk, dp, light.shape[0], hkeys, lens, sk, sp)
    assert np.array_equal(dk.cpu().numpy(), keys[order])
    assert np.array_equal(dp.cpu().numpy(), pays[order])


@pytest.mark.parametrize("kb,vb", [(4, 4), (8, 8), (4, 0)])
@pytest.mark.parametrize("G_", [1, 2, 3, 8, 17, 64, 1024])
def test_gpu_partition_matches_host_model(kb, vb, G_):
    """G <= 16: the prefix-table splitter router; G >= 17: the binary-search
    router; 1024 = the largest G dts_partition accepts."""
    import torch

    from paper_2401_00710_b200.distributed import CudaOps, choose_splitters

    rng = np.random.default_rng(G_ * 10 + kb)
    n = 500_000
    kdt = np.uint32 if kb == 4 else np.uint64
    hi_key = 1000 if G_ <= 8 else (1 << 30)
    keys = rng.integers(0, hi_key, size=n).astype(kdt)
    if G_ > 8:
        keys[rng.random(n) < 0.2] = 777  # splitters inside one key's run
    gbase = 12345
    gidx = np.arange(n, dtype=np.uint64) + np.uint64(gbase)
    samp = rng.integers(0, n, size=max(4096, 8 * G_))
    spk, spi = choose_splitters(keys[samp], gidx[samp], G_)
    # dest = #splitters strictly below (key, global index), lexicographic
    lo = np.searchsorted(spk, keys, side="left").astype(np.int64)
    hi = np.searchsorted(spk, keys, side="right").astype(np.int64)
    dest = lo.copy()
    for i in np.nonzero(hi > lo)[0]:
        dest[i] += int(np.count_nonzero(spi[lo[i]:hi[i]] < gidx[i]))
    order = np.argsort(dest, kind="stable")
    vals = None if vb == 0 else np.arange(n, dtype=np.uint32 if vb == 4 else np.uint64)
    tk = torch.from_numpy(keys.view(np.int32 if kb == 4 else np.int64).copy()).cuda()
    tv = None if vals is None else torch.from_numpy(vals.view(np.int32 if vb == 4 else np.int64).copy()).cuda()
    ok, ov, counts = CudaOps().partition(tk, tv, gbase, spk, spi)
    assert counts == np.bincount(dest, minlength=G_).tolist()
    assert np.array_equal(ok.cpu().numpy().view(kdt), keys[order])
    if vals is not None:
        assert np.array_equal(ov.cpu().numpy().view(vals.dtype), vals[order])
