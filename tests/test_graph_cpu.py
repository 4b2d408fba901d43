"""C5 workload pieces on the CPU: the R-MAT generator's host twin (the GPU
kernel k_gen_rmat is checked against it in test_gpu_graph.py), and the
oracle's stable sort of a small R-MAT edge list against numpy."""
import numpy as np

from oracle import oracle as ora
from paper_2401_00710_b200 import gen


def test_rmat_thresholds_follow_probabilities():
    t0, t1, t2 = gen.rmat_thresholds()
    assert (t0, t1, t2) == (int(0.57 * 2**32), int(0.76 * 2**32), int(0.95 * 2**32))
    assert gen.rmat_thresholds((0.25, 0.25, 0.25, 0.25)) == (2**30, 2**31, 3 * 2**30)


def test_rmat_host_deterministic_and_sliceable():
    d, s = gen.rmat_edges_host(5000, 20, seed=3)
    d2, s2 = gen.rmat_edges_host(5000, 20, seed=3)
    assert np.array_equal(d, d2) and np.array_equal(s, s2)
    # a slice at edge_base b equals the tail of the full list (global edge index)
    d3, s3 = gen.rmat_edges_host(1000, 20, seed=3, edge_base=4000)
    assert np.array_equal(d3, d[4000:]) and np.array_equal(s3, s[4000:])
    assert d.max() < 2**20 and s.max() < 2**20
    d4, _ = gen.rmat_edges_host(5000, 20, seed=4)
    assert not np.array_equal(d, d4)


def test_rmat_host_bit_probabilities():
    # dst bit = 1 with probability b + d = 0.24, src bit with c + d = 0.24
    d, s = gen.rmat_edges_host(200_000, 16, seed=0)
    for arr in (d, s):
        bits = np.unpackbits(arr.astype(">u4").view(np.uint8)).reshape(-1, 32)[:, 16:]
        p = bits.mean(axis=0)
        assert np.all(np.abs(p - 0.24) < 0.01), p


def test_rmat_edges_sorted_by_dst_with_oracle():
    d, s = gen.rmat_edges_host(300_000, 18, seed=1)
    k, v = ora.dt_sort(d, s)
    order = np.argsort(d, kind="stable")
    assert np.array_equal(k, d[order]) and np.array_equal(v, s[order])
    row_ptr = np.concatenate(([0], np.cumsum(np.bincount(k, minlength=2**18))))
    assert row_ptr[-1] == len(k)
