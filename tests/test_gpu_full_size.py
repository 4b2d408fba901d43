"""Parity at BASELINE.json's full sizes (10^9 records) through the O(n)
stable-sort certificate: with values = original index,
the output is THE stable sort iff
  1. keys are non-decreasing,
  2. values are a permutation of 0..n-1,
  3. values ascend inside every run of equal keys,
  4. out_keys[i] == in_keys[out_vals[i]].
This is the logic of the reference CLI's `verify` (bench.py:309-335); the
oracle is too slow for 10^9 records, so the byte comparison against it runs
at the sizes of tests/test_gpu_sort.py.  Chunked on the device so no
n-sized int64 temporaries are needed beyond the gather.

C5 (2^32 R-MAT edges, values = src, not an index) is checked through a
(dst, edge index) twin: the twin's output passes the certificate, then the
(dst, src) output must equal src_in[twin_index] record for record — the
reference's own transpose check (bench.py:339-360) at full size, through
sort_device's >= 2^32 split path (composite splitters + dts_partition)."""
import pytest

pytestmark = pytest.mark.gpu

CONFIGS = ["c2", "c3-zipf0.6", "c3-zipf1.0", "c3-zipf1.2", "c3-zipf1.5", "c4-exp1e-5", "c4-exp1e-7", "c4-bexp"]


def _u(t):
    import torch

    return t.to(torch.int64) & 0xFFFFFFFF if t.element_size() == 4 else t


@pytest.mark.parametrize("name", CONFIGS)
def test_gpu_full_size_certificate(name):
    import torch

    import bench
    from paper_2401_00710_b200 import SortConfig
    from paper_2401_00710_b200.dtsort import sort_device

    cfg = dict(bench.CONFIGS[name])
    n = cfg["n"]
    dev = torch.device("cuda", 0)
    k, v = bench.gen_device(cfg, n, 7, dev)
    k_in = k.clone()
    sort_device(k, v, SortConfig(seed=7), 0)
    torch.cuda.synchronize()
    unsigned64 = k.element_size() == 8
    CH = 1 << 27
    seen = torch.zeros(n, dtype=torch.bool, device=dev)
    for c0 in range(0, n, CH):
        c1 = min(n, c0 + CH + 1)
        kk, vv = _u(k[c0:c1]), _u(v[c0:c1])
        if unsigned64:  # compare as unsigned: flip the sign bit
            kk = kk ^ (-(2**63))
        same = kk[1:] == kk[:-1]
        assert bool((kk[1:] >= kk[:-1]).all()), f"{name}: keys not sorted near {c0}"
        assert bool((~same | (vv[1:] > vv[:-1])).all()), f"{name}: equal keys out of input order near {c0}"
        body = vv[: min(CH, n - c0)]
        assert bool(((body >= 0) & (body < n)).all()), f"{name}: value out of range near {c0}"
        seen[body] = True
        assert bool((k[c0:c0 + body.numel()] == k_in[body]).all()), f"{name}: key/value pairing broken near {c0}"
    assert bool(seen.all()), f"{name}: values are not a permutation of 0..n-1"


def test_gpu_c5_full_size_twin_certificate():
    import torch

    from paper_2401_00710_b200 import SortConfig, gen
    from paper_2401_00710_b200.certify import stable_sort_certificate
    from paper_2401_00710_b200.dtsort import sort_device, split_n

    n = 2**32
    assert n >= split_n()  # the split path is what runs
    dev = torch.device("cuda", 0)
    dk, sk = gen.rmat_edges(n, 28, 0, dev)
    del sk
    ik = dk.clone()
    iv = torch.arange(n, dtype=torch.int64, device=dev).to(torch.int32)  # u32 bit patterns 0..2^32-1
    sort_device(ik, iv, SortConfig(seed=0), 0)
    torch.cuda.synchronize()
    err = stable_sort_certificate(dk, ik, iv)
    assert err is None, f"C5 (dst, edge index) twin: {err}"
    del dk
    dk, sk = gen.rmat_edges(n, 28, 0, dev)
    sort_device(dk, sk, SortConfig(seed=0), 0)
    torch.cuda.synchronize()
    assert bool((dk == ik).all()), "C5 destinations differ from the twin's"
    del ik, dk
    _, src_in = gen.rmat_edges(n, 28, 0, dev)
    CH = 1 << 28
    for c0 in range(0, n, CH):
        idx = iv[c0:c0 + CH].to(torch.int64) & 0xFFFFFFFF
        assert bool((sk[c0:c0 + CH] == src_in[idx]).all()), f"C5 sources out of stable order near {c0}"
