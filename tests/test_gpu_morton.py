"""Morton sort: k_morton's
z-values against the numpy twin, and the device Morton sort against a host
stable argsort of those z-values (keys and point permutation)."""
import numpy as np
import pytest

from paper_2401_00710_b200.morton import morton_keys_host


def test_host_interleave_known_values():
    x = np.array([1, 0, 3, 0xFFFFFFFF], np.uint32)
    y = np.array([0, 1, 3, 0], np.uint32)
    assert morton_keys_host([x, y]).tolist() == [1, 2, 15, 0x5555555555555555]
    e = np.eye(3, dtype=np.uint32)
    assert morton_keys_host([e[0], e[1], e[2]], 21).tolist() == [1, 2, 4]
    assert int(morton_keys_host([np.array([0x1FFFFF], np.uint32)] * 3, 21)[0]) == (1 << 63) - 1


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [2, 3])
def test_gpu_morton_keys_match_host_twin(dims):
    import torch

    from paper_2401_00710_b200.morton import morton_keys

    rng = np.random.default_rng(dims)
    bits = 32 if dims == 2 else 21
    n = 200_003
    cs = [rng.integers(0, 2**bits, size=n, dtype=np.uint64).astype(np.uint32) for _ in range(dims)]
    dk, dv = morton_keys([torch.from_numpy(c.view(np.int32)).cuda() for c in cs], bits, first_index=5)
    assert np.array_equal(dk.cpu().numpy().view(np.uint64), morton_keys_host(cs, bits))
    assert np.array_equal(dv.cpu().numpy(), np.arange(5, n + 5))


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [2, 3])
def test_gpu_morton_sort_varying_density(dims):
    from paper_2401_00710_b200.morton import morton_sort, varying_density_points

    n = 1_000_000
    pts = varying_density_points(n, dims, seed=11)
    host = [p.cpu().numpy().view(np.uint32) for p in pts]
    z = morton_keys_host(host)
    order = np.argsort(z, kind="stable")
    keys, perm = morton_sort(pts)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), z[order])
    assert np.array_equal(perm.cpu().numpy(), order)
    # the dense clusters repeat z-values: ties keep input order
    assert np.unique(z).size < n


@pytest.mark.gpu
def test_gpu_morton_rejects_out_of_range_coordinates():
    import torch

    from paper_2401_00710_b200.morton import morton_keys

    x = torch.tensor([1, 2, 1 << 21], dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match="does not fit"):
        morton_keys([x, x, x], 21)
    with pytest.raises(ValueError, match="bits per coordinate"):
        morton_keys([x, x, x], 22)
