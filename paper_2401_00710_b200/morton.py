"""Morton sort on the GPU — the paper's second application
(/root/reference/PAPER.md:1149-1165): the z-value of a d-dimensional point
interleaves the bits of its coordinates; sorting the z-values orders the
points along a locality-preserving curve.

``morton_keys`` builds the 64-bit z-values (and point indices) with the
libdts kernel ``k_morton`` (include/dts.h ``dts_morton_keys``);
``morton_sort`` sorts them stably with ``dts_sort`` and returns the sorted
z-values and the point permutation.  Bit order: coordinate 0 takes the
lowest bit of every group (bit d*i + c of the key = bit i of coordinate c).

``varying_density_points`` is a seeded synthetic point set of clusters with
very different spreads — the shape of the paper's Varden datasets (points
of varying density), generated on the device.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._device import torch_mod
from .core import SortConfig

__all__ = ["morton_keys", "morton_sort", "morton_keys_host", "varying_density_points"]


def _u32(t):
    torch = torch_mod()
    if t.dtype not in (torch.int32, torch.uint32):
        raise ValueError("coordinates must be 32-bit integer CUDA tensors")
    if not t.is_cuda:
        raise ValueError("coordinates must be CUDA tensors")
    return t.contiguous()


def morton_keys(coords, bits: int | None = None, with_index: bool = True, first_index: int = 0):
    """(keys int64 CUDA tensor holding uint64 z-values, indices or None).

    ``coords`` = [x, y] or [x, y, z]: uint32 bit patterns (int32/uint32 CUDA
    tensors of equal length).  ``bits`` per coordinate defaults to 32 (2-D)
    or 21 (3-D); a coordinate at or above 2^bits raises ValueError."""
    torch = torch_mod()
    d = len(coords)
    if d not in (2, 3):
        raise ValueError("dims must be 2 or 3")
    cs = [_u32(c) for c in coords]
    n = int(cs[0].numel())
    if any(int(c.numel()) != n for c in cs):
        raise ValueError("coordinate arrays must have equal length")
    bits = bits or (32 if d == 2 else 21)
    dev = cs[0].device
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    vals = torch.empty(n, dtype=torch.int64, device=dev) if with_index else None
    ws = torch.empty(16, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = _lib.lib().dts_morton_keys(
            ctypes.c_void_p(cs[0].data_ptr()), ctypes.c_void_p(cs[1].data_ptr()),
            ctypes.c_void_p(cs[2].data_ptr() if d == 3 else 0), n, d, int(bits),
            ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(0 if vals is None else vals.data_ptr()),
            int(first_index), ctypes.c_void_p(ws.data_ptr()), 16, ctypes.c_void_p(stream))
    _lib.check(rc)
    return keys, vals


def morton_sort(coords, bits: int | None = None, cfg: SortConfig | None = None):
    """(sorted z-values, point permutation): points in Morton order, ties
    (equal z-values) in input order."""
    from .dtsort import sort_device

    keys, idx = morton_keys(coords, bits)
    sort_device(keys, idx, cfg or SortConfig(), _lib.MODE_DT)
    return keys, idx


def morton_keys_host(coords, bits: int | None = None) -> np.ndarray:
    """numpy twin of k_morton (tests): uint64 z-values."""
    d = len(coords)
    bits = bits or (32 if d == 2 else 21)
    out = np.zeros(np.asarray(coords[0]).shape[0], np.uint64)
    for c, arr in enumerate(coords):
        a = np.asarray(arr).astype(np.uint64)
        for i in range(bits):
            out |= ((a >> np.uint64(i)) & np.uint64(1)) << np.uint64(d * i + c)
    return out


def varying_density_points(n: int, dims: int = 2, bits: int | None = None, clusters: int = 64, seed: int = 0,
                           device=None):
    """n points (list of dims int32 CUDA tensors of uint32 coordinates < 2^bits)
    in `clusters` Gaussian clusters whose spreads range over many orders of
    magnitude (log-uniform from 1 to 2^(bits-2)), so local densities differ
    wildly and Morton keys repeat inside the densest clusters."""
    torch = torch_mod()
    bits = bits or (32 if dims == 2 else 21)
    device = device or torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    top = float(2**bits - 1)
    centers = torch.rand(clusters, dims, generator=g, device=device, dtype=torch.float64) * top
    spread = torch.exp2(torch.rand(clusters, generator=g, device=device, dtype=torch.float64) * (bits - 2))
    which = torch.randint(0, clusters, (n,), generator=g, device=device)
    out = []
    for c in range(dims):
        x = centers[which, c] + torch.randn(n, generator=g, device=device, dtype=torch.float64) * spread[which]
        x = torch.clamp(torch.round(x), 0.0, top).to(torch.int64)
        out.append(x.to(torch.int32) if bits < 32 else (x - (x >= 2**31).to(torch.int64) * 2**32).to(torch.int32))
    return out
