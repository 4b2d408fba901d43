"""Graph transpose on the GPU: the C5 workload's caller and consumer.

The reference's transpose demo (bench.py:338-360) regroups edges by
destination with a stable sort and builds CSR offsets with
``np.bincount`` + ``np.cumsum``.  Here the sort is `dt_sort` on the device
and the offsets come from the libdts kernel k_csr_offsets
(include/dts.h `dts_csr_offsets`).
"""
from __future__ import annotations

import ctypes

from . import _lib
from ._device import torch_mod
from .core import SortConfig

__all__ = ["csr_offsets", "transpose"]


def csr_offsets(sorted_keys, nverts: int):
    """row_ptr (int64 CUDA tensor of nverts + 1) of ascending keys < nverts:
    row_ptr[v] = number of keys < v (bench.py:348-349)."""
    torch = torch_mod()
    dev = sorted_keys.device
    n = int(sorted_keys.numel())
    row_ptr = torch.empty(int(nverts) + 1, dtype=torch.int64, device=dev)
    L = _lib.lib()
    ws = torch.empty(int(L.dts_csr_workspace_bytes(int(nverts))), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = L.dts_csr_offsets(ctypes.c_void_p(sorted_keys.data_ptr() if n else 0), n, sorted_keys.element_size(),
                               int(nverts), ctypes.c_void_p(row_ptr.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                               int(ws.numel()), ctypes.c_void_p(stream))
    _lib.check(rc)
    return row_ptr


def transpose(src, dst, nverts: int, cfg: SortConfig | None = None):
    """In-edges of every vertex: (row_ptr, sources_by_dst).

    ``src``/``dst`` are uint32 edge endpoints (CUDA tensors, int32 or uint32
    bit patterns); the edges are stably sorted by destination (sources of one
    destination keep input order, what CSR builders need, bench.py:341-343)."""
    from .dtsort import sort_device
    from . import _lib as L

    torch = torch_mod()
    k = dst.clone()
    v = src.clone()
    sort_device(k, v, cfg or SortConfig(), L.MODE_DT)
    return csr_offsets(k, nverts), v
