"""Dovetail merge on the B200 (drop-in for dtmerge.py:132-238).

Same signature, validation order and messages as the reference; the zone
is merged in place.  On the GPU (include/dts.h dts_merge) the heavy-key
insertion points come from a binary-search kernel, and the zone is permuted
out of place in one pass into a workspace and copied back (3-4 launches,
one read-back); ``MergeStats`` are the reference's piece-loop counts
(direct copy or two-flip shift, dtmerge.py:81-105), computed on the host
from the insertion points, so they equal the reference's exactly.  The sort path itself does not call this: the scatter
places heavy runs at their merged positions directly.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import Column, np_of, pick_device, torch_mod
from .core import _is_torch, _np_dtype

__all__ = ["MergeStats", "dt_merge"]


@dataclass(frozen=True)
class MergeStats:
    """Write counts of one merge (dtmerge.py:29-36)."""

    out_copies: int = 0
    in_array_moves: int = 0
    restore_copies: int = 0


def _len(x) -> int:
    return int(x.shape[0])


def _width(x) -> int:
    return int(x.element_size() if _is_torch(x) else np.asarray(x).itemsize)


def _addr(x) -> int:
    """Address of a scratch array (never dereferenced by dts_merge; non-null
    tells it scratch payloads were supplied)."""
    if _is_torch(x):
        return int(x.data_ptr()) or 1
    return int(np.asarray(x).ctypes.data) or 1


def dt_merge(
    zone_keys,
    zone_payloads,
    light_len: int,
    heavy_keys,
    heavy_lens,
    scratch_keys,
    scratch_payloads=None,
    validate: bool = True,
) -> MergeStats:
    """Merge a zone ``[light | heavy_1 | ... | heavy_m]`` in place."""
    hk = np.ascontiguousarray(np_of(heavy_keys))
    hl = np.ascontiguousarray(np.asarray(np_of(heavy_lens) if _is_torch(heavy_lens) else heavy_lens,
                                         dtype=np.int64)).reshape(-1)
    m = int(hk.shape[0])
    if hl.shape[0] != m:
        raise ValueError("heavy_keys and heavy_lens must have equal length")
    light_len = int(light_len)
    total = _len(zone_keys)
    heavy_total = int(hl.sum())
    small_side = min(light_len, heavy_total)
    if _len(scratch_keys) < small_side:
        raise ValueError(f"scratch holds {_len(scratch_keys)} records, need {small_side}")
    has_pay = zone_payloads is not None
    if has_pay and (scratch_payloads is None or _len(scratch_payloads) < small_side):
        raise ValueError("scratch payloads too small")
    kdt = _np_dtype(zone_keys)
    if kdt not in (np.dtype(np.uint32), np.dtype(np.uint64)):
        raise ValueError(f"keys must be uint32 or uint64, got {zone_keys.dtype}")
    hk = hk.astype(kdt, copy=False)
    if not validate and (np.any(hl < 0) or light_len + heavy_total != total):
        raise ValueError("light_len plus heavy run lengths must tile the zone")
    if not validate and (m == 0 or total == 0):
        return MergeStats()
    torch = torch_mod()
    device = pick_device(zone_keys, zone_payloads, scratch_keys)
    with torch.cuda.device(device):
        zk = Column(zone_keys, device, None)
        zv = Column(zone_payloads, device, None) if has_pay else None
        kb = zk.width
        vb = 0 if zv is None else zv.width
        # scratch is validated (the reference's contract) but not written:
        # the GPU permutes the zone through a workspace
        if _width(scratch_keys) != kb or (has_pay and _width(scratch_payloads) != vb):
            raise ValueError("scratch dtype must match the zone's")
        stats = (ctypes.c_uint64 * 3)()
        stream = torch.cuda.current_stream(device).cuda_stream
        L = _lib.lib()
        wsb = int(L.dts_merge_workspace_bytes(total, m, kb, vb))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=device)
        rc = L.dts_merge(
            ctypes.c_void_p(zk.ptr()),
            ctypes.c_void_p(0 if zv is None else zv.ptr()),
            total, light_len,
            ctypes.c_void_p(hk.ctypes.data if m else 0),
            hl.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            m,
            ctypes.c_void_p(_addr(scratch_keys)),
            ctypes.c_void_p(_addr(scratch_payloads) if has_pay else 0),
            _len(scratch_keys), kb, vb, int(bool(validate)), ctypes.c_void_p(ws.data_ptr()), wsb, stats,
            ctypes.c_void_p(stream),
        )
        _lib.check(rc)
        zk.writeback()
        if zv is not None:
            zv.writeback()
    return MergeStats(int(stats[0]), int(stats[1]), int(stats[2]))
