"""Device plumbing: move a column to the GPU (or use it in place) and write
the result back into the caller's object.  torch is used only for device
memory and streams."""
from __future__ import annotations

from typing import Any, Callable

import numpy as np

from .core import _is_torch


def torch_mod():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2401_00710_b200 sorts on a CUDA device (B200, sm_100a); "
            "no GPU is visible and there is no CPU fallback"
        )
    return torch


_SIGNED = {4: "int32", 8: "int64"}


def as_raw(t):
    """View a u32/u64 tensor as the same-width signed dtype (copy-safe)."""
    torch = torch_mod()
    return t.view(getattr(torch, _SIGNED[t.element_size()]))


class Column:
    """A device-resident view of one caller column with write-back."""

    def __init__(self, obj: Any, device, stream) -> None:
        torch = torch_mod()
        self.obj = obj
        self.device = device
        self._writeback: Callable[[], None] | None = None
        if _is_torch(obj):
            t = obj
        else:
            arr = obj
            if not arr.flags.writeable:
                raise ValueError("arrays must be writeable (the sort is in place)")
            if not arr.flags.c_contiguous or arr.dtype.byteorder == ">":
                raise ValueError("arrays must be C-contiguous little-endian")
            t = torch.from_numpy(arr)
        self.width = t.element_size()
        if t.is_cuda and t.is_contiguous():
            self.dev = t
            return
        raw = as_raw(t)
        dev = torch.empty(raw.shape, dtype=raw.dtype, device=device)
        dev.copy_(raw, non_blocking=raw.is_pinned() if not raw.is_cuda else True)
        self.dev = dev

        def wb() -> None:
            raw.copy_(dev, non_blocking=False)

        self._writeback = wb

    def ptr(self) -> int:
        return self.dev.data_ptr()

    def writeback(self) -> None:
        if self._writeback is not None:
            self._writeback()


def pick_device(*objs):
    torch = torch_mod()
    for o in objs:
        if o is not None and _is_torch(o) and o.is_cuda:
            return o.device
    return torch.device("cuda", torch.cuda.current_device())


def np_of(x) -> np.ndarray:
    if _is_torch(x):
        return x.detach().cpu().numpy()
    return np.asarray(x)
