"""ISRT dataset files — the on-disk format of the reference's harness
(/root/reference/pkg/src/dovetail/gen.py:217-278), read and written for
the GPU path.

Format (fixed by the reference, so files interoperate): a 16-byte header
``<4sBBBBQ`` = magic ``ISRT``, version 1, key bits (32|64), payload bytes
(0|4|8), a zero byte, record count; then the records packed as
(key, payload) little-endian.

This module is built around large files and device-resident sorting:

* ``read_dataset`` maps the file (``np.memmap``) and de-interleaves keys and
  payloads straight from the mapping — one copy, no whole-file ``bytes``;
* ``read_to_device`` streams the mapping through a pinned staging buffer
  into CUDA tensors in 2^24-record chunks (keys and payloads stay in their
  file widths, ready for ``dtsort.sort_device``);
* ``write_dataset`` / ``write_device`` interleave chunk by chunk into the
  file, so writing 10^9 records never materialises a second full copy.

Error messages are the reference's (tests match on them).
"""
from __future__ import annotations

import os
import struct
from typing import NamedTuple

import numpy as np

from .core import KEY_DTYPES, RecordArray

__all__ = ["Header", "read_header", "read_dataset", "read_to_device", "write_dataset", "write_device"]

_FMT = struct.Struct("<4sBBBBQ")
_MAGIC = b"ISRT"
_VERSION = 1
_CHUNK = 1 << 24


class Header(NamedTuple):
    key_bits: int
    payload_width: int  # bytes: 0, 4 or 8
    count: int

    @property
    def record_bytes(self) -> int:
        return self.key_bits // 8 + self.payload_width

    def dtype(self) -> np.dtype:
        kb = self.key_bits // 8
        if self.payload_width == 0:
            return np.dtype(f"<u{kb}")
        return np.dtype([("key", f"<u{kb}"), ("pay", f"<u{self.payload_width}")])


def read_header(path) -> Header:
    """Validated header of an ISRT file (size checked against the count)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_FMT.size)
    if len(head) < _FMT.size:
        raise ValueError("dataset file truncated before header")
    magic, version, kbits, pw, _, count = _FMT.unpack(head)
    if magic != _MAGIC:
        raise ValueError("not a dataset file (bad magic)")
    if version != _VERSION:
        raise ValueError(f"unsupported dataset version {version}")
    if kbits not in KEY_DTYPES:
        raise ValueError(f"unsupported key width {kbits}")
    if pw not in (0, 4, 8):
        raise ValueError(f"unsupported payload width {pw}")
    h = Header(kbits, pw, count)
    want = _FMT.size + count * h.record_bytes
    if size != want:
        raise ValueError(f"dataset length mismatch: expected {want} bytes, got {size}")
    return h


def _records(path, h: Header):
    if h.count == 0:
        return np.empty(0, h.dtype())
    return np.memmap(path, dtype=h.dtype(), mode="r", offset=_FMT.size, shape=(h.count,))


def read_dataset(path):
    """(RecordArray, payload_width_bytes); payloads come back as uint64 (the
    reference's RecordArray payload type)."""
    h = read_header(path)
    rec = _records(path, h)
    if h.payload_width == 0:
        return RecordArray(np.array(rec, dtype=KEY_DTYPES[h.key_bits])), 0
    keys = np.empty(h.count, KEY_DTYPES[h.key_bits])
    pays = np.empty(h.count, np.uint64)
    for c0 in range(0, h.count, _CHUNK):
        c1 = min(h.count, c0 + _CHUNK)
        keys[c0:c1] = rec["key"][c0:c1]
        pays[c0:c1] = rec["pay"][c0:c1]
    return RecordArray(keys, pays), h.payload_width


def read_to_device(path, device):
    """(keys, payloads or None, header): CUDA tensors in the file's widths
    (int32/int64 holding the unsigned bit patterns), streamed through a
    pinned buffer."""
    import torch

    h = read_header(path)
    rec = _records(path, h)
    tdt = {4: torch.int32, 8: torch.int64}
    kb = h.key_bits // 8
    keys = torch.empty(h.count, dtype=tdt[kb], device=device)
    pays = None if h.payload_width == 0 else torch.empty(h.count, dtype=tdt[h.payload_width], device=device)
    if h.count == 0:
        return keys, pays, h
    m = min(h.count, _CHUNK)
    hk = torch.empty(m, dtype=tdt[kb], pin_memory=True)
    hp = None if pays is None else torch.empty(m, dtype=pays.dtype, pin_memory=True)
    for c0 in range(0, h.count, _CHUNK):
        c1 = min(h.count, c0 + _CHUNK)
        w = c1 - c0
        torch.cuda.current_stream(device).synchronize()  # staging free again
        if pays is None:
            hk[:w].numpy()[:] = np.asarray(rec[c0:c1]).view(hk.numpy().dtype)
        else:
            hk[:w].numpy()[:] = rec["key"][c0:c1].view(hk.numpy().dtype)
            hp[:w].numpy()[:] = rec["pay"][c0:c1].view(hp.numpy().dtype)
            pays[c0:c1].copy_(hp[:w], non_blocking=True)
        keys[c0:c1].copy_(hk[:w], non_blocking=True)
    torch.cuda.current_stream(device).synchronize()
    return keys, pays, h


def _open_out(path, kbits: int, pw: int, n: int):
    fh = open(path, "wb")
    fh.write(_FMT.pack(_MAGIC, _VERSION, kbits, pw, 0, n))
    return fh


def write_dataset(path, records: RecordArray, payload_width: int | None = None) -> None:
    """Write records in the ISRT format; payload_width 0, 4 or 8 bytes
    (default: 8 with payloads, 0 without)."""
    if payload_width is None:
        payload_width = 0 if records.payloads is None else 8
    if payload_width not in (0, 4, 8):
        raise ValueError("payload_width must be 0, 4, or 8")
    if payload_width and records.payloads is None:
        raise ValueError("records carry no payloads to write")
    keys = np.asarray(records.keys)
    pays = None if payload_width == 0 else np.asarray(records.payloads)
    if payload_width == 4 and pays.size and int(pays.max()) > 0xFFFF_FFFF:
        raise ValueError("payloads do not fit in 4 bytes")
    h = Header(keys.dtype.itemsize * 8, payload_width, int(keys.shape[0]))
    with _open_out(path, h.key_bits, payload_width, h.count) as fh:
        _write_body(fh, h, lambda c0, c1: (keys[c0:c1], None if pays is None else pays[c0:c1]))


def write_device(path, keys, pays=None, payload_width: int | None = None) -> None:
    """Write CUDA tensors (unsigned bit patterns in int32/int64) as ISRT,
    copied back chunk by chunk."""
    kbits = keys.element_size() * 8
    if payload_width is None:
        payload_width = 0 if pays is None else pays.element_size()
    if payload_width not in (0, 4, 8):
        raise ValueError("payload_width must be 0, 4, or 8")
    if payload_width and pays is None:
        raise ValueError("records carry no payloads to write")
    h = Header(kbits, payload_width, int(keys.numel()))
    knp = KEY_DTYPES[kbits]

    def chunk(c0, c1):
        k = keys[c0:c1].cpu().numpy().view(knp)
        p = None
        if payload_width:
            p = pays[c0:c1].cpu().numpy().view(np.uint32 if pays.element_size() == 4 else np.uint64)
            if payload_width == 4 and p.dtype == np.uint64 and p.size and int(p.max()) > 0xFFFF_FFFF:
                raise ValueError("payloads do not fit in 4 bytes")
        return k, p

    with _open_out(path, kbits, payload_width, h.count) as fh:
        _write_body(fh, h, chunk)


def _write_body(fh, h: Header, get) -> None:
    buf = np.empty(min(max(h.count, 1), _CHUNK), h.dtype())
    for c0 in range(0, h.count, _CHUNK):
        c1 = min(h.count, c0 + _CHUNK)
        k, p = get(c0, c1)
        out = buf[: c1 - c0]
        if h.payload_width == 0:
            out[:] = k
        else:
            out["key"] = k
            out["pay"] = p
        fh.write(out.tobytes())
