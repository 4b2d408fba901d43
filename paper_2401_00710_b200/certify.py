"""O(n) stable-sort certificate on the device.

When the values are the original indices 0..n-1, ``out`` is THE stable sort
of ``in`` iff

1. the keys are non-decreasing,
2. the values are a permutation of 0..n-1,
3. the values ascend inside every run of equal keys,
4. ``out_keys[i] == in_keys[out_vals[i]]``.

This is the logic of the reference CLI's ``verify``
(/root/reference/pkg/src/dovetail/bench.py:304-336).  It runs on the GPU in
chunks (no n-sized int64 temporaries beyond one chunk) so it scales to the
10^9-record and 2^32-record configurations; it is a checker (tests, bench,
CLI ``verify``), never part of the sort.

``pair_checksum`` is a permutation-invariant digest of (key, value) pairs
(sum and xor of a 64-bit mix), used where the values are not indices
(C5's (dst, src) edges): equal digests before and after, plus sorted keys,
mean the output is a reordering of the input's records.
"""
from __future__ import annotations

__all__ = ["stable_sort_certificate", "pair_checksum", "keys_sorted"]

_CH = 1 << 27


def _u64(t):
    """Unsigned 64-bit order view: u32 bits widened, u64 bits sign-flipped
    (so signed int64 comparisons order them as unsigned)."""
    import torch

    if t.element_size() == 4:
        return t.to(torch.int64) & 0xFFFFFFFF
    return t ^ (-(2**63))


def keys_sorted(keys) -> bool:
    n = int(keys.numel())
    for c0 in range(0, max(n - 1, 0), _CH):
        kk = _u64(keys[c0:min(n, c0 + _CH + 1)])
        if not bool((kk[1:] >= kk[:-1]).all()):
            return False
    return True


def stable_sort_certificate(in_keys, out_keys, out_vals) -> str | None:
    """None when (out_keys, out_vals) is the stable sort of in_keys with
    index values; otherwise the first failed condition, as a message."""
    import torch

    n = int(out_keys.numel())
    if int(in_keys.numel()) != n or int(out_vals.numel()) != n:
        return "lengths differ"
    if n == 0:
        return None
    dev = out_keys.device
    seen = torch.zeros(n, dtype=torch.bool, device=dev)
    for c0 in range(0, n, _CH):
        c1 = min(n, c0 + _CH + 1)
        kk = _u64(out_keys[c0:c1])
        vv = out_vals[c0:c1].to(torch.int64)
        if out_vals.element_size() == 4:
            vv = vv & 0xFFFFFFFF
        if not bool((kk[1:] >= kk[:-1]).all()):
            return f"keys not in non-decreasing order near record {c0}"
        same = kk[1:] == kk[:-1]
        if not bool((~same | (vv[1:] > vv[:-1])).all()):
            return f"equal keys out of input order near record {c0}"
        body = vv[: min(_CH, n - c0)]
        if not bool(((body >= 0) & (body < n)).all()):
            return f"value out of range near record {c0}"
        seen[body] = True
        if not bool((out_keys[c0:c0 + body.numel()] == in_keys[body]).all()):
            return f"key/value pairing broken near record {c0}"
    if not bool(seen.all()):
        return "values are not a permutation of 0..n-1"
    return None


def pair_checksum(keys, vals) -> tuple[int, int]:
    """(sum, xor) over records of a 64-bit mix of (key, value); independent
    of record order."""
    import torch

    n = int(keys.numel())
    s = torch.zeros((), dtype=torch.int64, device=keys.device)
    x = torch.zeros((), dtype=torch.int64, device=keys.device)
    for c0 in range(0, n, _CH):
        c1 = min(n, c0 + _CH)
        k = _u64(keys[c0:c1])
        v = torch.zeros_like(k) if vals is None else _u64(vals[c0:c1])
        h = k * _s64(0x9E3779B97F4A7C15) + v * _s64(0x632BE59BD9B4E019)  # wraps mod 2^64
        h = h ^ (h >> 29)  # (arithmetic shift: still a fixed function of the pair)
        h = h * _s64(0x94D049BB133111EB)
        s = s + h.sum()
        x = x ^ _xor_reduce(h)
    return int(s.item()), int(x.item())


def _s64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


def _xor_reduce(h):
    import torch

    while h.numel() > 1:
        if h.numel() & 1:
            h = torch.cat([h, torch.zeros(1, dtype=h.dtype, device=h.device)])
        h = h[0::2] ^ h[1::2]
    return h[0] if h.numel() else torch.zeros((), dtype=torch.int64, device=h.device)
