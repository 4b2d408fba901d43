"""Worker-count knob (drop-in for parallel.py:20-38).

On the B200 every parallel section is a CUDA grid, so the count changes
nothing; it is validated and stored so callers of the reference keep
working, and — as in the reference — results never depend on it.
"""
from __future__ import annotations

import os

__all__ = ["num_workers", "set_num_workers"]

_DEFAULT_WORKERS = max(1, os.cpu_count() or 1)
_workers = _DEFAULT_WORKERS


def num_workers() -> int:
    return _workers


def set_num_workers(count: int | None) -> None:
    global _workers
    resolved = _DEFAULT_WORKERS if count is None else int(count)
    if resolved < 1:
        raise ValueError("worker count must be >= 1")
    _workers = resolved
