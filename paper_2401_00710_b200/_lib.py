"""ctypes binding of libdts.so (include/dts.h).

The library is the only compute path: when it is missing or no CUDA device
is present the entry points raise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import pathlib

__all__ = [
    "LIB_PATH",
    "DtsConfig",
    "DtsReport",
    "lib",
    "check",
    "K_CLASSES",
    "MODE_DT",
    "MODE_PLAIN",
]

LIB_PATH = pathlib.Path(__file__).resolve().parent / "_lib" / "libdts.so"

DTS_EINVAL = -1
DTS_ENOMEM = -2
DTS_ECUDA = -3
MODE_DT = 0
MODE_PLAIN = 1
K_CLASSES = ("sample", "histogram", "scan", "scatter", "local_sort", "copy", "bounds", "merge")
_NK = len(K_CLASSES)


class DtsConfig(ctypes.Structure):
    """Mirror of `dts_config` (SortConfig, core.py:106-151)."""

    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("gamma_lo", ctypes.c_int32),
        ("gamma_hi", ctypes.c_int32),
        ("base_case_threshold", ctypes.c_uint64),
        ("theory_mode", ctypes.c_int32),
        ("base_case_exponent", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("instrument", ctypes.c_int32),
        ("profile", ctypes.c_int32),
        ("stream_ordered", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 6),
    ]


class DtsReport(ctypes.Structure):
    """Mirror of `dts_report` (InstrumentReport, core.py:167-227)."""

    _fields_ = [
        ("moves", ctypes.c_uint64),
        ("merge_out_copies", ctypes.c_uint64),
        ("merge_in_array_moves", ctypes.c_uint64),
        ("base_case_records", ctypes.c_uint64),
        ("levels", ctypes.c_int32),
        ("skipped_bits", ctypes.c_int32),
        ("level_mass", ctypes.c_uint64 * 64),
        ("heavy_records_removed", ctypes.c_uint64 * 64),
        ("records_distributed", ctypes.c_uint64),
        ("gpu_launches", ctypes.c_uint64),
        ("kernel_ms", ctypes.c_double * _NK),
        ("kernel_launches", ctypes.c_uint64 * _NK),
        ("kernel_records", ctypes.c_uint64 * _NK),
    ]


_LIB = None

# (name, restype, argtypes) for every symbol include/dts.h declares
SIGNATURES = (
    ("dts_workspace_bytes", ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int]),
    (
        "dts_sort",
        ctypes.c_int,
        [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(DtsConfig),
            ctypes.POINTER(DtsReport), ctypes.c_void_p,
        ],
    ),
    (
        "dts_merge",
        ctypes.c_int,
        [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
            ctypes.POINTER(ctypes.c_int64), ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
            ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p,
        ],
    ),
    ("dts_merge_workspace_bytes", ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int]),
    (
        "dts_partition",
        ctypes.c_int,
        [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
            ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_size_t, ctypes.c_void_p,
        ],
    ),
    (
        "dts_gen_rmat",
        ctypes.c_int,
        [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
            ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
        ],
    ),
    ("dts_csr_workspace_bytes", ctypes.c_size_t, [ctypes.c_uint64]),
    (
        "dts_csr_offsets",
        ctypes.c_int,
        [
            ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
        ],
    ),
    (
        "dts_morton_keys",
        ctypes.c_int,
        [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
        ],
    ),
    ("dts_last_error", ctypes.c_char_p, []),
    ("dts_abi_version", ctypes.c_int, []),
    ("dts_build_arch", ctypes.c_int, []),
)


def lib() -> ctypes.CDLL:
    """Load libdts.so once (raises if it was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("DTS_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (make -C paper_2401_00710_b200/csrc). There is no CPU fallback."
        )
    handle = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = handle
    return handle


def check(rc: int) -> None:
    """Map a dts status code to the reference's exception types."""
    if rc == 0:
        return
    msg = lib().dts_last_error().decode(errors="replace")
    if rc == DTS_EINVAL:
        raise ValueError(msg)
    if rc == DTS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
