"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every symbol include/dts.h declares (no compute calls here)."""
import pathlib
import re
import subprocess

import pytest

from paper_2401_00710_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "dts.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dts_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ("dts_sort", "dts_merge", "dts_partition", "dts_workspace_bytes", "dts_last_error",
              "dts_abi_version", "dts_build_arch"):
        assert s in syms


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    for s in header_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    for s in header_symbols():
        assert re.search(rf"\bT {s}\b", out), s
    assert {name for name, _, _ in _lib.SIGNATURES} == set(header_symbols())


def test_abi_version_arch_and_workspace():
    L = _lib.lib()
    assert L.dts_abi_version() == 2  # 2: dts_merge takes a workspace
    assert L.dts_build_arch() == 100
    n = 10**6
    ws = L.dts_workspace_bytes(n, 4, 4)
    assert ws >= n * 8
    assert L.dts_workspace_bytes(n, 8, 8) >= n * 16
    assert L.dts_workspace_bytes(n, 3, 4) == 0  # invalid width


def test_cubin_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_invalid_arguments_fail_before_touching_the_device():
    import ctypes

    L = _lib.lib()
    cfg = _lib.DtsConfig()
    cfg.gamma_lo, cfg.gamma_hi = 8, 12
    rc = L.dts_sort(None, None, 10, 3, 4, None, 0, ctypes.byref(cfg), None, None)
    assert rc == -1 and b"key_bytes" in L.dts_last_error()
    rc = L.dts_sort(None, None, 0, 4, 4, None, 0, ctypes.byref(cfg), None, None)
    assert rc == 0  # n == 0 is a no-op
    cfg.gamma_lo = 0
    rc = L.dts_sort(None, None, 10, 4, 4, None, 0, ctypes.byref(cfg), None, None)
    assert rc == -1 and b"NULL" in L.dts_last_error()


def test_oversized_call_is_rejected_before_touching_the_device():
    import ctypes

    L = _lib.lib()
    cfg = _lib.DtsConfig()
    cfg.gamma_lo, cfg.gamma_hi = 8, 12
    dummy = ctypes.c_void_p(16)
    rc = L.dts_sort(dummy, None, 1 << 32, 4, 0, None, 0, ctypes.byref(cfg), None, None)
    assert rc == -1 and b"2^32" in L.dts_last_error()


def test_partition_rejects_more_splitters_than_its_tables_hold():
    """G <= 1024: the splitter / bucket tables of the partition scatter live in
    shared memory (ScatterTile HKC = NBC = 1024)."""
    import ctypes

    import numpy as np

    L = _lib.lib()
    sk = np.zeros(1024, np.uint32)
    si = np.zeros(1024, np.uint64)
    counts = np.zeros(1025, np.uint64)
    P64 = ctypes.POINTER(ctypes.c_uint64)
    rc = L.dts_partition(None, None, 0, 0, ctypes.c_void_p(sk.ctypes.data), si.ctypes.data_as(P64), 1024,
                         None, None, counts.ctypes.data_as(P64), 4, 4, None, 0, None)
    assert rc == -1 and b"1023" in L.dts_last_error()
