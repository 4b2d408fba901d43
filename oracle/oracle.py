"""ORACLE — TEST INFRASTRUCTURE ONLY (never the product path).

ctypes wrapper of oracle/build/libdts_oracle.so, the C++ restatement of the
reference DovetailSort (/root/reference/pkg/src/dovetail; see
dovetail_oracle.cpp for the file:line map).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.

Parity is pinned: tests/test_oracle_golden.py checks this oracle against
fixtures generated from the reference itself (tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "libdts_oracle.so"


class OraConfig(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("gamma_lo", ctypes.c_int32),
        ("gamma_hi", ctypes.c_int32),
        ("base_case_threshold", ctypes.c_uint64),
        ("theory_mode", ctypes.c_int32),
        ("base_case_exponent", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("parallel_grain", ctypes.c_uint64),
    ]


class OraReport(ctypes.Structure):
    _fields_ = [
        ("moves", ctypes.c_uint64),
        ("merge_out_copies", ctypes.c_uint64),
        ("merge_in_array_moves", ctypes.c_uint64),
        ("base_case_records", ctypes.c_uint64),
        ("levels", ctypes.c_int32),
        ("skipped_bits", ctypes.c_int32),
        ("level_mass", ctypes.c_uint64 * 64),
        ("heavy_records_removed", ctypes.c_uint64 * 64),
        ("level_mass_len", ctypes.c_int32),
        ("heavy_len", ctypes.c_int32),
        ("records_distributed", ctypes.c_uint64),
    ]


_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    L = ctypes.CDLL(str(LIB_PATH))
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    L.ora_sort.argtypes = [vp, vp, u64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(OraConfig),
                           ctypes.POINTER(OraReport)]
    L.ora_dt_merge.argtypes = [vp, vp, u64, u64, vp, ctypes.POINTER(ctypes.c_int64), u64, vp, vp,
                               u64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_uint64)]
    L.ora_counting_sort.argtypes = [vp, vp, u64, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int32), u64, vp, vp,
                                    ctypes.POINTER(ctypes.c_int64)]
    L.ora_reference_sort.argtypes = [vp, vp, u64, ctypes.c_int, ctypes.c_int]
    L.ora_philox_integers.argtypes = [u64, u64, u64, u64, ctypes.POINTER(ctypes.c_uint64)]
    L.ora_max_threads.restype = ctypes.c_int
    _LIB = L
    return L


def _ptr(a):
    return ctypes.c_void_p(0 if a is None else a.ctypes.data)


def make_cfg(seed=0, gamma_lo=8, gamma_hi=12, base_case_threshold=1 << 14, theory_mode=False,
             base_case_exponent=2, mode="dt", threads=0, parallel_grain=4096) -> OraConfig:
    c = OraConfig()
    c.seed = int(seed)
    c.gamma_lo, c.gamma_hi = int(gamma_lo), int(gamma_hi)
    c.base_case_threshold = int(base_case_threshold)
    c.theory_mode = int(bool(theory_mode))
    c.base_case_exponent = int(base_case_exponent)
    c.mode = 0 if mode == "dt" else 1
    c.threads = int(threads)
    c.parallel_grain = int(parallel_grain)
    return c


def report_dict(r: OraReport) -> dict:
    return {
        "moves": int(r.moves),
        "merge_out_copies": int(r.merge_out_copies),
        "merge_in_array_moves": int(r.merge_in_array_moves),
        "levels": int(r.levels),
        "level_mass": [int(r.level_mass[i]) for i in range(r.level_mass_len)],
        "base_case_records": int(r.base_case_records),
        "heavy_records_removed": [int(r.heavy_records_removed[i]) for i in range(r.heavy_len)],
        "skipped_bits": int(r.skipped_bits),
        "records_distributed": int(r.records_distributed),
    }


def sort_inplace(keys: np.ndarray, pays: np.ndarray | None = None, mode: str = "dt",
                 report: bool = False, **cfg) -> dict | None:
    """Stable in-place sort of (keys, pays) following dt_sort / plain_msd_sort."""
    assert keys.dtype in (np.uint32, np.uint64) and keys.flags.c_contiguous
    if pays is not None:
        assert pays.dtype in (np.uint32, np.uint64) and pays.shape == keys.shape
    c = make_cfg(mode=mode, **cfg)
    rep = OraReport()
    rc = lib().ora_sort(_ptr(keys), _ptr(pays), keys.shape[0], keys.itemsize,
                        0 if pays is None else pays.itemsize, ctypes.byref(c),
                        ctypes.byref(rep) if report else None)
    assert rc == 0
    return report_dict(rep) if report else None


def dt_sort(keys: np.ndarray, pays: np.ndarray | None = None, **cfg):
    """Sorted copies of (keys, pays)."""
    k = np.ascontiguousarray(keys).copy()
    p = None if pays is None else np.ascontiguousarray(pays).copy()
    sort_inplace(k, p, "dt", **cfg)
    return k, p


def plain_msd_sort(keys: np.ndarray, pays: np.ndarray | None = None, **cfg):
    k = np.ascontiguousarray(keys).copy()
    p = None if pays is None else np.ascontiguousarray(pays).copy()
    sort_inplace(k, p, "plain", **cfg)
    return k, p


MERGE_ERRORS = {
    1: "light_len plus heavy run lengths must tile the zone",
    2: "heavy run lengths must be nonnegative",
    3: "heavy keys must be strictly increasing",
    4: "light run must be sorted",
    5: "a heavy key also appears in the light run",
    6: "heavy run contains a foreign key",
    7: "scratch holds too few records",
}


def dt_merge(zone_keys, zone_pays, light_len, heavy_keys, heavy_lens, scratch_len=None,
             validate=True):
    """In-place dt_merge on numpy arrays; returns (out, in_array, restore)."""
    hk = np.ascontiguousarray(heavy_keys, dtype=zone_keys.dtype)
    hl = np.ascontiguousarray(heavy_lens, dtype=np.int64)
    m = hk.shape[0]
    small = min(int(light_len), int(hl.sum()))
    sl = small if scratch_len is None else scratch_len
    sk = np.empty(max(sl, 1), zone_keys.dtype)
    sp = None if zone_pays is None else np.empty(max(sl, 1), zone_pays.dtype)
    stats = (ctypes.c_uint64 * 3)()
    rc = lib().ora_dt_merge(_ptr(zone_keys), _ptr(zone_pays), zone_keys.shape[0], int(light_len),
                            _ptr(hk) if m else ctypes.c_void_p(0),
                            hl.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), m, _ptr(sk),
                            _ptr(sp), sl, zone_keys.itemsize,
                            8 if zone_pays is None else zone_pays.itemsize, int(validate), stats)
    if rc:
        raise ValueError(MERGE_ERRORS.get(rc, f"error {rc}"))
    return int(stats[0]), int(stats[1]), int(stats[2])


def counting_sort(keys, pays, bids, nbuckets):
    """Stable distribution by given bucket ids; returns (out_keys, out_pays, offsets)."""
    bids = np.ascontiguousarray(bids, dtype=np.int32)
    ok = np.empty_like(keys)
    op = None if pays is None else np.empty_like(pays)
    offs = np.zeros(nbuckets + 1, np.int64)
    rc = lib().ora_counting_sort(_ptr(keys), _ptr(pays), keys.shape[0], keys.itemsize,
                                 8 if pays is None else pays.itemsize,
                                 bids.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), nbuckets,
                                 _ptr(ok), _ptr(op), offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    assert rc == 0
    return ok, op, offs


def reference_sort(keys, pays=None):
    """bench.py:95-109 restated: bottom-up stable mergesort on copies."""
    k = np.ascontiguousarray(keys).copy()
    p = None if pays is None else np.ascontiguousarray(pays).copy()
    lib().ora_reference_sort(_ptr(k), _ptr(p), k.shape[0], k.itemsize,
                             8 if p is None else p.itemsize)
    return k, p


def philox_integers(k0: int, k1: int, high: int, cnt: int) -> np.ndarray:
    out = np.empty(cnt, np.uint64)
    lib().ora_philox_integers(k0, k1, high, cnt, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return out


def max_threads() -> int:
    return int(lib().ora_max_threads())


def stable_certificate(in_keys: np.ndarray, out_keys: np.ndarray, out_vals: np.ndarray) -> bool:
    """O(n) stable-sort certificate when values are original indices
    (the reference CLI `verify`, bench.py:309-335)."""
    n = in_keys.shape[0]
    if out_keys.shape[0] != n or out_vals.shape[0] != n:
        return False
    if n == 0:
        return True
    ok = out_keys.astype(np.uint64)
    if np.any(ok[1:] < ok[:-1]):
        return False
    v = out_vals.astype(np.int64)
    if v.min() < 0 or v.max() >= n or np.bincount(v, minlength=n).max() != 1:
        return False
    eq = ok[1:] == ok[:-1]
    if np.any(v[1:][eq] <= v[:-1][eq]):
        return False
    return bool(np.array_equal(in_keys[v], out_keys))


if os.environ.get("ORACLE_BUILD_ON_IMPORT"):
    lib()
