"""The sorters: dt_sort and plain_msd_sort on the B200.

Drop-in for /root/reference/pkg/src/dovetail/dtsort.py:64-108: same names,
same in-place contract (the caller's array objects receive the result),
same return value (None, or an InstrumentReport when cfg.instrument) and
the same TypeError for non-RecordArray input.  The whole MSD pipeline runs
in libdts.so (include/dts.h `dts_sort`) on the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os

from . import _lib
from ._device import Column, pick_device, torch_mod
from .core import InstrumentReport, RecordArray, SortConfig

__all__ = ["dt_sort", "plain_msd_sort", "make_config", "workspace_bytes"]


def dt_sort(records: RecordArray, cfg: SortConfig | None = None) -> InstrumentReport | None:
    """Sort ``records`` ascending by key, stably and in place (dtsort.py:64-71)."""
    return _run(records, cfg, _lib.MODE_DT)


def plain_msd_sort(records: RecordArray, cfg: SortConfig | None = None) -> InstrumentReport | None:
    """The ablation: no sampling, no heavy or overflow buckets (dtsort.py:74-78)."""
    return _run(records, cfg, _lib.MODE_PLAIN)


def make_config(cfg: SortConfig, mode: int, profile: bool = False, stream_ordered: bool = False) -> _lib.DtsConfig:
    if cfg.sample_rule is not None or cfg.block_policy is not None:
        raise NotImplementedError(
            "SortConfig.sample_rule / block_policy are Python callables and cannot run "
            "inside the CUDA kernels; the GPU sorter uses its own sample size and block plan"
        )
    c = _lib.DtsConfig()
    c.seed = int(cfg.seed)
    c.gamma_lo = int(cfg.gamma_lo)
    c.gamma_hi = int(cfg.gamma_hi)
    c.base_case_threshold = int(cfg.base_case_threshold)
    c.theory_mode = int(bool(cfg.theory_mode))
    c.base_case_exponent = int(cfg.base_case_exponent)
    c.mode = int(mode)
    c.instrument = int(bool(cfg.instrument))
    c.profile = int(bool(profile))
    c.stream_ordered = int(bool(stream_ordered))
    return c


def workspace_bytes(n: int, key_bytes: int, val_bytes: int) -> int:
    return int(_lib.lib().dts_workspace_bytes(int(n), int(key_bytes), int(val_bytes)))


def report_from(raw: _lib.DtsReport) -> InstrumentReport:
    rep = InstrumentReport()
    rep.moves = int(raw.moves)
    rep.merge_out_copies = int(raw.merge_out_copies)
    rep.merge_in_array_moves = int(raw.merge_in_array_moves)
    rep.levels = int(raw.levels)
    rep.base_case_records = int(raw.base_case_records)
    rep.skipped_bits = int(raw.skipped_bits)
    depth = max(rep.levels + 1, 1)
    rep.level_mass = [int(raw.level_mass[d]) for d in range(depth)]
    rep.heavy_records_removed = [int(raw.heavy_records_removed[d]) for d in range(rep.levels)]
    rep.records_distributed = int(raw.records_distributed)
    rep.gpu_launches = int(raw.gpu_launches)
    rep.kernel_ms = {k: float(raw.kernel_ms[i]) for i, k in enumerate(_lib.K_CLASSES)}
    rep.kernel_launches = {k: int(raw.kernel_launches[i]) for i, k in enumerate(_lib.K_CLASSES)}
    rep.kernel_records = {k: int(raw.kernel_records[i]) for i, k in enumerate(_lib.K_CLASSES)}
    return rep


# One dts_sort call keeps 32-bit positions inside a segment; larger inputs
# are split first (DTS_SPLIT_N lowers the bound for tests).
def split_n() -> int:
    return int(os.environ.get("DTS_SPLIT_N", (1 << 32) - (1 << 16)))


def _merge_reports(reps, n: int, extra_launches: int) -> InstrumentReport:
    out = InstrumentReport()
    out.levels = max(r.levels for r in reps)
    out.skipped_bits = max(r.skipped_bits for r in reps)
    for f in ("moves", "merge_out_copies", "merge_in_array_moves", "base_case_records", "records_distributed",
              "gpu_launches"):
        setattr(out, f, sum(getattr(r, f) for r in reps))
    out.gpu_launches += extra_launches
    depth = max(len(r.level_mass) for r in reps)
    out.level_mass = [sum(r.level_mass[d] for r in reps if d < len(r.level_mass)) for d in range(depth)]
    out.level_mass[0] = n
    hd = max(len(r.heavy_records_removed) for r in reps)
    out.heavy_records_removed = [sum(r.heavy_records_removed[d] for r in reps if d < len(r.heavy_records_removed))
                                 for d in range(hd)]
    out.kernel_ms = {k: sum(r.kernel_ms[k] for r in reps) for k in reps[0].kernel_ms}
    out.kernel_launches = {k: sum(r.kernel_launches[k] for r in reps) for k in reps[0].kernel_launches}
    out.kernel_records = {k: sum(r.kernel_records[k] for r in reps) for k in reps[0].kernel_records}
    return out


def _sort_split(keys, vals, cfg: SortConfig, mode: int, profile: bool, report: bool):
    """n >= SPLIT_N on one GPU: the multi-GPU algorithm without the exchange
    (distributed.py): G-1 composite (key, index) splitters from a sample, one
    stable G-way dts_partition, then dts_sort of every part in place; parts
    are key ranges in order and keep input order, so the result is the
    stable sort."""
    from .distributed import CudaOps, choose_splitters

    n = int(keys.numel())
    SPLIT_N = split_n()
    G = max(2, -(-n // (SPLIT_N // 2)))
    ops = CudaOps(cfg, mode)
    sk, si = ops.sample(keys, 0, min(n, 4096 * G), cfg.seed)
    spk, spi = choose_splitters(sk, si, G)
    pk, pv, counts = ops.partition(keys, vals, 0, spk, spi)
    if max(counts) >= SPLIT_N:
        raise RuntimeError(f"split sort: a part of {max(counts)} records exceeds {SPLIT_N}")
    reps, off = [], 0
    for c in counts:
        if c:
            r = sort_device(pk[off:off + c], None if pv is None else pv[off:off + c], cfg, mode, profile,
                            report=report or cfg.instrument or profile)
            if r is not None:
                reps.append(r)
        off += c
    keys.copy_(pk)
    if vals is not None:
        vals.copy_(pv)
    return _merge_reports(reps, n, 6) if reps else None


def sort_device(keys, vals, cfg: SortConfig, mode: int, profile: bool = False,
                workspace=None, report: bool = False, stream_ordered: bool = False) -> InstrumentReport | None:
    """Sort contiguous CUDA tensors in place (no validation beyond widths).

    ``keys``/``vals`` are torch CUDA tensors of 4/8-byte elements (any
    integer dtype of that width; bits are treated as unsigned).  Used by the
    public sorters, the multi-GPU driver and bench.py.  ``stream_ordered``:
    return once the last kernels are enqueued (the result is complete in
    the order of the current stream; no final host synchronisation).
    """
    torch = torch_mod()
    n = int(keys.numel())
    if n >= split_n():
        return _sort_split(keys, vals, cfg, mode, profile, report)
    kb = keys.element_size()
    vb = 0 if vals is None else vals.element_size()
    c = make_config(cfg, mode, profile, stream_ordered and n < split_n())
    raw = _lib.DtsReport() if (report or cfg.instrument or profile) else None
    L = _lib.lib()
    need = int(L.dts_workspace_bytes(n, kb, vb))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=keys.device)
    stream = torch.cuda.current_stream(keys.device).cuda_stream
    rc = L.dts_sort(
        ctypes.c_void_p(keys.data_ptr()),
        ctypes.c_void_p(0 if vals is None else vals.data_ptr()),
        n, kb, vb,
        ctypes.c_void_p(workspace.data_ptr()), int(workspace.numel()),
        ctypes.byref(c),
        ctypes.byref(raw) if raw is not None else None,
        ctypes.c_void_p(stream),
    )
    _lib.check(rc)
    return report_from(raw) if raw is not None else None


def _run(records: RecordArray, cfg: SortConfig | None, mode: int) -> InstrumentReport | None:
    if not isinstance(records, RecordArray):
        raise TypeError("records must be a RecordArray")
    cfg = cfg or SortConfig()
    n = len(records)
    if n == 0:
        make_config(cfg, mode)  # same NotImplementedError contract for callables
        if cfg.instrument:
            rep = InstrumentReport()
            rep.add_mass(0, 0)
            return rep
        return None
    device = pick_device(records.keys, records.payloads)
    torch = torch_mod()
    with torch.cuda.device(device):
        kcol = Column(records.keys, device, None)
        vcol = Column(records.payloads, device, None) if records.payloads is not None else None
        trace = _trace_sort(kcol.dev, cfg, mode) if cfg.instrument and n < split_n() else None
        rep = sort_device(kcol.dev, None if vcol is None else vcol.dev, cfg, mode)
        kcol.writeback()
        if vcol is not None:
            vcol.writeback()
        torch.cuda.current_stream(device).synchronize()
    if not cfg.instrument:
        return None
    if trace is not None:
        rep = _reference_report(rep, trace, cfg, mode)
    return rep


def _host_u(t):
    """Device tensor of 4/8-byte elements -> numpy unsigned array (bit copy)."""
    torch = torch_mod()
    import numpy as np

    if t.element_size() == 4:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.view(torch.int64).cpu().numpy().view(np.uint64)


def _trace_sort(keys, cfg: SortConfig, mode: int):
    """Instrument mode: the inputs of the counter replay (replay.py) — the
    keys in input order, and the stable (keys, index) sort done by dts_sort
    on the GPU before the caller's records are sorted."""
    torch = torch_mod()
    n = int(keys.numel())
    keys_in = _host_u(keys)
    ks = keys.clone()
    idx = torch.arange(n, dtype=torch.int32 if n < 2**31 else torch.int64, device=keys.device)
    sort_device(ks, idx, SortConfig(seed=cfg.seed), mode)
    return keys_in, _host_u(ks), idx.cpu().numpy().astype("int64")


def _reference_report(gpu: InstrumentReport, trace, cfg: SortConfig, mode: int) -> InstrumentReport:
    """The reference's counters (replay.py); the GPU's own structure stays
    available as ``rep.gpu`` and its timing / launch fields are carried over."""
    from .replay import replay_report

    keys_in, ks, perm = trace
    rep = replay_report(keys_in, ks, perm, cfg, plain=mode == _lib.MODE_PLAIN)
    rep.gpu = gpu
    if gpu is not None:
        rep.records_distributed = gpu.records_distributed
        rep.gpu_launches = gpu.gpu_launches
        rep.kernel_ms = gpu.kernel_ms
        rep.kernel_launches = gpu.kernel_launches
        rep.kernel_records = gpu.kernel_records
    return rep
