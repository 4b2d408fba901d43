"""Multi-GPU key-range sort: one process per GPU, torch.distributed (NCCL
over NVLink 5 / NVSwitch) for the exchange.

No reference counterpart (the reference is single-process); this is
north-star item (6), SURVEY.md §8(e).  Every rank holds a contiguous slice
of the global input (global index = rank offset + local index).  The ranks

1. draw (key, global index) samples, all-gather them and pick G-1
   composite splitters (identical on every rank);
2. stably partition their slice into G groups by (key, index) against the
   splitters (`dts_partition`, a G-bucket distribution pass);
3. exchange group sizes and then records with all_to_all_single;
4. stably sort the received records (`dts_sort`), chunks concatenated in
   source-rank order so equal keys keep global input order.

Rank g then holds exactly slice g of the global stable sort.  Composite
splitters balance the load even when one key holds most of the records.
The device work goes through an `ops` object; tests inject a host
implementation to exercise the exchange logic on CPU with gloo.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import SortConfig

__all__ = ["CudaOps", "DistStats", "dist_sort", "choose_splitters"]

_SIGNED = {4: "int32", 8: "int64"}


@dataclass
class DistStats:
    n_local_in: int
    n_local_out: int
    send_counts: list
    recv_counts: list
    bytes_sent_remote: int
    exchange_ms: float = 0.0     # record all-to-all (keys + values), CUDA events on the caller's stream
    local_distributed: int = 0   # records the local dts_sort distributed (its D)


def choose_splitters(sample_keys: np.ndarray, sample_idx: np.ndarray, G: int):
    """G-1 splitters at the quantiles of the (key, global index) sample,
    lexicographic order; identical on every rank given the same sample."""
    order = np.lexsort((sample_idx, sample_keys))
    sk, si = sample_keys[order], sample_idx[order]
    S = sk.shape[0]
    if G <= 1 or S == 0:
        return sk[:0], si[:0].astype(np.uint64)
    pos = [min(S - 1, ((j + 1) * S) // G) for j in range(G - 1)]
    return sk[pos].copy(), si[pos].astype(np.uint64)


class CudaOps:
    """Device work of the exchange on the local CUDA device."""

    def __init__(self, cfg: SortConfig | None = None, mode: int = _lib.MODE_DT):
        self.cfg = cfg or SortConfig()
        self.mode = mode
        self._ws = None  # partition workspace, reused across calls
        self.launches = 0  # libdts kernels launched (partition + local sort)

    def sample(self, keys, gbase: int, count: int, seed: int):
        import torch

        n = keys.numel()
        if n == 0 or count == 0:
            return np.empty(0, _np_dtype(keys)), np.empty(0, np.uint64)
        g = torch.Generator(device=keys.device)
        g.manual_seed(int(seed) * 1_000_003 + gbase)
        pos = torch.randint(0, n, (count,), generator=g, device=keys.device)
        pos = torch.sort(pos).values
        ks = keys[pos].cpu().numpy().view(_np_dtype(keys))
        return ks.copy(), (pos.cpu().numpy().astype(np.uint64) + np.uint64(gbase))

    def partition(self, keys, vals, gbase: int, split_keys: np.ndarray, split_idx: np.ndarray):
        import torch

        n = keys.numel()
        kb = keys.element_size()
        vb = 0 if vals is None else vals.element_size()
        G = split_keys.shape[0] + 1
        ok = torch.empty_like(keys)
        ov = None if vals is None else torch.empty_like(vals)
        counts = np.zeros(G, np.uint64)
        L = _lib.lib()
        # the partition uses the workspace for its metadata only (count
        # matrix, scan, tile lists): far less than a sort workspace
        need = min(int(L.dts_workspace_bytes(n, kb, vb)), (32 << 20) + n * (G + 4) // 512)
        ws = self._ws
        if ws is None or ws.numel() < need or ws.device != keys.device:
            ws = self._ws = torch.empty(need, dtype=torch.uint8, device=keys.device)
        skc = np.ascontiguousarray(split_keys.astype(np.uint32 if kb == 4 else np.uint64))
        sic = np.ascontiguousarray(split_idx.astype(np.uint64))
        stream = torch.cuda.current_stream(keys.device).cuda_stream
        rc = L.dts_partition(
            ctypes.c_void_p(keys.data_ptr()),
            ctypes.c_void_p(0 if vals is None else vals.data_ptr()),
            n, int(gbase),
            ctypes.c_void_p(skc.ctypes.data if skc.size else 0),
            sic.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            G - 1,
            ctypes.c_void_p(ok.data_ptr()),
            ctypes.c_void_p(0 if ov is None else ov.data_ptr()),
            counts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            kb, vb, ctypes.c_void_p(ws.data_ptr()), int(ws.numel()), ctypes.c_void_p(stream),
        )
        _lib.check(rc)
        self.launches += 6  # histogram, 3 scan kernels, bounds, scatter
        return ok, ov, [int(c) for c in counts]

    def sort(self, keys, vals):
        from .dtsort import sort_device

        rep = sort_device(keys, vals, self.cfg, self.mode, report=True)
        self.launches += int(rep.gpu_launches)
        return rep

    def empty_like(self, t, n):
        import torch

        return torch.empty(int(n), dtype=t.dtype, device=t.device)


def _np_dtype(t):
    import torch

    return {torch.int32: np.uint32, torch.uint32: np.uint32, torch.int64: np.uint64,
            torch.uint64: np.uint64}[t.dtype]


def _comm_view(t):
    """Signed view of the same bits (NCCL/gloo dtype support)."""
    import torch

    return t.view(getattr(torch, _SIGNED[t.element_size()]))


def dist_sort(keys, vals=None, group=None, ops=None, samples_per_rank: int = 1 << 12,
              seed: int = 0):
    """Globally stable sort of the rank-ordered concatenation of every rank's
    (keys, vals).  Returns (sorted local keys, sorted local vals, DistStats)."""
    import torch
    import torch.distributed as dist

    ops = ops or CudaOps()
    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = keys.device
    n_local = int(keys.numel())
    # global index base = exclusive prefix of the slice sizes
    ns = torch.zeros(G, dtype=torch.int64, device=dev)
    mine = torch.tensor([n_local], dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(ns, mine, group=group)
    ns_h = ns.cpu().numpy()
    N = int(ns_h.sum())
    gbase = int(ns_h[:rank].sum())
    # 1. samples proportional to slice size, all-gathered
    total_s = samples_per_rank * G
    cnt = int(min(n_local, -(-total_s * n_local // max(N, 1))))
    sk, si = ops.sample(keys, gbase, cnt, seed)
    scnt = torch.zeros(G, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(scnt, torch.tensor([cnt], dtype=torch.int64, device=dev),
                                group=group)
    smax = int(scnt.max().item())
    wide = keys.element_size() == 8
    pad_k = np.zeros(smax, np.uint64)
    pad_i = np.zeros(smax, np.uint64)
    pad_k[:cnt] = sk.astype(np.uint64)
    pad_i[:cnt] = si
    buf = torch.from_numpy(np.stack([pad_k, pad_i]).view(np.int64).reshape(-1)).to(dev)
    allb = torch.empty(G * buf.numel(), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allb, buf, group=group)
    allh = allb.cpu().numpy().view(np.uint64).reshape(G, 2, smax)
    sc = scnt.cpu().numpy()
    samp_k = np.concatenate([allh[r, 0, : sc[r]] for r in range(G)])
    samp_i = np.concatenate([allh[r, 1, : sc[r]] for r in range(G)])
    if not wide:
        samp_k = samp_k.astype(np.uint32)
    spk, spi = choose_splitters(samp_k, samp_i, G)
    # 2. stable partition by (key, global index)
    pk, pv, send = ops.partition(keys, vals, gbase, spk, spi)
    # 3. exchange sizes, then records (source-rank order on receipt)
    send_t = torch.tensor(send, dtype=torch.int64, device=dev)
    recv_t = torch.empty(G, dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_t, send_t, group=group)
    recv = [int(x) for x in recv_t.cpu().tolist()]
    n_out = sum(recv)
    rk = ops.empty_like(pk, n_out)
    timed = dev.type == "cuda"
    if timed:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    dist.all_to_all_single(_comm_view(rk), _comm_view(pk), recv, send, group=group)
    rv = None
    if vals is not None:
        rv = ops.empty_like(pv, n_out)
        dist.all_to_all_single(_comm_view(rv), _comm_view(pv), recv, send, group=group)
    if timed:
        e1.record()
    # 4. local stable sort of the received range
    rep = ops.sort(rk, rv)
    rec_bytes = keys.element_size() + (0 if vals is None else vals.element_size())
    remote = sum(send) - send[rank]
    st = DistStats(n_local, n_out, send, recv, remote * rec_bytes)
    if timed:
        e1.synchronize()
        st.exchange_ms = float(e0.elapsed_time(e1))
    st.local_distributed = int(getattr(rep, "records_distributed", 0) or 0)
    return rk, rv, st
