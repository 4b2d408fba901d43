"""Counter-faithful InstrumentReport.

The GPU sorter (libdts.so) picks its own digit widths, base-case size and
heavy-key sample; its output is the unique stable sort, but
its structure is not the reference's.  With ``SortConfig(instrument=True)``
the public sorters return the counters the *reference* recursion would
report on the same input: this module replays that recursion's decisions
over the GPU's results, moving no records.

Inputs: the keys in input order, the stably sorted keys ``ks`` and the
stable permutation ``perm`` (both produced by one extra dts_sort of
(keys, index) on the GPU).  Every reference subproblem is a set of key
ranges minus the heavy keys of its ancestors, i.e. a few intervals of
``ks``; bucket sizes are interval counts between binary-searched digit
boundaries, and a subproblem's records in buffer order (the order its
sample is drawn from) are its positions sorted by original index — every
stable distribution keeps input order inside a bucket.  The sample is drawn
with the reference's own Philox streams, so the counters equal the
reference's, value for value.

Followed line by line (reference pkg/src/dovetail):
  _run / _sort_rec          dtsort.py:81-108, :150-209
  _base_sort accounting     dtsort.py:127-147
  _plan_step                dtsort.py:212-241
  sample_count/draw_samples sampler.py:121-174 (_SAMPLE_TAG/_SAMPLE_CHUNK :37-38)
  detect_heavy              sampler.py:177-189
  plan_overflow             sampler.py:192-207
  counting_sort moves       counting.py:155
  _children_step            dtsort.py:244-318
  _merge_step / dt_merge    dtsort.py:321-354, dtmerge.py:58-78, :142-238
"""
from __future__ import annotations

import numpy as np

from .core import InstrumentReport, SortConfig, ceil_log2, gamma_for, rng_stream

_SAMPLE_CHUNK = 8192
_SAMPLE_TAG = 1 << 60


def _stream_id(depth: int, base_index: int, chunk: int) -> int:
    return _SAMPLE_TAG | ((depth & 0xFF) << 48) | ((base_index & 0xFF_FFFF_FFFF) << 8) | (chunk & 0xFF)


def _merge_stats(light_len: int, heavy_lens: np.ndarray, p: np.ndarray) -> tuple[int, int, int]:
    """MergeStats of dt_merge for a zone [light | heavy runs] (dtmerge.py:166-238):
    depends only on the run lengths and the insertion points."""
    m = len(heavy_lens)
    heavy_total = int(heavy_lens.sum())
    if m == 0 or light_len + heavy_total == 0:
        return 0, 0, 0
    prefix = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(heavy_lens, out=prefix[1:])
    bounds = np.empty(m + 2, dtype=np.int64)
    bounds[0] = 0
    bounds[1:m + 1] = p
    bounds[m + 1] = light_len
    out = inm = rest = 0
    if heavy_total >= light_len:
        out = light_len
        for i in range(m):
            ln = int(heavy_lens[i])
            src = light_len + int(prefix[i])
            dst = int(p[i]) + int(prefix[i])
            if ln == 0 or dst == src:
                continue
            inm += ln if dst + ln <= src else 2 * ln
        for i in range(m + 1):
            f0, f1 = int(bounds[i]), int(bounds[i + 1])
            if f1 - f0 and int(prefix[i]):
                rest += f1 - f0
    else:
        out = heavy_total
        for i in range(m, 0, -1):
            f0, f1 = int(bounds[i]), int(bounds[i + 1])
            flen = f1 - f0
            dst = f0 + int(prefix[i])
            if flen == 0 or dst == f0:
                continue
            inm += flen if f0 + flen <= dst else 2 * flen
        rest = int(heavy_lens[heavy_lens > 0].sum())
    return out, inm, rest


class _Replay:
    def __init__(self, keys_in: np.ndarray, ks: np.ndarray, perm: np.ndarray, cfg: SortConfig, plain: bool):
        self.keys_in = keys_in
        self.ks = ks
        self.perm = perm
        self.cfg = cfg
        self.plain = plain
        self.n = int(ks.shape[0])
        self.W = ks.dtype.itemsize * 8
        self.stride = ceil_log2(self.n)

    # number of R's records at global sorted positions < pos (vectorised)
    @staticmethod
    def _count(R, pos):
        pos = np.asarray(pos, dtype=np.int64)
        c = np.zeros(pos.shape, dtype=np.int64)
        for a, b in R:
            c += np.clip(pos, a, b) - a
        return c

    @staticmethod
    def _cut(R, a, b, holes):
        """R ∩ [a, b) minus the (sorted, disjoint) position ranges in holes."""
        out = []
        for x, y in R:
            x, y = max(x, a), min(y, b)
            if x >= y:
                continue
            for h0, h1 in holes:
                if h1 <= x or h0 >= y:
                    continue
                if h0 > x:
                    out.append((x, h0))
                x = max(x, h1)
                if x >= y:
                    break
            if x < y:
                out.append((x, y))
        return out

    def _in_order_keys(self, R, depth):
        if depth == 0:
            return self.keys_in
        pos = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in R])
        order = np.argsort(self.perm[pos], kind="stable")
        return self.ks[pos[order]]

    def _samples(self, R, n_sub, gamma, depth, lo):
        count = min(n_sub, (1 << gamma) * ceil_log2(self.n))
        if count <= 0:
            return np.empty(0, dtype=self.ks.dtype)
        keys = self._in_order_keys(R, depth)
        out = np.empty(count, dtype=self.ks.dtype)
        for c, off in enumerate(range(0, count, _SAMPLE_CHUNK)):
            cnt = min(_SAMPLE_CHUNK, count - off)
            g = rng_stream(self.cfg.seed, _stream_id(depth, lo, c))
            idx = g.integers(0, n_sub, size=cnt, dtype=np.uint64)
            out[off:off + cnt] = keys[idx]
        out.sort()
        return out

    def _base(self, rep, n):
        if n <= 0:
            return
        rep.base_case_records += n
        if n > 1:
            rep.moves += n

    def sort_rec(self, R, lo, consumed, depth, src, rep):
        cfg, W, ks = self.cfg, self.W, self.ks
        n_sub = sum(b - a for a, b in R)
        rep.add_mass(depth, n_sub)
        if n_sub == 0:
            return src
        remaining = W - consumed
        if remaining <= 0:
            return src
        gamma = gamma_for(n_sub, remaining, cfg)
        if n_sub < cfg.effective_theta(gamma):
            self._base(rep, n_sub)
            return src
        # ---- step 1: plan (dtsort.py:212-241) ----
        heavy = np.empty(0, dtype=ks.dtype)
        thr = None
        if not self.plain and n_sub >= 2 * min(n_sub, (1 << gamma) * ceil_log2(self.n)):
            S = self._samples(R, n_sub, gamma, depth, lo)
            if depth == 0 and consumed == 0:
                mx = int(S.max()) if S.shape[0] else 0
                clz = W - mx.bit_length()
                skip = min((clz // gamma) * gamma, ((W - 1) // gamma) * gamma)
                if skip > 0:
                    thr = 1 << (W - skip)
                    consumed = skip
                    gamma = min(gamma, W - consumed)
            if S.shape[0]:
                sub = S[::ceil_log2(self.n)]
                vals, cnts = np.unique(sub, return_counts=True)
                heavy = vals[cnts >= 2]
        if depth == 0 and consumed > 0:
            rep.skipped_bits = consumed
        shift = W - consumed - gamma
        nz = 1 << gamma
        # ---- step 2: bucket sizes (counting_sort: one write per record) ----
        a0 = R[0][0]
        prefix = (int(ks[a0]) >> (shift + gamma)) << (shift + gamma) if shift + gamma < W else 0
        end = R[-1][1]
        pthr = end
        if thr is not None:  # thr = 2^(W - skip) <= 2^(W-1): representable
            pthr = int(np.searchsorted(ks, np.array(thr, dtype=ks.dtype), "left"))
            pthr = max(min(pthr, end), a0)
        zb = np.empty(nz + 1, dtype=np.int64)
        zb[0], zb[nz] = a0, pthr
        if nz > 1:
            v = np.array([prefix + (z << shift) for z in range(1, nz)], dtype=ks.dtype)
            zb[1:nz] = np.clip(np.searchsorted(ks, v, "left"), a0, pthr)
        zcnt = np.diff(self._count(R, zb))
        ovf = n_sub - int(zcnt.sum())
        # heavy buckets: keys below the overflow threshold, in their zone
        hz = ((heavy.astype(np.uint64) >> np.uint64(shift)) & np.uint64(nz - 1)).astype(np.int64)
        hlo = np.searchsorted(ks, heavy, "left").astype(np.int64)
        hhi = np.searchsorted(ks, heavy, "right").astype(np.int64)
        hcnt = self._count(R, hhi) - self._count(R, hlo)
        if thr is not None:  # overflow outranks heavy (sampler.py:76-100)
            hcnt[heavy.astype(np.uint64) >= np.uint64(thr)] = 0
        zheavy = np.bincount(hz, weights=hcnt, minlength=nz).astype(np.int64) if heavy.shape[0] else \
            np.zeros(nz, dtype=np.int64)
        light = zcnt - zheavy
        rep.moves += n_sub
        rep.note_distribution(depth)
        rep.add_mass(depth + 1, 0)
        rep.add_heavy_removed(depth, n_sub - int(light.sum()) - ovf)
        o = 1 - src
        # ---- step 3: children (dtsort.py:244-318) ----
        rem_after = W - consumed - gamma
        zone_h = np.zeros(nz + 1, dtype=np.int64)
        if heavy.shape[0]:
            np.cumsum(np.bincount(hz, minlength=nz), out=zone_h[1:])
        if rem_after > 0:
            span = 0
            base = lo
            for z in range(nz):
                size = int(light[z])
                h0, h1 = int(zone_h[z]), int(zone_h[z + 1])
                if size > 0:
                    cg = gamma_for(size, rem_after, cfg)
                    if size < cfg.effective_theta(cg):
                        span += size
                    else:
                        if span:
                            rep.add_mass(depth + 1, span)
                            self._base(rep, span)
                            span = 0
                        holes = [(int(hlo[i]), int(hhi[i])) for i in range(h0, h1)]
                        CR = self._cut(R, int(zb[z]), int(zb[z + 1]), holes)
                        buf = self.sort_rec(CR, base, consumed + gamma, depth + 1, o, rep)
                        if buf != o:
                            rep.moves += size
                if h1 > h0 and span:
                    rep.add_mass(depth + 1, span)
                    self._base(rep, span)
                    span = 0
                base += int(zcnt[z])
            if span:
                rep.add_mass(depth + 1, span)
                self._base(rep, span)
        if ovf > 0:
            self._base(rep, ovf)
        # ---- step 4: dovetail merge per zone with heavy keys ----
        if not self.plain and heavy.shape[0]:
            for z in range(nz):
                h0, h1 = int(zone_h[z]), int(zone_h[z + 1])
                if h1 <= h0 or int(light[z]) + int(hcnt[h0:h1].sum()) == 0:
                    continue
                lens = hcnt[h0:h1]
                # light records below each heavy key: zone records below it
                # minus this zone's heavy records below it
                below = self._count(R, hlo[h0:h1]) - self._count(R, np.array([zb[z]]))[0]
                p = below - np.concatenate(([0], np.cumsum(lens)[:-1]))
                out, inm, rest = _merge_stats(int(light[z]), lens, p)
                rep.merge_out_copies += out
                rep.merge_in_array_moves += inm
                rep.moves += out + inm + rest
        return o


def replay_report(keys_in: np.ndarray, ks: np.ndarray, perm: np.ndarray, cfg: SortConfig,
                  plain: bool) -> InstrumentReport:
    """The reference InstrumentReport for sorting ``keys_in`` (dtsort.py:81-108)."""
    rep = InstrumentReport()
    n = int(ks.shape[0])
    if n == 0:
        rep.add_mass(0, 0)
        return rep
    r = _Replay(keys_in, ks, perm, cfg, plain)
    buf = r.sort_rec([(0, n)], 0, 0, 0, 0, rep)
    if buf == 1:
        rep.moves += n
    return rep
