"""Seeded synthetic workloads of BASELINE.json's configs, generated on the GPU.

The reference's own generators (gen.py) use other shapes; BASELINE.json
names these inputs:

* C1 ``u32full``   : uint32 keys uniform on [0, 2^32)
* C2 ``uniform1e9``: uint32 keys uniform on [0, 10^9)
* C3 ``zipf``      : Zipf(s) ranks on [1, 10^9] mapped through a seeded
                     random permutation of [0, 10^9) (heavy keys scattered)
* C4 ``exp``       : uint64 floor(X), X ~ Exponential(rate)
* C4 ``bexp``      : uint64 w >> g, w uniform 64-bit, g ~ Geometric(1/2)-1
Values are the original (global) index.

The Zipf ranks use rejection-inversion (Hörmann & Derflinger 1996),
vectorised over torch tensors; every distribution is exact, seeded and
reproducible for a given (seed, n).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["generate_device", "zipf_ranks_device", "zipf_keys_host"]


def _H(x, s):
    """Integral of t^-s (the rejection-inversion hull), numerically stable."""
    import torch

    lx = torch.log(x)
    if abs(1.0 - s) < 1e-12:
        return lx
    t = (1.0 - s) * lx
    return torch.where(t.abs() > 1e-8, torch.expm1(t) / t, 1.0 + t / 2) * lx


def _Hinv(y, s):
    import torch

    if abs(1.0 - s) < 1e-12:
        return torch.exp(y)
    t = (1.0 - s) * y
    f = torch.where(t.abs() > 1e-8, torch.log1p(t) / torch.where(t == 0, torch.ones_like(t), t),
                    1.0 - t / 2)
    return torch.exp(f * y)


def _Hs(x: float, s: float) -> float:
    if abs(1.0 - s) < 1e-12:
        return math.log(x)
    t = (1.0 - s) * math.log(x)
    return (math.expm1(t) / t if abs(t) > 1e-8 else 1.0 + t / 2) * math.log(x)


def _Hinvs(y: float, s: float) -> float:
    if abs(1.0 - s) < 1e-12:
        return math.exp(y)
    t = (1.0 - s) * y
    f = math.log1p(t) / t if abs(t) > 1e-8 else 1.0 - t / 2
    return math.exp(f * y)


def zipf_ranks_device(s: float, n: int, N: int, gen, device):
    """n ranks in [1, N] with P(k) ~ k^-s (s > 0), rejection-inversion."""
    import torch

    h_x1 = _Hs(1.5, s) - 1.0
    h_n = _Hs(N + 0.5, s)
    cut = 2.0 - _Hinvs(_Hs(2.5, s) - 2.0 ** (-s), s)
    out = torch.empty(n, dtype=torch.int64, device=device)
    todo = torch.arange(n, device=device)
    while todo.numel():
        u = torch.rand(todo.numel(), generator=gen, device=device, dtype=torch.float64)
        y = h_n + u * (h_x1 - h_n)
        x = _Hinv(y, s)
        k = torch.clamp(torch.floor(x + 0.5), 1, N)
        acc = ((k - x) <= cut) | (y >= _H(k + 0.5, s) - torch.pow(k, -s))
        out[todo[acc]] = k[acc].to(torch.int64)
        todo = todo[~acc]
    return out


def generate_device(cfgd: dict, n: int, seed: int, device, gbase: int = 0):
    """(keys, values) torch tensors on `device`; keys int32/int64 holding the
    unsigned bit patterns, values = global index."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    d = cfgd["dist"]
    kb, vb = cfgd["kb"], cfgd["vb"]
    if d == "uniform1e9":
        k = torch.randint(0, 10**9, (n,), generator=g, device=device, dtype=torch.int32)
    elif d == "u32full":
        k = torch.randint(-(2**31), 2**31, (n,), generator=g, device=device, dtype=torch.int32)
    elif d == "zipf":
        ranks = zipf_ranks_device(cfgd["s"], n, 10**9, g, device)
        perm = torch.randperm(10**9, generator=g, device=device, dtype=torch.int32)
        k = perm[ranks - 1]
        del perm, ranks
    elif d == "exp":
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        k = torch.floor(-torch.log1p(-u) / cfgd["rate"]).clamp(0, 2**63 - 1).to(torch.int64)
    elif d == "bexp":
        hi = torch.randint(-(2**31), 2**31, (n,), generator=g, device=device, dtype=torch.int64)
        lo = torch.randint(0, 2**32, (n,), generator=g, device=device, dtype=torch.int64)
        w = (hi << 32) | lo
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        gsh = torch.clamp(torch.floor(-torch.log2(1.0 - u)), 0, 63).to(torch.int64)
        mask = torch.where(gsh == 0, torch.full_like(gsh, -1), (torch.ones_like(gsh) << (64 - gsh)) - 1)
        k = (w >> gsh) & mask
    else:
        raise ValueError(d)
    if kb == 8 and k.dtype != torch.int64:
        k = k.to(torch.int64) & 0xFFFFFFFF
    if kb == 4 and k.dtype != torch.int32:
        k = k.to(torch.int32)
    v = None
    if vb:
        v = torch.arange(gbase, gbase + n, device=device, dtype=torch.int64)
        v = v.to(torch.int32) if vb == 4 else v
    return k.contiguous(), v


def zipf_keys_host(s: float, n: int, N: int, seed: int) -> np.ndarray:
    """Host copy of the C3 keys (generated on the GPU when one is present)."""
    import torch

    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    k, _ = generate_device(dict(dist="zipf", s=s, kb=4, vb=0), n, seed, dev)
    return k.cpu().numpy().view(np.uint32).copy()
