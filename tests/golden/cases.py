"""Deterministic parity cases shared by make_golden.py (which runs the
reference package to produce tests/golden/*.json|npz) and the tests.

Inputs are regenerated from numpy's PCG64 `default_rng(seed)` (stable
across numpy versions by numpy's stream-compatibility policy); the
fixtures store the reference's output digests and InstrumentReport
counters, plus the raw arrays of the small cases.
"""
from __future__ import annotations

import hashlib

import numpy as np

DEEP = dict(gamma_lo=4, gamma_hi=4, base_case_threshold=16)
THEORY = dict(theory_mode=True, base_case_exponent=2, gamma_lo=4, gamma_hi=4)


def _dist(name: str, n: int, width: int, rng: np.random.Generator) -> np.ndarray:
    dt = np.uint32 if width == 32 else np.uint64
    if name == "full":
        return rng.integers(0, (1 << 64) - 1, size=n, dtype=np.uint64, endpoint=True).astype(dt)
    if name == "few":
        return rng.integers(0, 7, size=n).astype(dt)
    if name == "sorted":
        return np.arange(n).astype(dt)
    if name == "reversed":
        return np.arange(n)[::-1].astype(dt)
    if name == "const":
        return np.full(n, 42, dt)
    if name == "two":
        return np.tile([9, 3], n // 2 + 1)[:n].astype(dt)
    if name == "small16":
        return rng.integers(0, 1 << 16, size=n).astype(dt)
    if name == "zipf":
        return (rng.zipf(1.3, size=n) % (1 << 31)).astype(dt)
    if name == "planted":
        k = rng.integers(0, (1 << 64) - 1, size=n, dtype=np.uint64, endpoint=True).astype(dt)
        k[: n // 3] = 0x12345678
        rng.shuffle(k)
        return k
    if name == "outliers":
        k = rng.integers(0, 1 << 12, size=n).astype(dt)
        if n >= 3:
            k[rng.integers(0, n, size=3)] = np.array([1 << 20, (1 << 32) - 1, 1 << 28]).astype(dt)
        return k
    if name == "exp":
        return np.floor(rng.exponential(1e5, size=n)).astype(dt)
    if name == "bexp":
        w = rng.integers(0, (1 << 64) - 1, size=n, dtype=np.uint64, endpoint=True)
        g = np.minimum(rng.geometric(0.5, size=n) - 1, 63).astype(np.uint64)
        k = w >> g
        return (k if width == 64 else (k >> np.uint64(32))).astype(dt)
    raise ValueError(name)


def make_input(case: dict) -> tuple[np.ndarray, np.ndarray | None]:
    rng = np.random.default_rng(case["seed"])
    keys = _dist(case["dist"], case["n"], case["width"], rng)
    pays = np.arange(case["n"], dtype=np.uint64) if case["payloads"] else None
    return keys, pays


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        if a is not None:
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sort_cases() -> list[dict]:
    out = []
    seed = 100
    for width in (32, 64):
        for n in (0, 1, 2, 17, 1000, 30_000):
            for dist in ("full", "few", "sorted", "reversed", "const", "two"):
                out.append(dict(name=f"{dist}-{width}-{n}", dist=dist, n=n, width=width,
                                seed=seed, payloads=True, cfg={}))
                seed += 1
        for dist in ("small16", "zipf", "planted", "outliers", "exp", "bexp"):
            out.append(dict(name=f"{dist}-{width}-120000", dist=dist, n=120_000, width=width,
                            seed=seed, payloads=True, cfg={}))
            seed += 1
        for dist in ("full", "few", "const", "zipf"):
            out.append(dict(name=f"deep-{dist}-{width}", dist=dist, n=20_000, width=width,
                            seed=seed, payloads=True, cfg=DEEP))
            seed += 1
        out.append(dict(name=f"theory-full-{width}", dist="full", n=40_000, width=width,
                        seed=seed, payloads=True, cfg=THEORY))
        seed += 1
        out.append(dict(name=f"keysonly-full-{width}", dist="full", n=5000, width=width,
                        seed=seed, payloads=False, cfg={}))
        seed += 1
    # larger cases that exercise sampling + heavy buckets at several levels
    out.append(dict(name="planted-32-1e6", dist="planted", n=1_000_000, width=32, seed=900,
                    payloads=True, cfg={}))
    out.append(dict(name="zipf-32-1e6", dist="zipf", n=1_000_000, width=32, seed=901,
                    payloads=True, cfg={}))
    out.append(dict(name="exp-64-1e6", dist="exp", n=1_000_000, width=64, seed=902,
                    payloads=True, cfg={}))
    return out


# dt_merge exhaustive grid (the reference test_dtmerge.py:62-82 shape)
def merge_grid():
    from itertools import combinations, combinations_with_replacement, product

    light_vals = (0, 2, 4, 6)
    lights = [list(c) for ln in range(5) for c in combinations_with_replacement(light_vals, ln)]
    heavies = [[]]
    for m in (1, 2, 3):
        for ks in combinations((1, 3, 5), m):
            for lens in product((1, 2, 3), repeat=m):
                heavies.append(list(zip(ks, lens)))
    return [(light, heavy) for light in lights for heavy in heavies]


def build_zone(light, heavy, key_dtype=np.uint32):
    parts = [np.asarray(light, dtype=key_dtype)]
    for key, ln in heavy:
        parts.append(np.full(ln, key, dtype=key_dtype))
    keys = np.concatenate(parts)
    pays = np.arange(keys.shape[0], dtype=np.uint64)
    return keys, pays
