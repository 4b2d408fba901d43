"""Randomised parity sweep against numpy's stable argsort (scratch diagnostic):
python tools/fuzz_check.py [cases] [seed]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import RecordArray, SortConfig, dt_sort, plain_msd_sort

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 150
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
fails = 0
for c in range(cases):
    kdt = rng.choice([np.uint32, np.uint64])
    pdt = rng.choice([None, np.uint32, np.uint64])
    w = 32 if kdt == np.uint32 else 64
    n = int(rng.choice([rng.integers(1, 5000), rng.integers(5000, 300_000), rng.integers(300_000, 3_000_000)]))
    bits = int(rng.integers(1, w + 1))  # key range
    hi = (1 << bits) - 1
    keys = rng.integers(0, hi, size=n, dtype=np.uint64, endpoint=True).astype(kdt)
    kind = rng.choice(["plain", "heavy", "manyheavy", "zipf", "shifted"])
    if kind == "heavy":  # a few keys with a large share (long bucket runs per tile)
        for _ in range(int(rng.integers(1, 4))):
            m = int(n * rng.uniform(0.02, 0.6))
            keys[rng.integers(0, n, size=m)] = kdt(rng.integers(0, hi, endpoint=True, dtype=np.uint64))
    elif kind == "manyheavy":  # dozens of moderately heavy keys
        hk = rng.integers(0, hi, size=int(rng.integers(5, 60)), endpoint=True, dtype=np.uint64).astype(kdt)
        sel = rng.random(n) < rng.uniform(0.2, 0.9)
        keys[sel] = hk[rng.integers(0, len(hk), size=int(sel.sum()))]
    elif kind == "zipf":
        keys = (rng.zipf(rng.uniform(1.1, 2.0), size=n).astype(np.uint64) % np.uint64(max(hi, 1))).astype(kdt)
    elif kind == "shifted":  # bit-skewed
        keys = (keys.astype(np.uint64) >> rng.geometric(0.5, size=n).astype(np.uint64).clip(0, 63)).astype(kdt)
    pays = None if pdt is None else np.arange(n, dtype=pdt)
    sorter = dt_sort if rng.random() < 0.8 else plain_msd_sort
    only = int(sys.argv[sys.argv.index("-only") + 1]) if "-only" in sys.argv else -1
    seed_c = int(rng.integers(0, 1000))
    if only >= 0 and c != only:
        continue
    if "-v" in sys.argv:
        print(c, kdt.__name__, None if pdt is None else pdt.__name__, n, bits, kind, sorter.__name__, flush=True)
    order = np.argsort(keys, kind="stable")
    rec = RecordArray(keys.copy(), None if pays is None else pays.copy())
    sorter(rec, SortConfig(seed=seed_c))
    ok = np.array_equal(rec.keys, keys[order]) and (pays is None or np.array_equal(rec.payloads, pays[order]))
    if not ok:
        fails += 1
        print("FAIL", c, kdt.__name__, None if pdt is None else pdt.__name__, n, bits, kind, sorter.__name__, flush=True)
print(f"fuzz: {cases - fails}/{cases} ok")
