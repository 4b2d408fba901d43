"""A few small sorts for compute-sanitizer (memcheck / racecheck / synccheck):
compute-sanitizer --tool racecheck python tools/san_check.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import RecordArray, SortConfig, dt_sort

rng = np.random.default_rng(5)
def run(keys, pdt, label):
    pays = None if pdt is None else np.arange(len(keys), dtype=pdt)
    order = np.argsort(keys, kind="stable")
    rec = RecordArray(keys.copy(), None if pays is None else pays.copy())
    dt_sort(rec, SortConfig(seed=0))
    ok = np.array_equal(rec.keys, keys[order]) and (pays is None or np.array_equal(rec.payloads, pays[order]))
    print(label, len(keys), "ok" if ok else "FAIL", flush=True)
    return ok

n = int(sys.argv[1]) if len(sys.argv) > 1 else 150_000
allok = True
for kdt, pdt in ((np.uint32, np.uint32), (np.uint64, np.uint64), (np.uint32, None), (np.uint64, np.uint32)):
    w = 32 if kdt == np.uint32 else 64
    uni = rng.integers(0, 10**9, size=n).astype(kdt)
    heavy = uni.copy(); heavy[: n // 3] = 777; heavy[n // 3: n // 2] = 123456; rng.shuffle(heavy)
    zipf = (rng.zipf(1.3, size=n) % (2**31)).astype(kdt)
    wide = rng.integers(0, 2**w - 1, size=n, dtype=np.uint64, endpoint=True).astype(kdt)
    for name, k in (("uniform", uni), ("heavy", heavy), ("zipf", zipf), ("wide", wide)):
        allok &= run(k, pdt, f"{kdt.__name__}/{None if pdt is None else pdt.__name__} {name}")
print("ALL OK" if allok else "SOME FAILED")
