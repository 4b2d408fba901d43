"""Quick GPU check: parity vs numpy stable argsort on many shapes + timing.

Scratch diagnostic (not a test): python tools/quick_check.py [--big]
"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import RecordArray, SortConfig, dt_sort, plain_msd_sort, dt_merge
from paper_2401_00710_b200.dtsort import sort_device

def check(keys, pays, cfg=None, sorter=dt_sort, label=""):
    order = np.argsort(keys, kind="stable")
    rec = RecordArray(keys.copy(), None if pays is None else pays.copy())
    rep = sorter(rec, cfg)
    ok = np.array_equal(rec.keys, keys[order]) and (pays is None or np.array_equal(rec.payloads, pays[order]))
    if not ok:
        bad = np.nonzero(rec.keys != keys[order])[0]
        print("FAIL", label, len(keys), keys.dtype, None if pays is None else pays.dtype, "first bad", bad[:5])
    return ok

rng = np.random.default_rng(0)
fails = 0
total = 0
DEEP = SortConfig(gamma_lo=4, gamma_hi=4, base_case_threshold=16)
for kdt in (np.uint32, np.uint64):
    for pdt in (None, np.uint32, np.uint64):
        for n in (0, 1, 2, 17, 1000, 8191, 8193, 30000, 100000, 1000003):
            w = 32 if kdt == np.uint32 else 64
            cases = {
                "full": rng.integers(0, 2**w - 1, size=n, dtype=np.uint64, endpoint=True).astype(kdt),
                "few": rng.integers(0, 7, size=n).astype(kdt),
                "sorted": np.arange(n).astype(kdt),
                "rev": np.arange(n)[::-1].astype(kdt),
                "const": np.full(n, 42, kdt),
                "zipfish": (rng.zipf(1.3, size=n) % (2**31)).astype(kdt),
                "small": rng.integers(0, 1 << 16, size=n).astype(kdt),
            }
            for name, keys in cases.items():
                pays = None if pdt is None else np.arange(n, dtype=pdt)
                for sorter in (dt_sort, plain_msd_sort):
                    total += 1
                    if not check(keys, pays, None, sorter, f"{name}/{sorter.__name__}"):
                        fails += 1
                if n <= 30000:
                    total += 1
                    if not check(keys, pays, DEEP, dt_sort, f"{name}/DEEP"):
                        fails += 1
print(f"parity: {total - fails}/{total} ok")

# planted heavy keys
n = 2_000_000
keys = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
keys[: n // 3] = 0x12345678
keys[n // 3 : n // 2] = 0x12345679
rng.shuffle(keys)
pays = np.arange(n, dtype=np.uint32)
rec = RecordArray(keys.copy(), pays.copy())
rep = dt_sort(rec, SortConfig(instrument=True))
order = np.argsort(keys, kind="stable")
print("heavy planted ok:", np.array_equal(rec.keys, keys[order]) and np.array_equal(rec.payloads, pays[order]), rep.heavy_records_removed, rep.levels, rep.skipped_bits)

# dt_merge known case
zk = np.array([1, 3, 5, 4, 4], np.uint32); zp = np.arange(5, dtype=np.uint64)
st = dt_merge(zk, zp, 3, np.array([4], np.uint32), [2], np.empty(2, np.uint32), np.empty(2, np.uint64))
print("merge:", zk.tolist(), zp.tolist(), st)

# timing on device
def gpu_time(n, kdt=torch.int32, hi=10**9, reps=3, vals=True):
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    src = torch.randint(0, hi, (n,), generator=g, device="cuda", dtype=torch.int64).to(kdt)
    vsrc = torch.arange(n, device="cuda", dtype=kdt) if vals else None
    k = torch.empty_like(src); v = torch.empty_like(vsrc) if vals else None
    ws = None
    ts = []
    for r in range(reps + 1):
        k.copy_(src)
        if vals: v.copy_(vsrc)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        rep = sort_device(k, v, SortConfig(), 0, profile=(r == reps), report=True)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ok = bool((k[1:] >= k[:-1]).all()) if kdt == torch.int64 or hi < 2**31 else None
    print(f"n={n} {kdt} ms={ts} min={min(ts[:-1]) if reps>1 else ts[0]:.3f} Gkeys/s={n/min(ts[:-1])/1e6:.2f} sorted={ok}")
    print("  levels", rep.levels, "mass", rep.level_mass, "D", rep.records_distributed, "launches", rep.gpu_launches)
    print("  kernel_ms", {k_: round(v_, 3) for k_, v_ in rep.kernel_ms.items()})
    print("  kernel_launches", rep.kernel_launches)

if '--parity-only' in sys.argv:
    sys.exit(0)
gpu_time(10**7)
gpu_time(10**8)
if "--big" in sys.argv:
    gpu_time(10**9)
