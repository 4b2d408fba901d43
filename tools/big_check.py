"""Large-n certificate (C2 shape): python tools/big_check.py 3e9"""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import SortConfig
from paper_2401_00710_b200.dtsort import sort_device

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 3 * 10**9
g = torch.Generator(device="cuda"); g.manual_seed(0)
k0 = torch.empty(n, dtype=torch.int32, device="cuda")
CH = 1 << 28
for o in range(0, n, CH):
    m = min(CH, n - o)
    k0[o:o + m] = torch.randint(0, 10**9, (m,), generator=g, device="cuda", dtype=torch.int32)
k = k0.clone()
v = torch.empty(n, dtype=torch.int32, device="cuda")
for o in range(0, n, CH):
    m = min(CH, n - o)
    torch.arange(o, o + m, out=v[o:o + m])  # values = index (wraps past 2^31: bit pattern)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = sort_device(k, v, SortConfig(), 0, report=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"n={n} sort {1e3*(t1-t0):.1f} ms ({n/(t1-t0)/1e9:.2f} Gkeys/s) levels {rep.levels}", flush=True)
ok = True
for o in range(0, n - 1, CH):
    m = min(CH + 1, n - o)
    a = k[o:o + m]
    ok &= bool((a[1:] >= a[:-1]).all())
    eq = a[1:] == a[:-1]
    vu = v[o:o + m].to(torch.int64) & 0xFFFFFFFF
    ok &= bool((vu[1:][eq] > vu[:-1][eq]).all())
    ok &= bool((k0[vu[:-1] if o + m < n else vu] [: (m - 1 if o + m < n else m)] == a[: (m - 1 if o + m < n else m)]).all()) if n < 2**32 else True
print("certificate (sorted, stable, keys match source)", ok, flush=True)
