"""Time dts_partition (the multi-GPU split pass) on one GPU:
python tools/part_time.py [n] [G]  — C2-shaped u32/u32 records, sampled splitters."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200.distributed import CudaOps, choose_splitters

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = torch.Generator(device="cuda"); g.manual_seed(1)
k = torch.randint(0, 10**9, (n,), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
v = torch.arange(n, device="cuda", dtype=torch.int32)
ops = CudaOps()
sk, si = ops.sample(k, 0, 1 << 15, 0)
spk, spi = choose_splitters(sk, si, G)
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pk, pv, send = ops.partition(k, v, 0, spk, spi)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"partition n={n} G={G}: {1e3 * (t1 - t0):.2f} ms  counts min {min(send)} max {max(send)}")
# check: stable partition (keys grouped by destination, values ascending inside each)
off = 0
ok = True
for d, c in enumerate(send):
    vv = pv[off:off + c]
    ok &= bool((vv[1:] > vv[:-1]).all().item()) if c > 1 else True
    off += c
print("stable inside destinations:", ok, " total", off == n)
