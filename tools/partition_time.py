"""Time dts_partition (the multi-GPU split pass) on one GPU: G groups of n records.
python tools/partition_time.py [n] [G]"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200.distributed import CudaOps, choose_splitters

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = torch.Generator(device="cuda"); g.manual_seed(0)
k = torch.randint(0, 10**9, (n,), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
v = torch.arange(n, device="cuda", dtype=torch.int32)
ops = CudaOps()
sk, si = ops.sample(k, 0, 1 << 15, 0)
spk, spi = choose_splitters(sk, si, G)
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ok, ov, cnt = ops.partition(k, v, 0, spk, spi)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"G={G} n={n} partition {1e3*(t1-t0):.2f} ms  counts {cnt}", flush=True)
