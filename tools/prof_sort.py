"""Profiling driver: one dt_sort of n u32/u32 (C2-shaped) records on cuda:0.
Usage: python tools/prof_sort.py [n] [kbytes] [vbytes]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import SortConfig
from paper_2401_00710_b200.dtsort import sort_device

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
kb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
vb = int(sys.argv[3]) if len(sys.argv) > 3 else 4
dt = {4: torch.int32, 8: torch.int64}
g = torch.Generator(device="cuda"); g.manual_seed(0)
k = torch.randint(0, 10**9, (n,), generator=g, device="cuda", dtype=torch.int64).to(dt[kb])
v = torch.arange(n, device="cuda", dtype=dt[vb]) if vb else None
rep = sort_device(k, v, SortConfig(), 0, report=True)
torch.cuda.synchronize()
print("ok levels", rep.levels, "launches", rep.gpu_launches, rep.kernel_launches)
