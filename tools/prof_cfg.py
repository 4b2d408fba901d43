"""Profiling driver: one sort of a bench.py workload on cuda:0 (inputs from
the bench's own generator).  Usage: python tools/prof_cfg.py <config> [n]"""
import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2401_00710_b200 import SortConfig, gen
from paper_2401_00710_b200.dtsort import sort_device

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfgd = dict(bench.CONFIGS[cfg])
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else cfgd["n"]
k, v = gen.generate_device(cfgd, n, 1000, torch.device("cuda", 0))
torch.cuda.synchronize()
rep = sort_device(k, v, SortConfig(seed=0), 0, report=True)
torch.cuda.synchronize()
print("ok", cfg, "levels", rep.levels, "launches", rep.gpu_launches)
