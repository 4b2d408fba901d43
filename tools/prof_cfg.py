"""Profiling driver: one dt_sort of a bench.py workload (its exact seeded input) on cuda:0.
Usage: python tools/prof_cfg.py <config> [n] [seed]"""
import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2401_00710_b200 import SortConfig, gen
from paper_2401_00710_b200.dtsort import sort_device

cfg = sys.argv[1]
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**9
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1000  # bench.py's rank-0 seed
k, v = gen.generate_device(bench.CONFIGS[cfg], n, seed, "cuda")
rep = sort_device(k, v, SortConfig(), 0, report=True)
torch.cuda.synchronize()
print("ok levels", rep.levels, "launches", rep.gpu_launches, rep.kernel_launches)
