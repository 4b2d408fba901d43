"""Scheduler trace of one bench config: DTS_TRACE=1 python tools/trace_cfg.py c4-exp1e-7 [n]"""
import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2401_00710_b200 import SortConfig
from paper_2401_00710_b200.dtsort import sort_device

cfg = dict(bench.CONFIGS[sys.argv[1]])
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else cfg["n"]
k, v = bench.gen_device(cfg, n, 1000, torch.device("cuda", 0))
k0, v0 = k.clone(), None if v is None else v.clone()
for r in range(2):
    k.copy_(k0)
    if v is not None:
        v.copy_(v0)
    torch.cuda.synchronize()
    print(f"--- rep {r}", file=sys.stderr, flush=True)
    rep = sort_device(k, v, SortConfig(), 0, report=True, profile=True)
    torch.cuda.synchronize()
    print(f"rep {r}: levels {rep.levels} D {rep.records_distributed} kernel_ms "
          f"{ {c: round(x, 3) for c, x in rep.kernel_ms.items()} } launches {rep.kernel_launches}", flush=True)
