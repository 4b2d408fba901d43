"""One profiled C2-shaped sort with DTS_TIMELINE=1 / DTS_TRACE=1: per-launch
start/end on the library's stream (gaps = host round trips).
Usage: DTS_TIMELINE=1 DTS_TRACE=1 python tools/timeline.py [n] [config]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import SortConfig, gen
from paper_2401_00710_b200.dtsort import sort_device
import bench

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
cfgd = dict(bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c2"])
k0, v0 = gen.generate_device(cfgd, n, 1000, torch.device("cuda", 0))
for it in range(3):
    k, v = k0.clone(), None if v0 is None else v0.clone()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rep = sort_device(k, v, SortConfig(seed=0), 0, profile=(it == 2), report=True)
    b.record(); b.synchronize()
    print(f"iter {it}: {a.elapsed_time(b):.3f} ms", {c: round(x, 3) for c, x in rep.kernel_ms.items()}, file=sys.stderr)
