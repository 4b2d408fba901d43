"""Host-scheduler trace: DTS_TRACE=1 python tools/trace_sort.py [n] [kb] [vb] [reps]"""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import SortConfig
from paper_2401_00710_b200.dtsort import sort_device

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
kb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
vb = int(sys.argv[3]) if len(sys.argv) > 3 else 4
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
dt = {4: torch.int32, 8: torch.int64}
g = torch.Generator(device="cuda"); g.manual_seed(0)
src = torch.randint(0, 10**9, (n,), generator=g, device="cuda", dtype=torch.int64).to(dt[kb])
k = torch.empty_like(src)
v = torch.empty(n, device="cuda", dtype=dt[vb]) if vb else None
for r in range(reps):
    k.copy_(src)
    if v is not None:
        torch.arange(n, out=v)
    torch.cuda.synchronize()
    print(f"--- rep {r}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    rep = sort_device(k, v, SortConfig(), 0, report=True, profile=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"rep {r}: {1e3*(t1-t0):.2f} ms wall, kernel_ms "
          f"{ {c: round(x, 3) for c, x in rep.kernel_ms.items()} }", flush=True)
