import sys, time, torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import gen, SortConfig
from paper_2401_00710_b200.dtsort import sort_device
n = int(float(sys.argv[1]))
t = time.time(); d, s = gen.rmat_edges(n, 28, 0); torch.cuda.synchronize(); print("gen", n, time.time() - t, flush=True)
for r in range(3):
    k = d.clone(); v = s.clone(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t = time.time(); a.record(); rep = sort_device(k, v, SortConfig(), 0, report=True); b.record(); b.synchronize()
    print("sort", r, a.elapsed_time(b), "ms wall", time.time() - t, "levels", rep.levels, {kk: round(vv, 1) for kk, vv in rep.kernel_ms.items()}, flush=True)
    del k, v
