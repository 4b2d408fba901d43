"""k_scatter phase profile (needs libdts_phase.so: make -C csrc ../_lib/libdts_phase.so).
DTS_LIB=paper_2401_00710_b200/_lib/libdts_phase.so python tools/phase_prof.py [n]"""
import ctypes, sys
import torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import SortConfig, _lib
from paper_2401_00710_b200.dtsort import sort_device

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
L = _lib.lib()
L.dts_debug_phases.restype = ctypes.c_int
buf = (ctypes.c_ulonglong * 16)()
import os
CFG = os.environ.get("DTS_CFG", "c2")  # bench.py workload name
import bench
from paper_2401_00710_b200 import gen
src, v0 = gen.generate_device(bench.CONFIGS[CFG], n, 0, "cuda")
k = torch.empty_like(src); v = torch.empty_like(v0)
LOCAL = os.environ.get("DTS_PHASE", "1") == "2"
if LOCAL:
    names = ["tma wait", "keys+diff", "zero(-)", "hist", "scan1", "scan2", "slots", "rank barrier", "write-out", "top", "rank (thread 0)"]
elif os.environ.get("DTS_WC", "1") != "0":
    names = ["stripe/top", "tma wait", "rank", "pair scan", "binfo+map", "placement",
             "check+write-out", "flush+claim", "carry", "plan+cst"]
else:
    names = ["top->issue", "issue->bar1", "tma wait", "rank", "prefix+scan", "tst", "placement",
             "lookback", "bar(lookback)", "write-out"]
for rep in range(2):
    k.copy_(src); v.copy_(v0); torch.cuda.synchronize()
    L.dts_debug_phases(buf, 16, 1)
    r = sort_device(k, v, SortConfig(), 0, report=True)
    torch.cuda.synchronize()
    L.dts_debug_phases(buf, 16, 0)
tiles = (r.kernel_records["local_sort"] / 4100.0) if LOCAL else (r.kernel_records["scatter"] / 9216.0)
ctas = buf[14]
tot = sum(buf[i] for i in range(11))
print(f"tiles ~{tiles:.0f}  CTA-runs {ctas}  spins {buf[15]}  order-fixes wc {buf[13]} lookback {buf[12]}")
for i, nm in enumerate(names[:11]):
    print(f"{nm:16s} {buf[i]/tiles:9.0f} cycles/tile  {100*buf[i]/tot:5.1f}%")
print(f"{'total':16s} {tot/tiles:9.0f} cycles/tile")
if LOCAL:
    print(f"local-sort spans: nibble path {buf[11]}, packed path {buf[10]}, LSD {buf[13]}, "
          f"all-equal {buf[15]}, re-sorted after an order check failure {buf[12]}")
