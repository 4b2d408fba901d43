"""Sweep library variants / env knobs on the C2 workload (scratch tool).
Usage: python tools/sweep.py n "LIB:ENV=..;ENV=.." ..."""
import os, subprocess, sys, json
n = sys.argv[1]
child = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2401_00710_b200 import SortConfig
from paper_2401_00710_b200.dtsort import sort_device
n = int(float(sys.argv[1]))
g = torch.Generator(device="cuda"); g.manual_seed(0)
src = torch.randint(0, 10**9, (n,), generator=g, device="cuda", dtype=torch.int64).to(torch.int32)
vsrc = torch.arange(n, device="cuda", dtype=torch.int32)
k = torch.empty_like(src); v = torch.empty_like(vsrc)
ws = torch.empty(int(1.2 * n * 8) + (64 << 20), dtype=torch.uint8, device="cuda")
ts = []
for r in range(4):
    k.copy_(src); v.copy_(vsrc); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); rep = sort_device(k, v, SortConfig(), 0, profile=(r == 3), workspace=ws, report=True); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ok = bool((k[1:] >= k[:-1]).all())
print(json.dumps({"ms": round(min(ts[1:3]), 3), "ok": ok, "levels": rep.levels,
                  "kms": {a: round(b, 3) for a, b in rep.kernel_ms.items() if b}}))
'''
for spec in sys.argv[2:]:
    lib, _, envs = spec.partition(":")
    env = dict(os.environ)
    if lib:
        env["DTS_LIB"] = f"paper_2401_00710_b200/_lib/{lib}"
    for kv in filter(None, envs.split(";")):
        k, _, v = kv.partition("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", child, n], env=env, capture_output=True, text=True)
    print(spec, "->", r.stdout.strip() or r.stderr[-500:], flush=True)
