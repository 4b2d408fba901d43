"""Calibration only (not a product path): torch.sort (CUB radix sort) timings."""
import torch
torch.cuda.init()
for n in (10**8, 10**9):
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    k = torch.randint(0, 10**9, (n,), generator=g, device="cuda", dtype=torch.int32)
    for stable in (True,):
        for it in range(3):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); s, i = torch.sort(k, stable=stable); b.record(); b.synchronize()
            print(f"n={n} torch.sort int32 keys + int64 idx stable={stable}: {a.elapsed_time(b):.2f} ms "
                  f"{n/a.elapsed_time(b)/1e6:.1f} Gkeys/s", flush=True)
            del s, i
    torch.cuda.empty_cache()
