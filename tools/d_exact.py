"""D (records the reference's counting_sort distributes) on
bench.py's EXACT inputs: each config's keys are generated on the device as
bench.py generates them (seed 1000 + rank 0, gbase 0), copied to the host,
and sorted by the oracle (C++ restatement of the reference's dt_sort with
SortConfig(seed=0), oracle/dovetail_oracle.cpp) whose records_distributed
counter sums len(keys) over every counting_sort call (the wrapper
measurement SURVEY.md §8(d) prescribes).  Writes profiles/D_exact.json.
Usage (GPU box): python tools/d_exact.py [config ...]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import oracle as ora  # noqa: E402

out_path = os.path.join(bench.ROOT, "profiles", "D_exact.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
names = sys.argv[1:] or ["c2", "c3-zipf0.6", "c3-zipf1.0", "c3-zipf1.2", "c3-zipf1.5", "c4-exp1e-5", "c4-exp1e-7",
                         "c4-bexp"]
dev = torch.device("cuda", 0)
for name in names:
    cfgd = dict(bench.CONFIGS[name])
    n = cfgd["n"]
    k, _ = bench.gen_device(dict(cfgd, vb=0), n, 1000, dev)
    kh = k.cpu().numpy().view("uint32" if cfgd["kb"] == 4 else "uint64").copy()
    del k
    torch.cuda.empty_cache()
    t0 = time.time()
    rep = ora.sort_inplace(kh, None, "dt", report=True, seed=0)
    res[name] = {"n": n, "D": rep["records_distributed"], "levels": rep["levels"],
                 "level_mass": rep["level_mass"], "heavy_records_removed": rep["heavy_records_removed"],
                 "skipped_bits": rep["skipped_bits"], "oracle_s": round(time.time() - t0, 1),
                 "threads": ora.max_threads(),
                 "input": "bench.py gen_device(config, n, seed=1000, cuda:0) — the bench's rank-0 input"}
    print(name, res[name]["D"], res[name]["oracle_s"], flush=True)
    json.dump(res, open(out_path, "w"), indent=1)
