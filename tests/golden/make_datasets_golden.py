"""Writes tests/golden/datasets_golden.json from the REFERENCE's generators
and dataset writer (run here, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_datasets_golden.py

SHA-256 of the keys / payload bytes of gen.generate for every grid family at
two widths, of gen.generate_edges, and of a written ISRT file."""
import hashlib
import json
import os
import pathlib
import tempfile

import numpy as np
from dovetail.core import RecordArray
from dovetail.gen import DistSpec, generate, generate_edges, write_dataset

OUT = pathlib.Path(__file__).resolve().parent / "datasets_golden.json"
SPECS = [("uniform", 10.0), ("uniform", 1e9), ("exp", 1.0), ("exp", 7.0), ("zipf", 0.6), ("zipf", 1.2),
         ("bexp", 10.0), ("bexp", 300.0)]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


cases = []
for fam, p in SPECS:
    for bits in (32, 64):
        for n, seed in ((100_000, 0), (70_001, 5)):
            r = generate(DistSpec(fam, p, n, bits, seed))
            cases.append(dict(family=fam, param=p, n=n, bits=bits, seed=seed, keys=sha(r.keys), pays=sha(r.payloads)))
src, dst = generate_edges(1 << 16, 200_000, 1.0, 3)
edges = dict(vertices=1 << 16, edges=200_000, skew=1.0, seed=3, src=sha(src), dst=sha(dst))
files = []
with tempfile.TemporaryDirectory() as td:
    r = generate(DistSpec("zipf", 1.0, 5000, 32, 1))
    for pw in (0, 4, 8):
        path = os.path.join(td, f"f{pw}.isrt")
        rec = r if pw else RecordArray(r.keys)
        write_dataset(path, rec, payload_width=pw)
        files.append(dict(family="zipf", param=1.0, n=5000, bits=32, seed=1, payload_width=pw,
                          sha=hashlib.sha256(open(path, "rb").read()).hexdigest()))
OUT.write_text(json.dumps(dict(generate=cases, edges=edges, files=files), indent=1))
print(f"wrote {OUT}: {len(cases)} generate cases, {len(files)} files")
