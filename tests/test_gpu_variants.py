"""GPU parity of the alternative code paths, each in a fresh process (the
switches are read once per process): the look-back scatter (DTS_WC=0) and
the forced-repair build (every tile / span goes through the order repair
path, libdts_fixup.so)."""
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2401_00710_b200" / "_lib"

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import cases
from oracle import oracle as ora
from paper_2401_00710_b200 import RecordArray, dt_sort, plain_msd_sort
bad = 0
for kb, vb in ((4, 4), (8, 8), (4, 0)):
    for dist in ("full", "few", "zipf", "planted", "bexp", "sorted"):
        for n in (4353, 300_001):
            rng = np.random.default_rng(n + kb * 3 + vb)
            keys = cases._dist(dist, n, kb * 8, rng)
            vdt = {{0: None, 4: np.uint32, 8: np.uint64}}[vb]
            vals = None if vdt is None else np.arange(n).astype(vdt)
            wk, wv = ora.reference_sort(keys, vals)
            for fn in (dt_sort, plain_msd_sort):
                rec = RecordArray(keys.copy(), None if vals is None else vals.copy())
                fn(rec)
                ok = np.array_equal(rec.keys, wk) and (vals is None or np.array_equal(rec.payloads, wv))
                if not ok:
                    bad += 1
                    print("MISMATCH", kb, vb, dist, n, fn.__name__)
print("bad", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("variant", ["lookback", "fixup"])
def test_gpu_variant_paths_match_oracle(variant):
    env = dict(os.environ)
    if variant == "lookback":
        env["DTS_WC"] = "0"
    else:
        lib = LIB / "libdts_fixup.so"
        if not lib.exists():
            pytest.skip("libdts_fixup.so not built")
        env["DTS_LIB"] = str(lib)
    code = SCRIPT.format(root=str(ROOT), tests=str(ROOT / "tests" / "golden"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
