"""The multi-GPU driver's device path (CudaOps: sample, dts_partition,
NCCL all_to_all_single, dts_sort) on the one GPU of the box: world size 1
over NCCL in a fresh process.  The exchange logic with world size 2 is
covered on CPU (tests/test_distributed_gloo.py)."""
import os
import pathlib
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, {root!r})
from oracle import oracle as ora
from paper_2401_00710_b200.distributed import dist_sort
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
rng = np.random.default_rng(4)
for kb, n in ((4, 1_000_003), (8, 300_000)):
    dt = np.uint32 if kb == 4 else np.uint64
    keys = rng.integers(0, 10**6, size=n).astype(dt)
    keys[: n // 5] = 77
    rng.shuffle(keys)
    vals = np.arange(n, dtype=dt)
    wk, wv = ora.reference_sort(keys, vals)
    tk = torch.from_numpy(keys.view(np.int32 if kb == 4 else np.int64)).cuda()
    tv = torch.from_numpy(vals.view(np.int32 if kb == 4 else np.int64)).cuda()
    rk, rv, st = dist_sort(tk, tv)
    ok = np.array_equal(rk.cpu().numpy().view(dt), wk) and np.array_equal(rv.cpu().numpy().view(dt), wv)
    assert ok and st.n_local_out == n and st.bytes_sent_remote == 0, (kb, n)
    assert st.exchange_ms > 0.0 and st.local_distributed >= n, (st.exchange_ms, st.local_distributed)
dist.destroy_process_group()
print("ok")
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gpu_dist_sort_world1_nccl():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT))], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
