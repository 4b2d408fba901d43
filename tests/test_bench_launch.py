"""bench.py's multi-rank launch (VERDICT r1 "next" item 2): `python bench.py
--gpus N` outside torchrun re-executes itself as N ranks.  CPU: world size 2
over gloo with the host ops double; GPU: the NCCL path at world size 1 and
the refusal to run N ranks on fewer GPUs."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, timeout=timeout, env=env, cwd=ROOT)


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_self_launch_two_gloo_ranks():
    r = _bench("--gpus", "2", "--gloo-selftest", "--n", "3000")
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["records_out"] == 6000 and d["sorted"] is True


@pytest.mark.gpu
def test_self_launch_refuses_more_ranks_than_gpus():
    import torch

    n = torch.cuda.device_count()
    r = _bench("--gpus", str(n + 1), "--steps", "1", "--warmup", "3")
    assert r.returncode != 0 and "visible GPUs" in r.stderr


@pytest.mark.gpu
def test_force_dist_line_at_world_size_one():
    r = _bench("--gpus", "1", "--force-dist", "--n", str(10**7), "--steps", "2", "--warmup", "3",
               "--no-cpu-baseline", "--no-e2e")
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["roofline"]["bound"] == "hbm+nvlink"
