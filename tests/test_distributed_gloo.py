"""World-size-2 gloo test of the multi-GPU exchange logic on CPU
(SURVEY.md §8e).  The device kernels are replaced by a host test double
(numpy stable partition / sort) injected through `ops`; the splitter
choice, size exchange, record all-to-all and source-rank concatenation are
the product code in paper_2401_00710_b200/distributed.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_00710_b200.distributed import choose_splitters, dist_sort

from dist_hostops import HostOps


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys, vals = case
        n = keys.shape[0]
        lo, hi = rank * n // world, (rank + 1) * n // world
        kt = torch.from_numpy(keys[lo:hi].astype(np.int32 if keys.dtype == np.uint32 else np.int64))
        vt = torch.from_numpy(vals[lo:hi].astype(np.int32))
        rk, rv, st = dist_sort(kt, vt, ops=HostOps(), samples_per_rank=256, seed=3)
        q.put((rank, rk.numpy().copy(), rv.numpy().copy(), st.send_counts, st.recv_counts))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(keys, vals, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (keys, vals), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    return res


@pytest.mark.parametrize("dist_name", ["uniform", "heavy", "tiny"])
def test_two_rank_exchange_is_the_global_stable_sort(dist_name):
    rng = np.random.default_rng(11)
    n = {"uniform": 20_000, "heavy": 20_000, "tiny": 5}[dist_name]
    keys = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    if dist_name == "heavy":
        keys[rng.random(n) < 0.6] = 777  # one key holds ~60% of the records
    vals = np.arange(n, dtype=np.uint32)
    res = _run(keys, vals)
    got_k = np.concatenate([r[1].view(np.uint32) for r in res])
    got_v = np.concatenate([r[2].view(np.uint32) for r in res])
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(got_k, keys[order])
    assert np.array_equal(got_v, vals[order])
    # size exchange consistent: what rank a sends to b is what b receives from a
    assert res[0][3][1] == res[1][4][0] and res[1][3][0] == res[0][4][1]
    if dist_name == "heavy":
        # composite (key, index) splitters keep the ranks balanced
        sizes = [len(r[1]) for r in res]
        assert max(sizes) <= 0.65 * n


def test_choose_splitters_lexicographic():
    k = np.array([5, 5, 5, 1, 9], np.uint32)
    i = np.array([10, 2, 7, 0, 1], np.uint64)
    sk, si = choose_splitters(k, i, 2)
    # sorted pairs: (1,0) (5,2) (5,7) (5,10) (9,1) -> quantile 5//2 = 2 -> (5,7)
    assert sk.tolist() == [5] and si.tolist() == [7]
