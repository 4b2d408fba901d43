"""Host test double for the device ops of distributed.dist_sort (numpy
stable partition / sort).  Test infrastructure only: used by
tests/test_distributed_gloo.py and by `bench.py --gloo-selftest` to run the
multi-rank exchange logic on CPU with gloo; never on a product path."""
import numpy as np
import torch


class HostOps:
    def sample(self, keys, gbase, count, seed):
        n = keys.numel()
        rng = np.random.default_rng(seed + gbase)
        pos = np.sort(rng.integers(0, n, size=count)) if n and count else np.empty(0, np.int64)
        kn = keys.numpy().view(np.uint32 if keys.element_size() == 4 else np.uint64)
        return kn[pos].copy(), pos.astype(np.uint64) + np.uint64(gbase)

    def partition(self, keys, vals, gbase, split_keys, split_idx):
        kn = keys.numpy().view(np.uint32 if keys.element_size() == 4 else np.uint64)
        gidx = np.arange(kn.shape[0], dtype=np.uint64) + np.uint64(gbase)
        dest = np.zeros(kn.shape[0], np.int64)
        for sk, si in zip(split_keys, split_idx):
            dest += (kn > sk) | ((kn == sk) & (gidx > si))
        order = np.argsort(dest, kind="stable")
        G = len(split_keys) + 1
        counts = np.bincount(dest, minlength=G)
        ok = torch.from_numpy(keys.numpy()[order].copy())
        ov = None if vals is None else torch.from_numpy(vals.numpy()[order].copy())
        return ok, ov, [int(c) for c in counts]

    def sort(self, keys, vals):
        kn = keys.numpy().view(np.uint32 if keys.element_size() == 4 else np.uint64)
        order = np.argsort(kn, kind="stable")
        keys.copy_(torch.from_numpy(keys.numpy()[order].copy()))
        if vals is not None:
            vals.copy_(torch.from_numpy(vals.numpy()[order].copy()))

    def empty_like(self, t, n):
        return torch.empty(int(n), dtype=t.dtype)
