"""B200-native DovetailSort (arXiv 2401.00710): stable MSD integer sort with
heavy-key buckets, running as hand-written sm_100a kernels behind a C ABI.

Drop-in for the reference package ``dovetail``
(/root/reference/pkg/src/dovetail/__init__.py:20-45)::

    from paper_2401_00710_b200 import RecordArray, SortConfig, dt_sort
    rec = RecordArray(keys_u32, values_u32)   # numpy or torch (host or CUDA)
    dt_sort(rec, SortConfig(seed=7))          # stable, in place, on the GPU
"""
from .core import InstrumentReport, RecordArray, SortConfig, ceil_log2, gamma_for, rng_stream
from .dtmerge import MergeStats, dt_merge
from .dtsort import dt_sort, plain_msd_sort
from .parallel import num_workers, set_num_workers

__version__ = "0.1.0"

__all__ = [
    "InstrumentReport",
    "MergeStats",
    "RecordArray",
    "SortConfig",
    "ceil_log2",
    "dt_merge",
    "dt_sort",
    "gamma_for",
    "num_workers",
    "plain_msd_sort",
    "rng_stream",
    "set_num_workers",
    "__version__",
]
