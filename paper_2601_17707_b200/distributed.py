"""Multi-GPU counting: one process per GPU, start vertices partitioned, one all-reduce.

SURVEY.md 8(e): every rank holds the replicated device CSR, counts the anchors of its
partition (task indices part, part + P, part + 2P, ... of the dispatch order -- the
same mapping the kernel applies through bbc_opts.part_index / part_count), and the
per-rank (balanced, unbalanced) are summed with a single all-reduce.  The fork-pool
analogue in the reference is count_balanced_parallel's exact integer sum of worker
subtotals (pkg/src/bbcount/buckets.py:236-243).

The all-reduce carries each 128-bit count as four 32-bit limbs in int64 lanes, so the
sum is exact for up to 2^31 ranks with either backend (NCCL over NVLink on GPUs, gloo in
the CPU tests) and overflow past 2^64 - 1 is detected after the reduction.
"""

from __future__ import annotations

import numpy as np

from .errors import CountOverflowError, U64_MAX

_LIMBS = 4  # 4 x 32 bits = 128 bits per count


def partition_task_indices(ntasks: int, part: int, parts: int) -> np.ndarray:
    """Dispatch-order indices handled by partition ``part`` (mirrors k_count's gidx)."""
    if not 0 <= part < parts:
        raise ValueError("part must lie in [0, parts)")
    return np.arange(part, ntasks, parts, dtype=np.int64)


def to_limbs(values: list[int]) -> list[int]:
    out = []
    for x in values:
        if x < 0 or x >= 1 << (32 * _LIMBS):
            raise ValueError("count outside the 128-bit range")
        out += [(x >> (32 * i)) & 0xFFFFFFFF for i in range(_LIMBS)]
    return out


def from_limbs(limbs: list[int]) -> list[int]:
    vals = []
    for j in range(0, len(limbs), _LIMBS):
        vals.append(sum(int(limbs[j + i]) << (32 * i) for i in range(_LIMBS)))
    return vals


def allreduce_counts(balanced: int, unbalanced: int, group=None, device=None) -> tuple[int, int]:
    """Exact sum of (balanced, unbalanced) over the ranks of ``group``."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(to_limbs([balanced, unbalanced]), dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    bal, unb = from_limbs(t.tolist())
    return bal, unb


def count_partitioned(n_u: int, n_v: int, u, v, s, group=None, device: int | None = None, algo: str = "gbbc++",
                      check_overflow: bool = True) -> tuple[int, int]:
    """(balanced, unbalanced) of the whole graph from every rank of ``group``.

    Each rank builds the device CSR from the same host arrays (replicated), counts its
    start-vertex partition on ``device`` (default: LOCAL_RANK) and joins the all-reduce.
    """
    import os

    import torch
    import torch.distributed as dist

    from . import _lib

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    g = _lib.DeviceGraph.from_host(n_u, n_v, u, v, s, device)
    try:
        code = _lib.ALGO_GBBCPP if algo == "gbbc++" else _lib.ALGO_GBBC
        r = g.count(code, part_index=rank, part_count=world)
    finally:
        g.close()
    bal, unb = r.balanced, r.unbalanced
    if world > 1:
        backend = dist.get_backend(group)
        dev = torch.device("cuda", device) if backend == "nccl" else None
        bal, unb = allreduce_counts(bal, unb, group, dev)
    if check_overflow and (bal > U64_MAX or unb > U64_MAX):
        raise CountOverflowError("butterfly count exceeded 64-bit range")
    return bal, unb
