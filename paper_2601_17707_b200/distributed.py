"""Multi-GPU counting: one process per GPU, start vertices partitioned, one all-reduce.

SURVEY.md 8(e): every rank holds the replicated device CSR, counts the anchors of its
partition (task indices part, part + P, part + 2P, ... of the dispatch order -- the
same mapping the kernel applies through bbc_opts.part_index / part_count), and the
per-rank (balanced, unbalanced) are summed with a single all-reduce.  The fork-pool
analogue in the reference is count_balanced_parallel's exact integer sum of worker
subtotals (pkg/src/bbcount/buckets.py:236-243).

Replication without N host uploads: rank r uploads only edge shard r (ceil(m / P)
edges), the shards are all-gathered over NVLink (NCCL all_gather_into_tensor, 9 B per
edge), and every rank builds the CSR from the gathered device arrays
(bbc_graph_create_device).  The build is a few ms of device kernels that run on all
ranks at once, so replicating it costs no wall time, while the host->device traffic per
rank drops to 1/P of the edge list.

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


def shard_bounds(m: int, rank: int, world: int) -> tuple[int, int]:
    """Edge range [lo, hi) of rank's shard: ceil(m / world) edges each (the last may be short)."""
    if not 0 <= rank < world:
        raise ValueError("rank must lie in [0, world)")
    chunk = -(-m // world) if m else 0
    lo = min(m, rank * chunk)
    return lo, min(m, lo + chunk)


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


def gather_edges(m: int, shard_u, shard_v, shard_s, group=None, device=None):
    """Every rank's shard -> the whole edge list on every rank (one all-gather per array).

    ``shard_*`` are this rank's edges [lo, hi) of shard_bounds (host arrays or tensors);
    with ``device`` (NCCL) the result lives on that GPU, else on the host (gloo).  Returns
    torch tensors (int32, int32, int8) of length m.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(m, rank, world)
    chunk = -(-m // world) if m else 0
    out = []
    for x, dt in ((shard_u, torch.int32), (shard_v, torch.int32), (shard_s, torch.int8)):
        src = torch.as_tensor(np.ascontiguousarray(x) if isinstance(x, np.ndarray) else x)
        if src.numel() != hi - lo:
            raise ValueError(f"rank {rank}: shard has {src.numel()} edges, expected {hi - lo}")
        shard = torch.zeros(chunk, dtype=dt, device=device)
        if hi > lo:
            shard[: hi - lo].copy_(src.to(dt), non_blocking=True)
        full = torch.empty(chunk * world, dtype=dt, device=device)
        if world > 1:
            dist.all_gather_into_tensor(full, shard, group=group)
        else:
            full.copy_(shard)
        out.append(full[:m])
    return tuple(out)


def build_replicated(n_u: int, n_v: int, m: int, shard_u, shard_v, shard_s, device: int, group=None,
                     side_rule: int | None = None):
    """Device CSR of the whole graph on ``device`` from this rank's edge shard (NCCL group).

    Returns (DeviceGraph, gathered tensors) -- keep the tensors alive until the graph is
    built (bbc_graph_create_device reads them; it copies what it keeps)."""
    import torch

    from . import _lib

    dev = torch.device("cuda", device)
    du, dv, ds = gather_edges(m, shard_u, shard_v, shard_s, group, dev)
    torch.cuda.synchronize(dev)  # the build runs on the library's own stream
    rule = _lib.SIDE_CHEAPER if side_rule is None else side_rule
    g = _lib.DeviceGraph.from_device_ptrs(n_u, n_v, m, du.data_ptr(), dv.data_ptr(), ds.data_ptr(), device, rule)
    return g, (du, dv, ds)


def count_partitioned(n_u: int, n_v: int, u, v, s, group=None, device: int | None = None, algo: str = "gbbc++",
                      check_overflow: bool = True) -> tuple[int, int]:
    """(balanced, unbalanced) of the whole graph from every rank of ``group``.

    Rank r contributes edge shard r of the host arrays; the shards are all-gathered (on
    the GPU with NCCL, on the host with gloo), every rank builds the device CSR, counts
    its start-vertex partition on ``device`` (default: LOCAL_RANK) and joins the
    all-reduce.
    """
    import os

    import torch
    import torch.distributed as dist

    from . import _lib

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    m = len(u)
    lo, hi = shard_bounds(m, rank, world)
    nccl = world > 1 and dist.get_backend(group) == "nccl"
    if nccl:
        g, _keep = build_replicated(n_u, n_v, m, u[lo:hi], v[lo:hi], s[lo:hi], device, group)
    else:
        tu, tv, ts = gather_edges(m, u[lo:hi], v[lo:hi], s[lo:hi], group, None)
        g = _lib.DeviceGraph.from_host(n_u, n_v, tu.numpy(), tv.numpy(), ts.numpy(), device)
    try:
        code = _lib.ALGO_GBBCPP if algo == "gbbc++" else _lib.ALGO_GBBC
        r = g.count(code, part_index=rank, part_count=world)
    finally:
        g.close()
    bal, unb = r.balanced, r.unbalanced
    if world > 1:
        dev = torch.device("cuda", device) if nccl else None
        bal, unb = allreduce_counts(bal, unb, group, dev)
    if check_overflow and (bal > U64_MAX or unb > U64_MAX):
        raise CountOverflowError("butterfly count exceeded 64-bit range")
    return bal, unb
