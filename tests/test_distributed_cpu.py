"""Multi-process host logic on CPU (gloo, world_size 2): the exact 128-bit all-reduce of
the counters and the start-vertex partition rule.  The device side of the N > 1 path
(bbc_opts.part_index / part_count) is covered by tests/test_gpu_parity.py."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2601_17707_b200.distributed import allreduce_counts, from_limbs, partition_task_indices, to_limbs

VALUES = {0: (2**64 - 5, 7), 1: (9, 2**63 + 11)}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bal, unb = allreduce_counts(*VALUES[rank])
        q.put((rank, bal, unb))
    finally:
        dist.destroy_process_group()


def test_limbs_roundtrip():
    for x in (0, 1, 2**32 - 1, 2**64 - 1, 2**64, 2**100 + 12345):
        assert from_limbs(to_limbs([x, 3])) == [x, 3]
    with pytest.raises(ValueError):
        to_limbs([-1])


def test_partition_rule_covers_every_task_once():
    for n in (0, 1, 7, 100, 1001):
        for parts in (1, 2, 3, 8):
            allidx = np.concatenate([partition_task_indices(n, p, parts) for p in range(parts)])
            assert sorted(allidx.tolist()) == list(range(n))
    with pytest.raises(ValueError):
        partition_task_indices(10, 2, 2)


def test_gloo_allreduce_exact_past_64_bits():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (VALUES[0][0] + VALUES[1][0], VALUES[0][1] + VALUES[1][1])
    assert want[0] > 2**64 - 1  # exercises the carry into the third limb
    for _, bal, unb in results:
        assert (bal, unb) == want


def _gather_worker(rank: int, world: int, port: int, m: int, q):
    import torch.distributed as dist

    from paper_2601_17707_b200.distributed import gather_edges, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        u = rng.integers(0, 1000, m).astype(np.int32)
        v = rng.integers(0, 1000, m).astype(np.int32)
        s = np.where(rng.random(m) < 0.3, -1, 1).astype(np.int8)
        lo, hi = shard_bounds(m, rank, world)
        gu, gv, gs = gather_edges(m, u[lo:hi], v[lo:hi], s[lo:hi])
        q.put((rank, bool((gu.numpy() == u).all() and (gv.numpy() == v).all() and (gs.numpy() == s).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world, m", [(2, 1001), (3, 7), (2, 0)])
def test_gloo_shard_gather_rebuilds_the_edge_list(world, m):
    """Each rank holds only its shard; the all-gather gives every rank the whole list (the
    host side of the sharded-upload replication, distributed.gather_edges)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in results)


def test_shard_bounds_cover_the_edges():
    from paper_2601_17707_b200.distributed import shard_bounds

    for m in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            b = [shard_bounds(m, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == m
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
