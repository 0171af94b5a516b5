"""The N > 1 path end to end on a real device: two processes (gloo for the counter
all-reduce, both ranks on cuda:0 since this box has one GPU) each build the replicated
CSR, count their start-vertex partition with the CUDA kernel and all-reduce; the sum must
equal the single-process count bit for bit (distributed.count_partitioned, the code the
multi-GPU bench path mirrors)."""

import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, key: str, algo: str, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2601_17707_b200 import synth
    from paper_2601_17707_b200.distributed import count_partitioned

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.golden_config(key)
        u, v, s = synth.generate(cfg)
        q.put((rank, count_partitioned(cfg.n_u, cfg.n_v, u, v, s, device=0, algo=algo)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world, algo", [(2, "gbbc++"), (3, "gbbc")])
def test_partitioned_ranks_sum_to_the_whole(gpu, golden, world, algo):
    key = "2@0.05"
    rec = golden["configs"][key]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, key, algo, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, (bal, unb) in results:
        assert (bal, unb) == (rec["balanced"], rec["unbalanced"])


def test_in_process_multi_device_handle(gpu, golden):
    """bbc_multi_* (csrc/bbc_multi.cu): sharded upload, NCCL all-gather, replicated build,
    partition counts and one NCCL all-reduce -- on the devices this box has (one here, so
    the communicator has one rank; the partition / limb logic is the same for N)."""
    import numpy as np

    from paper_2601_17707_b200 import DuplicateEdgeError, IndexOutOfRangeError, _lib, synth

    key = "2@0.05"
    rec = golden["configs"][key]
    cfg = synth.golden_config(key)
    u, v, s = synth.generate(cfg)
    devs = list(range(_lib.device_count()))
    mg = _lib.MultiGraph(cfg.n_u, cfg.n_v, u, v, s, devs)
    try:
        assert mg.w_s == min(rec["w_u"], rec["w_v"])
        for algo in (_lib.ALGO_GBBC, _lib.ALGO_GBBCPP):
            r = mg.count(algo)
            assert (r.balanced, r.unbalanced) == (rec["balanced"], rec["unbalanced"])
            assert r.wedges == mg.w_s
    finally:
        mg.close()
    with pytest.raises(ValueError):
        _lib.MultiGraph(cfg.n_u, cfg.n_v, u, v, s, [0, 0])
    with pytest.raises(DuplicateEdgeError):
        _lib.MultiGraph(3, 3, np.array([0, 1, 0]), np.array([1, 2, 1]), np.array([1, 1, -1]), devs)
    with pytest.raises(IndexOutOfRangeError):
        _lib.MultiGraph(3, 3, np.array([0, 5]), np.array([1, 2]), np.array([1, 1]), devs)
    # the one-shot entry point
    import ctypes

    out = (ctypes.c_uint64 * 2)()
    st = _lib.Stats()
    d = (ctypes.c_int32 * len(devs))(*devs)
    uu, vv, ss = (np.ascontiguousarray(x) for x in (u, v, s))
    rc = _lib.load().bbc_count_multi(len(devs), d, cfg.n_u, cfg.n_v, cfg.m, uu.ctypes.data, vv.ctypes.data,
                                     ss.ctypes.data, _lib.SIDE_CHEAPER, None, out, ctypes.byref(st))
    assert rc == 0 and (out[0], out[1]) == (rec["balanced"], rec["unbalanced"])
