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
