"""The N > 1 path of bench.py on CPU (gloo, world size 2): every rank runs an
independent replica with its own seed, and the reported step time is the max over
ranks (replicas only, no collective on the data path)."""
import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c1", 8, 2)
    seed = bench.replica_seed(0, rank)
    _, b, _ = workloads.draw(cfg, 225, seed)
    t = bench.max_over_ranks(1.0 + rank)          # rank 1 is the slow one
    out.put((rank, t, seed, float(b[0])))
    dist.destroy_process_group()


def test_two_rank_replicas_max_time():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [r[1] for r in res] == [2.0, 2.0]          # both ranks see the max
    assert res[0][2] != res[1][2]                     # independent replicas
    assert res[0][3] != res[1][3]


def test_single_process_identity():
    import bench
    assert bench.max_over_ranks(3.5) == 3.5
