"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): the
max-over-ranks step time and the whole-job throughput aggregation."""
from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms_local = 10.0 + 5.0 * rank  # rank 1 is the slow one
    ms, value = bench.aggregate(ms_local, 1000, world, dist, "cpu")
    dist.barrier()
    q.put((rank, ms, value))
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms, value in res:
        assert ms == pytest.approx(15.0)  # the max over ranks, on every rank
        assert value == pytest.approx(1000 * world / 0.015)  # all ranks' units / max time


def test_single_rank_aggregate():
    import bench
    ms, value = bench.aggregate(4.0, 500, 1)
    assert ms == 4.0 and value == pytest.approx(500 / 0.004)
