"""N > 1 host logic of bench.py on CPU (gloo, world_size 2): weak scaling = distinct
collections per rank, step time = max over ranks, whole-job throughput."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


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
    try:
        local_ms = [12.5, 20.0][rank]
        mx = bench.reduce_max_ms(local_ms, "cpu", world)
        v = bench.weak_throughput(100, world, mx)
        seeds = bench.rank_seeds(4, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, seeds)
        q.put((rank, mx, v, gathered))
    finally:
        dist.destroy_process_group()


def test_two_rank_timing_and_seeds():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, v, gathered in res:
        assert mx == 20.0                       # the slowest rank defines the step
        assert v == pytest.approx(100 * 2 / 0.020)
        assert gathered[0] != gathered[1]       # distinct collections / query sets per rank
        assert gathered[0] == bench.rank_seeds(4, 0)


def test_single_rank_is_identity():
    assert bench.reduce_max_ms(7.0, "cpu", 1) == 7.0
    assert bench.weak_throughput(100, 1, 10.0) == pytest.approx(10000.0)
