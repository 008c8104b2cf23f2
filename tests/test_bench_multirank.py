"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): the
max-over-ranks device time and the whole-job weak-scaling throughput. The GPU
path runs the same functions over NCCL (one process per GPU, no collective
on the data path: requests are independent)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    mine = [10.0 + rank * 5.0, 20.0 - rank, 100.0 + rank]
    got = bench.max_over_ranks(mine, torch.device("cpu"))
    out[rank] = (got, bench.job_throughput(world, 4, 16416, got[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        got, value = out[r]
        assert got == [15.0, 20.0, 101.0]
        assert value == pytest.approx(2 * 4 * 16416 / 0.015)


def test_job_throughput_weak_scaling():
    import bench
    one = bench.job_throughput(1, 5, 16416, 250.0)
    eight = bench.job_throughput(8, 5, 16416, 250.0)
    assert eight == pytest.approx(8 * one)
