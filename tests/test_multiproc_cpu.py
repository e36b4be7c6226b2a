"""The N>1 path of bench.py (one process per GPU, replicas only) on CPU: two gloo ranks
exercise the max-over-ranks device clock and the weak-scaling whole-job value."""

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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    ms = 10.0 + 5.0 * rank  # rank 1 is the slow one
    got = bench.reduce_max_ms(ms, dist, torch.device("cpu"))
    val = bench.weak_scaling_value(1 << 20, 4, world, got)
    dist.barrier()
    out[rank] = (got, val)
    dist.destroy_process_group()


def test_two_rank_gloo_max_and_weak_scaling():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0][0] == pytest.approx(15.0) and out[1][0] == pytest.approx(15.0)
    assert out[0][1] == pytest.approx((1 << 20) * 4 * 2 / 0.015)


def test_single_rank_no_dist():
    import bench

    assert bench.reduce_max_ms(3.5, None, None) == 3.5
