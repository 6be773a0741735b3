"""The N > 1 host logic of bench.py on CPU (gloo, world_size 2, 127.0.0.1):
replicas only, so the only cross-rank step is the aggregation of the timed
region — max over ranks of the device time, sum of the iterations."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = [12.5, 20.0][rank]
    iters = [48, 50][rank]
    t, k = bench.reduce_over_ranks(ms, iters, torch.device("cpu"))
    out[rank] = (t, k)
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_over_ranks_gloo_two_ranks():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        assert res[r] == (20.0, 98)   # max time, summed iterations, on every rank
