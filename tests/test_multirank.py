"""The N>1 bench path (independent replicas, one system per rank): the max-over-ranks timing and
the whole-job aggregation, run with world_size 2 over gloo on the CPU."""
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


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    t = 10.0 + 5.0 * rank  # rank-local device time (ms) of K steps
    ms = bench.max_over_ranks(t, world, device="cpu")
    E, K = 1000, 50
    value = world * E * K / (ms / 1e3)
    bench.barrier(world)
    q.put((rank, ms, value))
    dist.destroy_process_group()


def test_replicas_take_the_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get(timeout=5) for _ in range(2))
    assert [o[1] for o in out] == [15.0, 15.0]  # both ranks report the slowest
    assert out[0][2] == out[1][2] == pytest.approx(2 * 1000 * 50 / 0.015)
