"""bench.py's process plumbing on CPU: the max-over-ranks device time and
the barrier the multi-GPU runs use, across two gloo ranks (torchrun sets the
same environment variables), and the JSON contract of the reference arm's
line shape without a GPU."""

import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.barrier(world)
    m = bench.max_over_ranks(10.0 * (rank + 1), world)
    if rank == 0:
        q.put(m)
    dist.destroy_process_group()


def test_max_over_ranks_two_gloo_ranks():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    assert q.get(timeout=120) == 20.0
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0


def test_single_rank_helpers():
    import bench

    assert bench.max_over_ranks(3.5, 1) == 3.5
    bench.barrier(1)
    peak, kind = bench._peaks()
    assert peak > 1000 and kind in ("measured", "fallback")


def test_clock_sampler_without_nvidia_smi(monkeypatch):
    import bench

    monkeypatch.setenv("PATH", "/nonexistent")
    with bench.ClockSampler(0) as c:
        pass
    s = c.summary()
    assert "reasons" in s
