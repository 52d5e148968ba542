"""Host side of the particle-sharded run, on CPU.

The device kernels (csrc/cdf.cuh cdf_shard_total / cdf_top_shard) split the
reference's adder tree (prefix_sum.py:46-106) at shard boundaries: each shard
contributes one subtree total, every shard rebuilds the top levels and gets
its node value, carry and the stratum bounds of all shards.  These tests pin
that decomposition against the unsharded oracle bit for bit -- in one
process for G = 1..8, and across two gloo ranks exchanging only the shard
totals (torch.distributed all_gather), as the multi-GPU run does."""

import os
import socket

import numpy as np
import pytest

from oracle import restate as R


def _weights(n, seed, zero_fraction=0.0, dtype=np.float64):
    rng = np.random.default_rng(seed)
    w = rng.exponential(size=n)
    if zero_fraction:
        w[rng.random(n) < zero_fraction] = 0.0
    return w.astype(dtype)


def _sharded_q(w, G):
    n = len(w)
    ns = n // G
    parts = [w[g * ns:(g + 1) * ns] for g in range(G)]
    totals = np.array([R.forward_adder(p)[-1][0] for p in parts], dtype=w.dtype)
    root, nodes, carries, lend = R.shard_exchange(totals, n)
    q = np.concatenate([R.tree_cdf_shard(parts[g], g, nodes[g], carries[g], root, n) for g in range(G)])
    return q, lend


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_sharded_cdf_is_the_reference_tree(G, dtype):
    for seed, zf in ((0, 0.0), (1, 0.3), (2, 0.9)):
        w = _weights(1 << 12, seed, zf, dtype)
        q, lend = _sharded_q(w, G)
        ref = R.tree_cdf(w)
        assert q.dtype == ref.dtype
        assert np.array_equal(q, ref)
        # each shard's cut-table entries end where the next shard's begin
        bounds = np.ceil(ref * ref.dtype.type(len(w))).astype(np.int64)
        ns = len(w) // G
        assert np.array_equal(lend, bounds[ns - 1::ns])


def test_point_mass_in_one_shard():
    w = np.zeros(1 << 10)
    w[700] = 1.0
    q, lend = _sharded_q(w, 4)
    assert np.array_equal(q, R.tree_cdf(w))
    assert list(lend) == [0, 0, len(w), len(w)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, n, seed, result):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = _weights(n, seed)
    ns = n // world
    mine = w[rank * ns:(rank + 1) * ns]
    # the only CDF exchange: one subtree total per shard
    tot = torch.tensor([R.forward_adder(mine)[-1][0]], dtype=torch.float64)
    allt = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allt, tot)
    totals = np.array([t.item() for t in allt])
    root, nodes, carries, lend = R.shard_exchange(totals, n)
    q = R.tree_cdf_shard(mine, rank, nodes[rank], carries[rank], root, n)
    qt = torch.from_numpy(q)
    gathered = [torch.zeros(ns, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, qt)
    if rank == 0:
        result.put(np.concatenate([g.numpy() for g in gathered]).tobytes())
    dist.barrier()
    dist.destroy_process_group()


def test_two_gloo_ranks_exchange_only_totals():
    import torch.multiprocessing as mp

    n, seed, world = 1 << 12, 7, 2
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, n, seed, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    q = np.frombuffer(q_out.get(timeout=120), dtype=np.float64)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(q, R.tree_cdf(_weights(n, seed)))
