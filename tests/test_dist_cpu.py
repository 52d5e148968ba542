"""Host side of the one-process-per-GPU sharded run (distributed.py), on CPU
over gloo: slot ownership, Backend(process_group=...) validation, and the
output publication every rank performs after the device loop (rank 0's
summaries broadcast, every rank's slots of the per-particle outputs
gathered), with two real gloo ranks."""
import os
import socket

import numpy as np
import pytest

import paper_1212_1639_b200 as P
from paper_1212_1639_b200.distributed import ShardRank, shard_slots


def test_shard_slots_partition_the_particles():
    n = 1 << 14
    for world in (1, 2, 4, 8):
        cover = np.concatenate([np.arange(*shard_slots(n, r, world)) for r in range(world)])
        assert np.array_equal(cover, np.arange(n))
    with pytest.raises(ValueError):
        shard_slots(n, 0, 3)


def test_process_group_needs_initialised_torch_distributed():
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    with pytest.raises(ValueError):
        P.Backend("cuda", process_group=True)
    with pytest.raises(ValueError):
        P.Backend("cuda", shards=2, process_group=True)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, result):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = P.Backend("cuda", device=0, process_group=True)
    assert (b.rank, b.world, b.distributed) == (rank, world, True)
    t_len, n = 5, 64
    ns = n // world
    # what each rank's device loop leaves behind: rank 0 the summaries, every
    # rank its own slots of indices and final particles
    arrays = {"filtered_mean": np.zeros(t_len), "sigma2_quantiles": np.zeros((t_len, 5)),
              "indices": np.zeros((t_len, n), dtype=np.int64), "final_states": np.zeros(n)}
    local = {"indices": (np.arange(t_len * ns, dtype=np.int64).reshape(t_len, ns) + 1000 * rank),
             "final_states": np.full(ns, float(rank))}
    if rank == 0:
        arrays["filtered_mean"][:] = np.arange(t_len) * 0.5
        arrays["sigma2_quantiles"][:] = np.arange(t_len * 5).reshape(t_len, 5)
        local["filtered_mean"] = arrays["filtered_mean"]
        local["sigma2_quantiles"] = arrays["sigma2_quantiles"]
    sr = ShardRank.__new__(ShardRank)
    sr.dist, sr.group, sr.rank, sr.world, sr.nccl, sr.device, sr.h = dist, None, rank, world, False, 0, None
    sr._publish(arrays, local, t_len, ns)
    result.put((rank, {k: v.tobytes() for k, v in arrays.items()}))
    dist.barrier()
    dist.destroy_process_group()


def test_two_gloo_ranks_publish_the_full_outputs():
    import torch.multiprocessing as mp

    world, t_len, n = 2, 5, 64
    ns = n // world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want_idx = np.concatenate([np.arange(t_len * ns).reshape(t_len, ns) + 1000 * r for r in range(world)], axis=1)
    for r in range(world):
        a = got[r]
        assert np.array_equal(np.frombuffer(a["filtered_mean"]), np.arange(t_len) * 0.5)
        assert np.array_equal(np.frombuffer(a["sigma2_quantiles"]), np.arange(t_len * 5, dtype=float))
        assert np.array_equal(np.frombuffer(a["indices"], dtype=np.int64).reshape(t_len, n), want_idx)
        assert np.array_equal(np.frombuffer(a["final_states"]), np.repeat([0.0, 1.0], ns))


def _agree_main(rank, world, port, result):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sr = ShardRank.__new__(ShardRank)
    sr.dist, sr.group, sr.rank, sr.world, sr.nccl, sr.device, sr.h = dist, None, rank, world, False, 0, None
    seen = []
    # (a) only rank 1 fails: every rank raises its error (no rank left in a collective)
    # (b) only rank 0 fails with a step-carrying degeneracy: rank 1 rebuilds it with the step
    # (c) nobody fails: no exception
    cases = [(1, P.NonFiniteWeightError("bad weight on rank 1")), (0, P.AllWeightsZeroError(step=3)), (None, None)]
    for who, exc in cases:
        try:
            sr._raise_agreed(exc if rank == who else None)
            seen.append(None)
        except Exception as e:  # noqa: BLE001
            seen.append((type(e).__name__, str(e), getattr(e, "step", None)))
    result.put((rank, seen))
    dist.barrier()
    dist.destroy_process_group()


def test_two_gloo_ranks_agree_on_failure():
    """a failure on any one rank is raised on every rank, rebuilt
    from the failing rank's type, message and step."""
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_agree_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0] == got[1]
    assert got[0][0] == ("NonFiniteWeightError", "bad weight on rank 1", None)
    assert got[0][1] == ("AllWeightsZeroError", "all particle weights are zero (at time step 3)", 3)
    assert got[0][2] is None
