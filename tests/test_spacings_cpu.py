"""K7 (spacings) host logic on CPU: the oracle restatement against the
reference's exact semantics, and the sharded exchange -- two gloo ranks each
scan their half of the slots and exchange only their exponential totals
(torch.distributed all_gather), giving the same ordered uniforms as one scan."""
import os
import socket

import numpy as np

from oracle import restate as R


def _words(n, seed, t):
    return R.block_words(seed, np.arange(n, dtype=np.uint64), t)[3]


def test_ordered_uniforms_are_sorted_uniform_order_statistics():
    n = 1 << 14
    u = R.spacings_uniforms(_words(n, 3, 1), 3, 1)
    assert (np.diff(u) >= 0).all() and u[0] > 0 and u[-1] < 1
    # order statistics of n uniforms: E[U_(k)] = k / (n + 1); the max gap is O(log n / n)
    k = np.arange(1, n + 1)
    assert np.max(np.abs(u - k / (n + 1))) < 5 / np.sqrt(n)


def test_spacings_ancestors_are_multinomial_and_ordered():
    # exact multinomial like the reference's `sorted` (resampling.py:57-67):
    # pooled counts over steps match n w / W (chi-square), zero weights never chosen
    rng = np.random.default_rng(1)
    n, steps = 2048, 60
    w = rng.exponential(size=n)
    w[rng.random(n) < 0.1] = 0.0
    q = R.tree_cdf(w)
    cuts = R.cut_points(q)
    counts = np.zeros(n)
    for t in range(1, steps + 1):
        idx = R.spacings_indices(q, cuts, _words(n, 9, t), 9, t)
        assert (np.diff(idx) >= 0).all()
        counts += np.bincount(idx - 1, minlength=n)
    assert counts[w == 0].sum() == 0
    live = w > 0
    expect = steps * n * w / w.sum()
    chi2 = float(np.sum((counts[live] - expect[live]) ** 2 / expect[live]))
    dof = int(live.sum()) - 1
    assert abs((chi2 - dof) / np.sqrt(2 * dof)) < 4


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, n, q_out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ns = n // world
    words = _words(n, 5, 2)[rank * ns:(rank + 1) * ns]
    mine = torch.tensor([float(np.sum(-np.log(R.unit_open(words))))], dtype=torch.float64)
    parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, mine)  # the only exchange: one total per shard
    totals = [float(p.item()) for p in parts]
    q_out.put((rank, R.spacings_uniforms_shard(words, totals, rank, 5, 2)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_gloo_ranks_exchange_only_their_totals():
    import torch.multiprocessing as mp

    n, world = 1 << 13, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    u = np.concatenate([got[r] for r in range(world)])
    one = R.spacings_uniforms(_words(n, 5, 2), 5, 2)
    assert (np.diff(u) >= 0).all()
    # same ordered uniforms up to the scan's rounding (a few 2^-53 units)
    assert np.max(np.abs(u - one)) < 1e-12
