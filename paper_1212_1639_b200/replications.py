"""Independent Monte Carlo replications of one filter (BASELINE configs[4]:
the paper's timing experiment, PAPER.md:600-618 -- R replications of the
N-particle particle-learning run, replication r seeded with r).

Replications are embarrassingly parallel: no data-path collective.  On one
device they reuse one resident engine (the device buffers, gamma tables and
kernel configuration are built once); across devices / ranks each takes the
seeds ``seeds[rank::world]`` ("replicas only")."""

from __future__ import annotations

from .backend import Backend
from .filtering import run_batch, run_particle_filter, run_particle_learning
from .models import Priors


def rank_seeds(seeds, rank, world):
    """The replications one rank of ``world`` runs (round robin)."""
    return list(seeds)[rank::world]


def run_replications(spec, y, n, seeds, backend=None, concurrency=1, batch=1, **kwargs):
    """Run one filter per seed and return the list of FilterOutput (in seed
    order).

    ``batch`` > 1 runs that many replications per kernel launch sequence
    (filtering.run_batch / pf_engine_run_batch: R filters side by side in
    every launch, one tree per replication) -- the way to fill the B200 at
    N ~ 2^20, where one filter's per-step kernels are latency-bound.  Batched
    runs return the per-step summaries (``precision`` and
    ``track_quantiles`` are the only other keywords).

    ``spec`` is a ``Priors`` (particle learning) or a ``TrendNoiseModel``
    (known parameters); the remaining keywords are those of
    run_particle_learning / run_particle_filter.  A caller-supplied
    ``backend`` keeps its engine (and device) across the replications.
    ``concurrency`` > 1 runs that many engines at once on the device, each
    with its own CUDA streams, from as many host threads (the C ABI calls
    release the GIL): small filters (N ~ 2^20) leave the B200 partly idle
    one at a time."""
    fn = run_particle_learning if isinstance(spec, Priors) else run_particle_filter
    seeds = [int(s) for s in seeds]
    if batch > 1:
        extra = set(kwargs) - {"precision", "track_quantiles"}
        if extra:
            raise NotImplementedError(f"batched replications do not support {sorted(extra)}")
        own = backend is None
        if own:
            backend = Backend()
        try:
            out = []
            for lo in range(0, len(seeds), batch):
                out.extend(run_batch(spec, y, n, seeds[lo:lo + batch], backend=backend, **kwargs))
            return out
        finally:
            if own:
                backend.close()
    if concurrency <= 1 or len(seeds) <= 1:
        own = backend is None
        if own:
            backend = Backend()
        try:
            return [fn(spec, y, n, seed=s, backend=backend, **kwargs) for s in seeds]
        finally:
            if own:
                backend.close()
    from concurrent.futures import ThreadPoolExecutor

    device = backend.device if backend is not None else 0
    k = min(int(concurrency), len(seeds))
    backends = [Backend("cuda", device=device) for _ in range(k)]
    out = [None] * len(seeds)

    def lane(i):
        b = backends[i]
        for pos in range(i, len(seeds), k):
            out[pos] = fn(spec, y, n, seed=seeds[pos], backend=b, **kwargs)

    try:
        with ThreadPoolExecutor(k) as pool:
            for f in [pool.submit(lane, i) for i in range(k)]:
                f.result()
    finally:
        for b in backends:
            b.close()
    return out


__all__ = ["rank_seeds", "run_replications"]
