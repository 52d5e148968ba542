"""Independent Monte Carlo replications of one filter (BASELINE configs[4]:
the paper's timing experiment, PAPER.md:600-618 -- R replications of the
N-particle particle-learning run, replication r seeded with r).

Replications are embarrassingly parallel: no data-path collective.  On one
device they reuse one resident engine (the device buffers, gamma tables and
kernel configuration are built once); across devices / ranks each takes the
seeds ``seeds[rank::world]`` ("replicas only")."""

from __future__ import annotations

from .backend import Backend
from .filtering import run_particle_filter, run_particle_learning
from .models import Priors


def rank_seeds(seeds, rank, world):
    """The replications one rank of ``world`` runs (round robin)."""
    return list(seeds)[rank::world]


def run_replications(spec, y, n, seeds, backend=None, **kwargs):
    """Run one filter per seed and return the list of FilterOutput.

    ``spec`` is a ``Priors`` (particle learning) or a ``TrendNoiseModel``
    (known parameters); the remaining keywords are those of
    run_particle_learning / run_particle_filter.  A caller-supplied
    ``backend`` keeps its engine (and device) across the replications."""
    fn = run_particle_learning if isinstance(spec, Priors) else run_particle_filter
    own = backend is None
    if own:
        backend = Backend()
    try:
        return [fn(spec, y, n, seed=int(s), backend=backend, **kwargs) for s in seeds]
    finally:
        if own:
            backend.close()


__all__ = ["rank_seeds", "run_replications"]
