"""Particle-sharded runs: one filter split over G shards must be
bit-identical to the single-device engine in ancestors and final particles
(every shard is a subtree of the reference's adder tree, prefix_sum.py:46-91),
with moments equal to rounding and the same weighted quantiles.  The shards
share one B200 here; the exchange and the cross-shard resampling reads take
the same peer-memory path they take across NVLink-connected GPUs."""

import numpy as np
import pytest

import paper_1212_1639_b200 as P

pytestmark = pytest.mark.gpu


def _series(t_len, seed=1):
    _, y = P.simulate(P.TrendNoiseModel(), t_len, P.RngStream(seed, P.rng.AUX_STREAM_BASE + 1))
    return y


def _run(fn, spec, y, n, shards, **kw):
    with P.Backend("cuda", shards=shards) as b:
        return fn(spec, y, n, seed=5, backend=b, keep_indices=True, keep_final=True, **kw)


def _assert_same(a, b, learn=True, quantiles=True):
    assert np.array_equal(a.resampled_indices, b.resampled_indices)
    assert np.array_equal(a.final_particles.states, b.final_particles.states)
    np.testing.assert_allclose(a.filtered_mean, b.filtered_mean, rtol=1e-12, atol=1e-13)
    if learn:
        for name in ("sigma2", "tau2"):
            assert np.array_equal(getattr(a.final_particles.params, name), getattr(b.final_particles.params, name))
            np.testing.assert_allclose(a.param_posterior[name].mean, b.param_posterior[name].mean, rtol=1e-12)
            np.testing.assert_allclose(a.param_posterior[name].sd, b.param_posterior[name].sd, rtol=1e-9)
            if quantiles:
                assert np.array_equal(a.param_posterior[name].quantiles, b.param_posterior[name].quantiles)
    if quantiles and a.filtered_quantiles is not None:
        assert np.array_equal(a.filtered_quantiles, b.filtered_quantiles)


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_sharded_learning_matches_single_device(gpu, shards):
    y = _series(24)
    n = 1 << 15
    one = _run(P.run_particle_learning, P.Priors(), y, n, 1)
    many = _run(P.run_particle_learning, P.Priors(), y, n, shards)
    _assert_same(one, many)


def test_sharded_filter_matches_single_device(gpu):
    y = _series(16, seed=2)
    model = P.TrendNoiseModel()
    one = _run(P.run_particle_filter, model, y, 1 << 14, 1)
    many = _run(P.run_particle_filter, model, y, 1 << 14, 4)
    _assert_same(one, many, learn=False)


def test_sharded_single_precision(gpu):
    y = _series(12, seed=3)
    one = _run(P.run_particle_learning, P.Priors(), y, 1 << 14, 1, precision="single")
    many = _run(P.run_particle_learning, P.Priors(), y, 1 << 14, 2, precision="single")
    _assert_same(one, many)


def test_sharded_large_against_rank_tables(gpu):
    """At N = 2^22 the single engine resolves ancestors with its L2-resident
    rank tables; two shards of 2^21 use the cross-shard cut tables."""
    y = _series(6, seed=4)
    n = 1 << 22
    one = _run(P.run_particle_learning, P.Priors(), y, n, 1, track_quantiles=False)
    many = _run(P.run_particle_learning, P.Priors(), y, n, 2, track_quantiles=False)
    assert np.array_equal(one.resampled_indices, many.resampled_indices)
    assert np.array_equal(one.final_particles.states, many.final_particles.states)
    np.testing.assert_allclose(one.filtered_mean, many.filtered_mean, rtol=1e-12)


def test_sharded_errors(gpu):
    y = _series(4)
    with pytest.raises(ValueError):
        _run(P.run_particle_learning, P.Priors(), y, 1 << 12, 2)  # < 4096 slots per shard
    with pytest.raises(NotImplementedError):
        with P.Backend("cuda", shards=2) as b:
            P.run_particle_learning(P.Priors(), y, 1 << 14, backend=b, store_particles=True)
