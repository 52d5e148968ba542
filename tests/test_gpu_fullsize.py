"""Parity at BASELINE.json's full sizes, through size-independent properties
(the oracle cannot run these sizes in test time):

* configs[2] N = 2^24: the single-device engine and the same filter split
  into 4 shards give bit-identical ancestors and summaries -- every shard is
  a subtree of the reference's adder tree (prefix_sum.py:46-91) -- and the
  run is repeatable, indices in range, quantiles ordered, means inside the
  quantile band;
* configs[3] N = 2^27 (one B200 holds it): the single engine against 8
  shards, summaries only (a [T, 2^27] index array is 1 GiB per step)."""
import numpy as np
import pytest

import paper_1212_1639_b200 as P

pytestmark = pytest.mark.gpu


def _y(t_len, seed=0):
    _, y = P.simulate(P.TrendNoiseModel(), t_len, P.RngStream(seed, P.rng.AUX_STREAM_BASE + 1))
    return y


def _properties(o, n):
    q = o.filtered_quantiles
    assert (q[:, 0] <= q[:, 1]).all() and (q[:, 1] <= q[:, 2]).all()
    for nm in ("sigma2", "tau2"):
        s = o.param_posterior[nm]
        assert (np.diff(s.quantiles, axis=1) >= 0).all()
        assert ((s.quantiles[:, 0] <= s.mean) & (s.mean <= s.quantiles[:, 4])).all()
        assert (s.sd > 0).all()
    if o.resampled_indices is not None:
        assert o.resampled_indices.min() >= 1 and o.resampled_indices.max() <= n


def _same_summaries(a, b):
    np.testing.assert_allclose(a.filtered_mean, b.filtered_mean, rtol=1e-12, atol=1e-13)
    assert np.array_equal(a.filtered_quantiles, b.filtered_quantiles)
    for nm in ("sigma2", "tau2"):
        np.testing.assert_allclose(a.param_posterior[nm].mean, b.param_posterior[nm].mean, rtol=1e-12)
        np.testing.assert_allclose(a.param_posterior[nm].sd, b.param_posterior[nm].sd, rtol=1e-9)
        assert np.array_equal(a.param_posterior[nm].quantiles, b.param_posterior[nm].quantiles)


def test_configs2_full_size_shard_invariance(gpu):
    n, y = 1 << 24, _y(4)
    with P.Backend("cuda") as b:
        one = P.run_particle_learning(P.Priors(), y, n, seed=0, backend=b, keep_indices=True)
        again = P.run_particle_learning(P.Priors(), y, n, seed=0, backend=b, keep_indices=True)
    with P.Backend("cuda", shards=4) as b:
        four = P.run_particle_learning(P.Priors(), y, n, seed=0, backend=b, keep_indices=True)
    _properties(one, n)
    assert np.array_equal(one.resampled_indices, again.resampled_indices)
    assert np.array_equal(one.resampled_indices, four.resampled_indices)
    _same_summaries(one, four)
    _same_summaries(one, again)


def test_configs3_full_size_single_device_vs_8_shards(gpu):
    n, y = 1 << 27, _y(3)
    with P.Backend("cuda") as b:
        one = P.run_particle_learning(P.Priors(), y, n, seed=0, backend=b)
    with P.Backend("cuda", shards=8) as b:
        eight = P.run_particle_learning(P.Priors(), y, n, seed=0, backend=b)
    _properties(one, n)
    _same_summaries(one, eight)
