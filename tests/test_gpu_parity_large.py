"""Oracle parity on the benchmarked kernel path.

At N >= 2^21 the engine runs the fused-draws step kernel (draws computed in
the step kernel, csrc/step.cuh step_kernel<..., true>), strata rank-table
lookups (N >= 2^21) and the top tree in K2's last CTA -- the path bench.py
measures at configs[2].  These tests feed the reference's own noise draws
(oracle mode; tests/oracle_feed.py regenerates them with scipy exactly as
the reference does) and compare with the CPU oracle's run_loop
(oracle/restate.py, pinned to the reference's golden runs):

* ancestor indices of every step and the final particles: bit-identical;
* filtered mean, parameter mean and sd: within 1e-10 relative;
* weighted quantiles: equal.

Each test asserts through pf_engine_last_path that the benchmarked variant
actually ran.  The native-mode test checks the fused draws against the
separate draws kernel bit for bit (same tables, same Philox words), and the
tau2 = 0 test drives the weighted-quantile candidate window into overflow
(long runs of identical states after resampling) against the oracle.
"""

import numpy as np
import pytest

import paper_1212_1639_b200 as P
from oracle import restate as R
from oracle_feed import make_feed

pytestmark = pytest.mark.gpu

REL = 1e-10  # fp64 tolerance for sums evaluated in a different order


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def _engine(b):
    (eng,) = b._engines.values()
    return eng


def _check_against_oracle(out, ref, learn):
    assert np.array_equal(out.resampled_indices, ref["indices"])
    assert np.array_equal(out.final_particles.states, ref["final"]["states"])
    assert np.array_equal(out.filtered_quantiles, ref["filtered_quantiles"])
    assert np.max(np.abs(out.filtered_mean - ref["filtered_mean"])) <= REL * np.max(np.abs(ref["filtered_mean"]))
    if learn:
        fp = out.final_particles
        for nm, key in (("sigma2", "b_sigma"), ("tau2", "b_tau")):
            s = out.param_posterior[nm]
            assert np.array_equal(s.quantiles, ref[nm]["quantiles"]), nm
            assert _rel(s.mean, ref[nm]["mean"]) <= REL, nm
            assert _rel(s.sd, ref[nm]["sd"]) <= REL, nm
            assert np.array_equal(getattr(fp.suffstats, key), ref["final"][key]), nm
        assert np.array_equal(fp.params.sigma2, ref["final"]["sigma2"])
        assert np.array_equal(fp.params.tau2, ref["final"]["tau2"])


@pytest.mark.parametrize("k,t_len", [(22, 3), (24, 2)])
def test_oracle_mode_benchmarked_path(gpu, k, t_len):
    """configs[2]'s kernel path (N = 2^24 is configs[2] itself) against the
    CPU oracle fed the same draws."""
    n, seed = 1 << k, 11
    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 5)
    feed = make_feed(n, t_len, seed)
    with P.Backend("cuda") as b:
        out = P.run_particle_learning(P.Priors(), y, n, seed=seed, keep_indices=True, keep_final=True,
                                      track_quantiles=True, noise=feed, backend=b)
        path = _engine(b).last_path()
    assert path == {"fused_draws": True, "rank_tables": True, "fused_top": True}, path
    rec = {}
    ref = R.run_loop(y, n, seed, keep_indices=True, keep_final=True, feed=feed, record=rec)
    _check_against_oracle(out, ref, learn=True)
    # the ESS extension from the same per-CTA / per-shard weight sums
    ess = [float(w.sum()) ** 2 / float(np.dot(w, w)) for w in (rec["w"][t] for t in range(1, t_len + 1))]
    assert _rel(out.ess, ess) <= REL


def test_native_fused_draws_equal_draws_kernel(gpu, monkeypatch):
    """Native mode (device ndtri / gamma tables): the draws computed inside
    the step kernel equal the separate draws kernel's bit for bit, so the
    whole run -- ancestors, particles, summaries -- is identical."""
    n, t_len = 1 << 22, 4
    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 8)
    outs, paths = [], []
    for v in ("1", "0"):
        monkeypatch.setenv("PF_FUSED_DRAWS", v)
        with P.Backend("cuda") as b:
            outs.append(P.run_particle_learning(P.Priors(), y, n, seed=3, keep_indices=True, keep_final=True,
                                                track_quantiles=True, backend=b))
            paths.append(_engine(b).last_path()["fused_draws"])
    assert paths == [True, False]
    a, c = outs
    assert np.array_equal(a.resampled_indices, c.resampled_indices)
    assert np.array_equal(a.final_particles.states, c.final_particles.states)
    assert np.array_equal(a.final_particles.params.sigma2, c.final_particles.params.sigma2)
    assert np.array_equal(a.filtered_quantiles, c.filtered_quantiles)
    # the two kernels' CTA widths differ (512 / 256 threads), so the fp64
    # moment sums are added in a different order: equal to rounding
    assert _rel(a.filtered_mean, c.filtered_mean) <= REL
    for nm in ("sigma2", "tau2"):
        assert _rel(a.param_posterior[nm].mean, c.param_posterior[nm].mean) <= REL
        assert _rel(a.param_posterior[nm].sd, c.param_posterior[nm].sd) <= REL
        assert np.array_equal(a.param_posterior[nm].quantiles, c.param_posterior[nm].quantiles)


@pytest.mark.parametrize("learn", [False, True])
def test_quantile_window_overflow_collapse(gpu, learn):
    """tau2 = 0 (filter) or tau2 = 1e-20 (learning, sigma2 learned): states
    barely move, so resampling piles up copies of a few states and a state
    quantile's candidate window holds more particles than the candidate list
    (cap = max(4096, n/4)) -- exact duplicates in the filter, values whose
    float32 keys tie but whose doubles differ in the learner.  The exact
    select over every particle in the window must give the reference's
    weighted_quantiles (filtering.py:135-140), never a truncated answer."""
    n, t_len, seed = 1 << 14, 40, 2
    tau2 = 1e-20 if learn else 0.0
    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 4)
    feed = make_feed(n, t_len, seed, sigma2_shape=5.0 if learn else None, tau2_shape=None)
    with P.Backend("cuda") as b:
        if learn:
            out = P.run_particle_learning(P.Priors(tau2=tau2), y, n, seed=seed, keep_indices=True,
                                          keep_final=True, track_quantiles=True, noise=feed, backend=b)
        else:
            out = P.run_particle_filter(P.TrendNoiseModel(sigma2=1.0, tau2=tau2), y, n, seed=seed,
                                        keep_indices=True, keep_final=True, track_quantiles=True,
                                        noise=feed, backend=b)
        stats = _engine(b).quantile_stats()
    assert stats["unresolved"] == 0
    assert stats["max_candidates"] > max(4096, n // 4), stats  # the overflow path ran
    ref = R.run_loop(y, n, seed, keep_indices=True, keep_final=True, tau2=tau2,
                     sigma2=(5.0, 4.0) if learn else 1.0, feed=feed)
    assert np.array_equal(out.resampled_indices, ref["indices"])
    assert np.array_equal(out.final_particles.states, ref["final"]["states"])
    assert np.array_equal(out.filtered_quantiles, ref["filtered_quantiles"])
    if learn:
        assert np.array_equal(out.param_posterior["sigma2"].quantiles, ref["sigma2"]["quantiles"])
        assert _rel(out.param_posterior["sigma2"].mean, ref["sigma2"]["mean"]) <= REL
