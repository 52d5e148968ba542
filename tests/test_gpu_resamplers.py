"""The reference's sequential baseline resamplers on the device
(resampling.py:29-87 inside the loop, filtering.py:299-316): the CDF is the
reference's left-to-right cumsum (prefix_sum.py:130-134), reproduced by one
sequential device thread, and the search is searchsorted 'right'.  Oracle
mode (the reference's own normal / gamma draws fed in): ancestor indices and
particles bit-identical to the reference's runs, including non-power-of-two
N and float32, and at BASELINE configs[0] size (N = 10^4, T = 100) against
the CPU oracle."""

import numpy as np
import pytest

import paper_1212_1639_b200 as P
from conftest import fixture_run_kwargs, golden
from oracle import restate as R

pytestmark = pytest.mark.gpu

RUNS = ["run_pl_sorted", "run_pl_systematic", "run_pl_stratified", "run_pl_naive", "run_pf_sorted"]
REL = 1e-10


def _feed(d):
    f = {"z": d["z"]}
    for k in ("g_sigma", "g_tau"):
        if k in d:
            f[k] = d[k]
    return f


def _run(d, **kw):
    kind, spec = fixture_run_kwargs(d)
    args = dict(seed=int(d["seed"]), keep_indices=True, keep_final=True, track_quantiles=True,
                precision=str(d["precision"]), noise=_feed(d), resampler=str(d["resampler"]))
    args.update(kw)
    fn = P.run_particle_learning if kind == "learn" else P.run_particle_filter
    return fn(spec, d["y"], int(d["n"]), **args)


@pytest.mark.parametrize("name", RUNS)
def test_baseline_resamplers_match_reference(gpu, name):
    d = golden(name)
    out = _run(d)
    assert np.array_equal(out.resampled_indices, d["indices"])
    assert np.array_equal(out.final_particles.states, d["final_states"])
    scale = np.max(np.abs(d["filtered_mean"]))
    assert np.max(np.abs(out.filtered_mean - d["filtered_mean"])) <= REL * scale
    assert np.array_equal(out.filtered_quantiles, d["filtered_quantiles"])
    for nm in ("sigma2", "tau2"):
        if f"{nm}_mean" in d:
            s = out.param_posterior[nm]
            assert np.max(np.abs(s.mean - d[f"{nm}_mean"]) / d[f"{nm}_mean"]) <= REL
            assert np.array_equal(s.quantiles, d[f"{nm}_quantiles"])


def test_sorted_single_precision(gpu):
    d = golden("run_pl_sorted_single")
    out = _run(d)
    assert np.array_equal(out.resampled_indices, d["indices"])
    assert np.array_equal(out.final_particles.states, d["final_states"])


def test_config0_size_against_oracle(gpu):
    """BASELINE configs[0]: N = 10^4 (not a power of two), T = 100, the
    reference's CPU comparator `sorted` -- device vs the CPU oracle fed the
    same draws."""
    n, t_len, seed = 10_000, 100, 0
    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 0)
    rec = {}
    ref = R.run_loop(y, n, seed, track_quantiles=False, keep_indices=True, record=rec, resampler="sorted")
    feed = {k: np.stack([rec[k][t] for t in range(t_len + 1)]) for k in ("z", "g_sigma", "g_tau")}
    out = P.run_particle_learning(P.Priors(), y, n, seed=seed, resampler="sorted", keep_indices=True,
                                  track_quantiles=False, noise=feed)
    assert np.array_equal(out.resampled_indices, ref["indices"])
    np.testing.assert_allclose(out.filtered_mean, ref["filtered_mean"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(out.param_posterior["sigma2"].mean, ref["sigma2"]["mean"], rtol=1e-10)


def test_kernel_level_merge_and_resamplers(gpu):
    rng = np.random.default_rng(11)
    for n in (1, 7, 1000, 4096):
        w = rng.exponential(size=n)
        q = R.sequential_cdf(w)
        u = rng.random(3 * n + 5)
        assert np.array_equal(P.resampling.merge_indices(q, u), R.merge_indices(q, u))
        assert np.array_equal(P.resampling.merge_indices(q, u, sort_first=True),
                              R.merge_indices(q, np.sort(u)))
    q = R.sequential_cdf(rng.exponential(size=256))
    s1 = P.StreamArray.for_lanes(3, 256)
    u = R.uniforms_at(3, np.arange(256, dtype=np.uint64), np.zeros(256, dtype=np.uint64))
    assert np.array_equal(P.resample_naive(q, s1), R.merge_indices(q, u))
    s2 = P.StreamArray.for_lanes(3, 256)
    assert np.array_equal(P.resample_stratified(q, s2), R.merge_indices(q, (np.arange(256) + u) / 256))
    idx, _ = P.resample_sorted(q, P.StreamArray.for_lanes(3, 256))
    assert np.array_equal(idx, R.merge_indices(q, np.sort(u)))


def test_non_power_of_two_only_for_baselines(gpu):
    y = np.array([0.1, -0.2, 0.3])
    out = P.run_particle_filter(P.TrendNoiseModel(), y, 1001, resampler="systematic", keep_indices=True)
    assert out.resampled_indices.shape == (3, 1001)
    assert out.resampled_indices.min() >= 1 and out.resampled_indices.max() <= 1001
    with pytest.raises(P.NotPowerOfTwoError):
        P.run_particle_filter(P.TrendNoiseModel(), y, 1001, resampler="cutpoint")
    one = P.run_particle_learning(P.Priors(), y, 1, resampler="naive", keep_indices=True)
    assert np.all(one.resampled_indices == 1)
