"""K7: the ordered-uniform (`spacings`) perf-mode resampler (csrc/cdf.cuh).

Not a reference algorithm: it is exact multinomial resampling like the
reference's `sorted` scheme (resampling.py:57-67, merge against sorted
uniforms), with the sorted uniforms generated in order by exponential
spacings instead of by a sort.  Checked three ways:

* against its CPU restatement (oracle/restate.py spacings_indices, the same
  words, the same cut-point lookup): ancestors agree except where the device
  scan's rounding moves a uniform across a CDF value (expected ~0 per step);
* statistically against the reference's exact resamplers: ensemble means
  over seeds (the reference's tests/test_filtering.py:169-182 protocol) and a
  chi-square of ancestor counts under fixed fed weights;
* structurally: ancestors nondecreasing in the slot, zero weights never
  selected -- the locality the scheme exists for.
"""

import numpy as np
import pytest

import paper_1212_1639_b200 as P
from oracle import restate as R
from oracle_feed import make_feed

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [14, 21, 22])
def test_spacings_matches_cpu_restatement(gpu, k):
    n, t_len, seed = 1 << k, 3, 5
    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 6)
    feed = make_feed(n, t_len, seed)
    out = P.run_particle_learning(P.Priors(), y, n, seed=seed, keep_indices=True, keep_final=True,
                                  noise=feed, resampler="spacings")
    ref = R.run_loop(y, n, seed, keep_indices=True, keep_final=True, feed=feed, resampler="spacings")
    idx = out.resampled_indices
    assert (np.diff(idx, axis=1) >= 0).all()          # ordered uniforms -> ordered ancestors
    agree = float(np.mean(idx == ref["indices"]))
    assert agree >= 0.999, agree
    assert np.max(np.abs(out.filtered_mean - ref["filtered_mean"])) <= 1e-6 * np.max(np.abs(ref["filtered_mean"]))


def test_spacings_interchangeable_with_exact_resamplers(gpu):
    # reference tests/test_filtering.py:169-182: ensemble means of two exact
    # multinomial resamplers agree within Monte Carlo error over many seeds
    model = P.TrendNoiseModel()
    _, y = R.simulate(1.0, 0.1, 0.0, 20, 99)
    means = {}
    with P.Backend() as b:
        for resampler in ("naive", "spacings"):
            runs = [P.run_particle_filter(model, y, 1 << 10, seed=s, resampler=resampler, backend=b,
                                          track_quantiles=False).filtered_mean for s in range(60)]
            means[resampler] = np.array(runs)
    a, c = means["naive"], means["spacings"]
    se = np.sqrt(a.var(axis=0, ddof=1) / len(a) + c.var(axis=0, ddof=1) / len(c))
    assert (np.abs(a.mean(axis=0) - c.mean(axis=0)) <= 4 * se).all()


def test_spacings_counts_are_multinomial(gpu):
    """Fixed fed weights (with exact zeros) for T steps: each step's ancestor
    counts are Multinomial(n, w / W); the pooled counts pass a chi-square
    test, zero-weight particles are never chosen, and every step's ancestors
    are nondecreasing."""
    n, t_len = 4096, 120
    rng = np.random.default_rng(3)
    w = rng.exponential(size=n)
    w[rng.random(n) < 0.1] = 0.0
    feed = {"w": np.tile(w, (t_len + 1, 1))}
    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 2)
    out = P.run_particle_filter(P.TrendNoiseModel(), y, n, seed=11, keep_indices=True, noise=feed,
                                resampler="spacings", track_quantiles=False)
    idx = out.resampled_indices - 1
    assert (np.diff(idx, axis=1) >= 0).all()
    counts = np.bincount(idx.ravel(), minlength=n)
    assert counts[w == 0].sum() == 0
    expect = t_len * n * w / w.sum()
    live = w > 0
    chi2 = float(np.sum((counts[live] - expect[live]) ** 2 / expect[live]))
    dof = int(live.sum()) - 1
    z = (chi2 - dof) / np.sqrt(2 * dof)
    assert abs(z) < 4, (chi2, dof, z)


def test_spacings_native_large_n_tracks_kalman(gpu):
    """Native mode at N = 2^22 (fused-draws step kernel, rank tables): the
    filter tracks the Kalman mean as closely as cut-point resampling does."""
    model = P.TrendNoiseModel()
    _, y = R.simulate(1.0, 0.1, 0.0, 30, 17)
    km, _ = P.kalman_filter(y, 1.0, 0.1, 0.0, 10.0)
    n = 1 << 22
    with P.Backend() as b:
        sp = P.run_particle_filter(model, y, n, seed=1, resampler="spacings", keep_indices=True, backend=b,
                                   track_quantiles=False)
    assert (np.diff(sp.resampled_indices, axis=1) >= 0).all()
    assert np.max(np.abs(sp.filtered_mean - km)) < 5e-3


def _series(t_len, seed=1):
    _, y = P.simulate(P.TrendNoiseModel(), t_len, P.RngStream(seed, P.rng.AUX_STREAM_BASE + 1))
    return y


def _locality(idx, shards):
    """Fraction of each step's ancestors owned by the slot's own shard."""
    n = idx.shape[1]
    ns = n // shards
    owner_slot = np.arange(n) // ns
    return float(np.mean((idx - 1) // ns == owner_slot[None, :]))


@pytest.mark.parametrize("shards", [2, 4])
def test_spacings_sharded_group_is_local_and_matches_single(gpu, shards):
    """G shards (pf_group, one GPU): every shard scans its own exponentials and
    the shard totals ride in the exchange records (no extra collective); the
    ancestors are globally nondecreasing, stay in the slot's shard except at
    the shard ends, and match the one-device run (whose scan rounds
    differently) except at near-ties."""
    n, y = 1 << 16, _series(8)
    with P.Backend("cuda") as b:
        one = P.run_particle_learning(P.Priors(), y, n, seed=4, keep_indices=True, backend=b, resampler="spacings")
    with P.Backend("cuda", shards=shards) as b:
        sh = P.run_particle_learning(P.Priors(), y, n, seed=4, keep_indices=True, backend=b, resampler="spacings")
    idx = sh.resampled_indices
    assert (np.diff(idx, axis=1) >= 0).all()
    assert float(np.mean(idx == one.resampled_indices)) >= 0.999
    assert _locality(idx, shards) >= 0.95  # spill = the shards' weight-share imbalance
    assert np.max(np.abs(sh.filtered_mean - one.filtered_mean)) <= 1e-6 * np.max(np.abs(one.filtered_mean))
    # cut-point (parity mode) ancestors are uniform over the shards: ~1/G local
    with P.Backend("cuda", shards=shards) as b:
        cp = P.run_particle_learning(P.Priors(), y, n, seed=4, keep_indices=True, backend=b)
    assert _locality(cp.resampled_indices, shards) < 1.0 / shards + 0.05


@pytest.mark.parametrize("world", [2, 4])
def test_spacings_process_group_gloo(gpu, tmp_path, world):
    """One process per GPU (ranks sharing the B200 over gloo): the same
    ordered-uniform resampler through distributed.py -- every rank returns the
    same outputs, nondecreasing and shard-local ancestors, and the run agrees
    with the one-device spacings run except at near-ties."""
    import test_gpu_dist as TD

    n, t_len = 1 << 15, 8
    d = TD._launch(tmp_path, world, "--particles", str(n), "--series-len", str(t_len), "--resampler", "spacings")
    y = TD._series(t_len)
    with P.Backend("cuda") as b:
        one = P.run_particle_learning(P.Priors(), y, n, seed=5, keep_indices=True, backend=b, resampler="spacings",
                                      track_quantiles=True)
    idx = d["indices0"]
    assert (np.diff(idx, axis=1) >= 0).all()
    assert float(np.mean(idx == one.resampled_indices)) >= 0.999
    assert _locality(idx, world) >= 0.95  # spill = the shards' weight-share imbalance
    np.testing.assert_allclose(d["fmean0"], one.filtered_mean, rtol=1e-6, atol=1e-9)
