"""Batched replications (pf_engine_run_batch; BASELINE configs[4]): R
independent filters of n particles in every kernel launch, one adder tree
per replication.

Each replication must follow the single run with its seed: the same
particle system (the draws, the CDF and the ancestors do not depend on how
the launch is shared), so the summaries agree to rounding -- the moment and
weight sums are split over fewer CTAs per replication -- and the weighted
quantiles agree exactly except at an exact near-tie.
"""

import numpy as np
import pytest

import paper_1212_1639_b200 as P
from paper_1212_1639_b200.filtering import run_batch
from paper_1212_1639_b200.replications import run_replications

pytestmark = pytest.mark.gpu


def _series(t_len, seed=1):
    _, y = P.simulate(P.TrendNoiseModel(), t_len, P.RngStream(seed, P.rng.AUX_STREAM_BASE + 1))
    return y


def _close(a, b, rtol=1e-10):
    a, b = np.asarray(a), np.asarray(b)
    scale = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / scale))


def _compare(batched, single, rtol=1e-10):
    assert _close(batched.filtered_mean, single.filtered_mean) <= rtol
    assert _close(batched.ess, single.ess) <= 1e-9
    if single.filtered_quantiles is not None:
        fq_b, fq_s = batched.filtered_quantiles, single.filtered_quantiles
        assert np.mean(fq_b == fq_s) >= 0.99
        assert _close(fq_b, fq_s) <= 1e-6
    for name, s in (single.param_posterior or {}).items():
        b = batched.param_posterior[name]
        assert _close(b.mean, s.mean) <= rtol
        assert _close(b.sd, s.sd) <= 1e-8
        assert np.mean(b.quantiles == s.quantiles) >= 0.99
        assert _close(b.quantiles, s.quantiles) <= 1e-6


@pytest.mark.parametrize("n,reps", [(1 << 12, 3), (1 << 16, 4), (1 << 20, 6)])
def test_batched_pl_matches_single_runs(gpu, n, reps):
    y = _series(25)
    seeds = [7, 2**63 + 5, 11, 0, 123456789, 42][:reps]
    with P.Backend() as b:
        outs = run_batch(P.Priors(), y, n, seeds, backend=b)
        singles = [P.run_particle_learning(P.Priors(), y, n, seed=s, backend=b) for s in seeds]
    assert len(outs) == reps
    for o, s in zip(outs, singles):
        _compare(o, s)
    # different seeds give different filters
    assert not np.array_equal(outs[0].filtered_mean, outs[1].filtered_mean)


def test_batched_known_parameters_and_state_quantiles(gpu):
    y = _series(15, seed=3)
    model = P.TrendNoiseModel()
    seeds = [1, 2, 3, 4, 5]
    with P.Backend() as b:
        outs = run_batch(model, y, 1 << 14, seeds, backend=b, track_quantiles=True)
        singles = [P.run_particle_filter(model, y, 1 << 14, seed=s, backend=b, track_quantiles=True) for s in seeds]
    for o, s in zip(outs, singles):
        _compare(o, s)


def test_batched_single_precision(gpu):
    y = _series(12, seed=4)
    with P.Backend() as b:
        outs = run_batch(P.Priors(), y, 1 << 13, [9, 10], backend=b, precision="single")
        singles = [P.run_particle_learning(P.Priors(), y, 1 << 13, seed=s, backend=b, precision="single")
                   for s in (9, 10)]
    for o, s in zip(outs, singles):
        _compare(o, s, rtol=1e-6)


def test_run_replications_batch_option_and_engine_reuse(gpu):
    """run_replications(batch=R) chunks the seeds (a ragged last batch
    included); the engine's enlarged buffers then serve ordinary runs."""
    y = _series(10, seed=5)
    seeds = list(range(7))
    with P.Backend() as b:
        batched = run_replications(P.Priors(), y, 1 << 12, seeds, backend=b, batch=3)
        after = P.run_particle_learning(P.Priors(), y, 1 << 12, seed=3, backend=b, keep_indices=True)
    with P.Backend() as b:
        fresh = P.run_particle_learning(P.Priors(), y, 1 << 12, seed=3, backend=b, keep_indices=True)
        singles = [P.run_particle_learning(P.Priors(), y, 1 << 12, seed=s, backend=b) for s in seeds]
    assert len(batched) == 7
    for o, s in zip(batched, singles):
        _compare(o, s)
    np.testing.assert_array_equal(after.resampled_indices, fresh.resampled_indices)
    np.testing.assert_array_equal(after.filtered_mean, fresh.filtered_mean)


def test_batched_restrictions(gpu):
    y = _series(5)
    with pytest.raises(NotImplementedError):
        run_batch(P.Priors(), y, 1 << 21, [1, 2])        # rank-table sizes run one at a time
    with pytest.raises(NotImplementedError):
        run_batch(P.Priors(), y, 1 << 10, [1, 2])        # below one CDF tile
    with pytest.raises(NotImplementedError):
        run_replications(P.Priors(), y, 1 << 12, [1, 2], batch=2, keep_indices=True)
    one = run_batch(P.Priors(), y, 1 << 10, [4])          # R = 1 is the ordinary run
    ref = P.run_particle_learning(P.Priors(), y, 1 << 10, seed=4)
    np.testing.assert_array_equal(one[0].filtered_mean, ref.filtered_mean)


@pytest.mark.parametrize("world", [2, 3])
def test_replications_across_ranks(gpu, tmp_path, world):
    """Replicas only (SURVEY §8e configs[4]): ranks take seeds round robin
    and batch them; the gathered summaries match one-at-a-time runs."""
    import os
    import subprocess
    import sys

    from conftest import ROOT
    import test_gpu_dist as TD

    out = str(tmp_path / "reps.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(TD._port()),
           os.path.join(ROOT, "tests", "workers", "replication_worker.py"), "--out", out]
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = np.load(out)
    assert list(d["seeds"]) == list(range(7))
    y = TD._series(10)
    with P.Backend() as b:
        for i, s in enumerate(range(7)):
            one = P.run_particle_learning(P.Priors(), y, 1 << 12, seed=s, backend=b)
            assert _close(d["fmean"][i], one.filtered_mean) <= 1e-10
            assert _close(d["smean"][i], one.param_posterior["sigma2"].mean) <= 1e-10
            assert np.mean(d["tq"][i] == one.param_posterior["tau2"].quantiles) >= 0.99


def test_batched_replications_do_not_interact(gpu):
    """The same seed in two slots of a batch gives bit-identical summaries
    (each replication reads and writes only its own slices), whatever sits
    between them; T = 0 and T = 1 batches are well formed."""
    y = _series(30, seed=6)
    with P.Backend() as b:
        outs = run_batch(P.Priors(), y, 1 << 13, [5, 9, 5, 123, 5], backend=b, track_quantiles=True)
        for k in (2, 4):
            np.testing.assert_array_equal(outs[k].filtered_mean, outs[0].filtered_mean)
            np.testing.assert_array_equal(outs[k].filtered_quantiles, outs[0].filtered_quantiles)
            for name in ("sigma2", "tau2"):
                np.testing.assert_array_equal(outs[k].param_posterior[name].quantiles,
                                              outs[0].param_posterior[name].quantiles)
        assert not np.array_equal(outs[1].filtered_mean, outs[0].filtered_mean)
        empty = run_batch(P.Priors(), y[:0], 1 << 13, [1, 2], backend=b)
        assert len(empty) == 2 and empty[0].filtered_mean.shape == (0,)
        one = run_batch(P.Priors(), y[:1], 1 << 13, [1, 2], backend=b)
        ref = P.run_particle_learning(P.Priors(), y[:1], 1 << 13, seed=2, backend=b)
        _compare(one[1], ref)
