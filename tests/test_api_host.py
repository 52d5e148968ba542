"""Host-side API behaviour that needs no device: validation order and error
classes (filtering.py:126-148, 191-192, 203-210), model / prior specs,
Backend, estimators' sklearn contract, kalman oracle."""

import math

import numpy as np
import pytest

import paper_1212_1639_b200 as P


def test_non_power_of_two_rejected_before_device():
    with pytest.raises(P.NotPowerOfTwoError):
        P.run_particle_filter(P.TrendNoiseModel(), [1.0], 100, resampler="cutpoint")


def test_nan_observations_rejected():
    with pytest.raises(P.NonFiniteWeightError):
        P.run_particle_filter(P.TrendNoiseModel(), [1.0, float("nan")], 16)


def test_unknown_resampler_and_precision_rejected():
    with pytest.raises(ValueError):
        P.run_particle_filter(P.TrendNoiseModel(), [1.0], 16, resampler="bogus")
    with pytest.raises(ValueError):
        P.run_particle_filter(P.TrendNoiseModel(), [1.0], 16, precision="half")


def test_bad_particle_count():
    with pytest.raises(ValueError):
        P.run_particle_filter(P.TrendNoiseModel(), [1.0], 0)


def test_priors_type_required():
    with pytest.raises(TypeError):
        P.run_particle_learning(P.TrendNoiseModel(), [1.0], 16)


def test_observations_must_be_1d():
    with pytest.raises(ValueError):
        P.run_particle_filter(P.TrendNoiseModel(), np.ones((2, 2)), 16)


def test_model_and_prior_validation():
    with pytest.raises(ValueError):
        P.TrendNoiseModel(sigma2=0.0)
    with pytest.raises(ValueError):
        P.TrendNoiseModel(tau2=-0.1)
    with pytest.raises(ValueError):
        P.InverseGammaPrior(0.0, 1.0)
    with pytest.raises(ValueError):
        P.Priors(tau2=-1.0)
    p = P.Priors(sigma2=P.InverseGammaPrior(5, 4), tau2=0.1)
    assert p.learns_sigma2 and not p.learns_tau2
    assert P.InverseGammaPrior(5.0, 4.0).mean == pytest.approx(1.0)
    assert P.InverseGammaPrior(1.0, 4.0).mean == math.inf


def test_backend_modes_and_split():
    with P.Backend("parallel", lanes=3, min_chunk=3) as b:
        assert b.split(10) == [(0, 4), (4, 7), (7, 10)]
    assert P.Backend().mode == "cuda"
    with pytest.raises(ValueError):
        P.Backend("gpu-ish")
    with pytest.raises(ValueError):
        P.Backend("parallel", lanes=0)


def test_check_weights_and_normalize():
    with pytest.raises(P.NonFiniteWeightError):
        P.check_weights([1.0, np.inf])
    with pytest.raises(ValueError):
        P.check_weights([1.0, -1.0])
    with pytest.raises(P.AllWeightsZeroError):
        P.normalize_weights(np.zeros(3))
    assert np.allclose(P.normalize_weights([1.0, 3.0]), [0.25, 0.75])
    assert P.is_power_of_two(1024) and not P.is_power_of_two(0)


def test_all_weights_zero_message_carries_step():
    e = P.AllWeightsZeroError(step=7)
    assert e.step == 7 and "time step 7" in str(e)


def test_kalman_filter_closed_forms():
    m, v = P.kalman_filter([2.0], sigma2=1.0, tau2=0.0, m0=0.0, c0=10.0)
    assert m[0] == pytest.approx(20.0 / 11.0, rel=1e-14)
    rng = np.random.default_rng(2)
    _, v = P.kalman_filter(rng.normal(size=100), 1.0, 0.0, 0.0, 10.0)
    assert v[-1] == pytest.approx(10.0 / (1.0 + 100 * 10.0), abs=1e-9)


def test_log_likelihood_matches_formula():
    model = P.TrendNoiseModel(sigma2=1.0)
    assert P.log_likelihood(model, 2.0, 2.0) == pytest.approx(-0.5 * math.log(2 * math.pi))
    with pytest.raises(P.NonFiniteWeightError):
        P.log_likelihood(model, float("nan"), 0.0)


def test_estimators_sklearn_contract():
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError

    est = P.ParticleLearner(n_particles=256, seed=3)
    c = clone(est)
    assert c.get_params()["n_particles"] == 256 and c.get_params()["mode"] == "cuda"
    with pytest.raises(NotFittedError):
        c.predict()
    f = P.ParticleFilter(sigma2=2.0)
    assert f.get_params()["sigma2"] == 2.0


def test_param_summary_accessor():
    s = P.ParamSummary(mean=np.zeros(2), sd=np.zeros(2), quantiles=np.arange(10.0).reshape(2, 5))
    assert np.array_equal(s.quantile(0.5), [2.0, 7.0])


def test_phase_timings_total():
    t = P.PhaseTimings(initialize=1, cdf=2, resample=3, resample_sort_only=1, propagate=4,
                       store=5, other=6)
    assert t.total == 21 and t.as_dict()["cdf_ns"] == 2


def test_replication_seeds_partition():
    from paper_1212_1639_b200.replications import rank_seeds

    seeds = list(range(1000))
    parts = [rank_seeds(seeds, r, 8) for r in range(8)]
    assert sorted(x for p in parts for x in p) == seeds
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_backend_shard_arguments():
    import paper_1212_1639_b200 as P

    b = P.Backend("cuda", shards=4, devices=[0, 1, 2, 3])
    assert b.shards == 4 and b.devices == [0, 1, 2, 3]
    assert P.Backend("cuda", shards=2, device=1).devices == [1, 1]
    with pytest.raises(ValueError):
        P.Backend("cuda", shards=3)
    with pytest.raises(ValueError):
        P.Backend("cuda", shards=2, devices=[0])


def test_backend_run_covers_ranges_and_reraises():
    """Backend.run (reference backend.py:52-70): fn(lo, hi) over disjoint lane
    ranges covering [0, n), a barrier in both modes, lane exceptions re-raised."""
    for mode, lanes in (("sequential", 1), ("parallel", 4), ("cuda", 1)):
        b = P.Backend(mode, lanes=lanes, min_chunk=16)
        out = np.zeros(1000, dtype=np.int64)

        def fn(lo, hi):
            out[lo:hi] += np.arange(lo, hi)

        b.run(1000, fn)
        assert np.array_equal(out, np.arange(1000))
        b.run(0, fn)  # no-op
        if mode == "parallel":
            assert len(b.split(1000)) == 4

        def bad(lo, hi):
            if hi == 1000:  # the last lane fails
                raise ValueError("lane failed")

        with pytest.raises(ValueError):
            b.run(1000, bad)
        b.close()


def test_spacings_resampler_is_accepted_and_needs_power_of_two():
    with pytest.raises(P.NotPowerOfTwoError):
        P.run_particle_filter(P.TrendNoiseModel(), [1.0], 100, resampler="spacings")
    from paper_1212_1639_b200 import _lib
    from paper_1212_1639_b200.filtering import PERF_RESAMPLERS

    assert "spacings" in PERF_RESAMPLERS and _lib.RESAMPLER_CODES["spacings"] == 5


def test_cuda_tensor_detection_without_a_device():
    """The kernel-level wrappers take the device-pointer path only for CUDA
    tensors; numpy arrays and CPU tensors stay on the host-array path."""
    import numpy as np
    import torch

    from paper_1212_1639_b200 import _lib

    assert not _lib.is_cuda_tensor(np.ones(4))
    assert not _lib.is_cuda_tensor(torch.ones(4))
    assert not _lib.is_cuda_tensor([1.0, 2.0])
    assert _lib.device_dtype_code(torch.ones(2, dtype=torch.float32)) == _lib.PF_DTYPE_F32
    assert _lib.device_dtype_code(torch.ones(2, dtype=torch.float64)) == _lib.PF_DTYPE_F64


def test_run_replications_batch_rejects_unsupported_options():
    import numpy as np
    import pytest

    import paper_1212_1639_b200 as P
    from paper_1212_1639_b200.replications import run_replications

    with pytest.raises(NotImplementedError):
        run_replications(P.Priors(), np.zeros(3), 1 << 12, [1, 2], batch=2, store_particles=True)
