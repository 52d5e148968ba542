"""Particle filtering / particle learning drivers -- the drop-in boundary.

``run_particle_filter`` / ``run_particle_learning`` keep the reference's
signatures, validation, error classes and outputs (filtering.py:165-197);
the cycle itself -- propagate, weight, CDF, resample, store, summaries
(filtering.py:200-374) -- runs as sm_100a kernels inside one device engine
with no host round trips between steps.  Host work is limited to argument
validation, one upload of the configuration and one download of the [T]
summaries (plus particles when asked for).

Phase attribution (``PhaseTimings``) uses CUDA events between the fused
kernels: *propagate* is the step kernel, which also performs the previous
step's cut-point lookup and joint gather (the reference's per-step resample
work is fused there and so is charged to propagate); *cdf* covers the adder
tree and cut table; *other* the summaries; *store* the per-step snapshot
copies; *resample* the final step's resample.  The fields sum to the total.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .backend import Backend
from .core import ParamDraws, ParticleSystem, SuffStats, check_power_of_two
from .engine import Engine, Group, make_config
from .errors import NonFiniteWeightError
from .models import Priors

RESAMPLERS = ("naive", "sorted", "stratified", "systematic", "cutpoint")
PARAM_QUANTILE_PROBS = (0.005, 0.05, 0.5, 0.95, 0.995)
STATE_QUANTILE_PROBS = (0.05, 0.5, 0.95)


@dataclass
class PhaseTimings:
    """Per-phase elapsed nanoseconds (filtering.py:44-74)."""

    initialize: int = 0
    cdf: int = 0
    resample: int = 0
    resample_sort_only: int = 0
    propagate: int = 0
    store: int = 0
    other: int = 0

    @property
    def total(self):
        return (self.initialize + self.cdf + self.resample
                + self.propagate + self.store + self.other)

    def as_dict(self):
        return {"initialize_ns": self.initialize, "cdf_ns": self.cdf,
                "resample_ns": self.resample, "resample_sort_only_ns": self.resample_sort_only,
                "propagate_ns": self.propagate, "store_ns": self.store, "other_ns": self.other}


@dataclass
class ParamSummary:
    """Posterior summary of one parameter at every step (filtering.py:90-100)."""

    mean: np.ndarray
    sd: np.ndarray
    quantiles: np.ndarray
    probs: tuple = PARAM_QUANTILE_PROBS

    def quantile(self, p):
        return self.quantiles[:, self.probs.index(p)]


@dataclass
class FilterOutput:
    filtered_mean: np.ndarray
    filtered_quantiles: np.ndarray | None
    param_posterior: dict | None
    timings: PhaseTimings
    final_particles: ParticleSystem | None = None
    particle_history: list | None = None
    resampled_indices: np.ndarray | None = None
    # extension (not in the reference): effective sample size per step,
    # (sum w)^2 / sum w^2 of the pre-resample weights, from the device's
    # per-shard weight sums
    ess: np.ndarray | None = None


def snapshot_store(particles, dest):
    """Deep-copy a particle system into ``dest``; returns elapsed ns
    (filtering.py:114-123)."""
    import time

    t0 = time.perf_counter_ns()
    dest.append(particles.copy())
    return max(1, time.perf_counter_ns() - t0)


def check_observations(y):
    """filtering.py:126-132."""
    y = np.asarray(y, dtype=np.float64)
    if y.ndim != 1:
        raise ValueError("observations must be a 1-d array")
    if y.size and not np.isfinite(y).all():
        raise NonFiniteWeightError("observations contain NaN or infinity")
    return y


def weighted_quantiles(values, weights, probs):
    """Smallest value (stable order) with cumulative weight >= p*W, on the
    device (filtering.py:135-140)."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    w = np.asarray(weights)
    if w.dtype not in (np.float32, np.float64):
        w = w.astype(np.float64)
    w = np.ascontiguousarray(w)
    p = np.ascontiguousarray(np.atleast_1d(np.asarray(probs, dtype=np.float64)))
    out = np.empty(len(p))
    lib = _lib.require_device()
    _lib.check(lib.pf_weighted_quantiles(_lib.ptr(v), _lib.vptr(w), _lib.dtype_code(w.dtype),
                                         len(v), _lib.ptr(p), len(p), _lib.ptr(out)), lib)
    return out


def _dtype_for(precision):
    if precision == "double":
        return np.float64
    if precision == "single":
        return np.float32
    raise ValueError(f"precision must be 'single' or 'double', got {precision!r}")


def run_particle_filter(model, y, n, seed=0, backend=None, resampler="cutpoint",
                        precision="double", store_particles=False, keep_final=False,
                        track_quantiles=True, keep_indices=False, debug_checks=False,
                        noise=None):
    """Filter with known parameters (filtering.py:165-175)."""
    return _run_loop(model=model, priors=None, y=y, n=n, seed=seed, backend=backend,
                     resampler=resampler, precision=precision, store_particles=store_particles,
                     keep_final=keep_final, track_quantiles=track_quantiles,
                     keep_indices=keep_indices, debug_checks=debug_checks, noise=noise)


def run_particle_learning(priors, y, n, seed=0, backend=None, resampler="cutpoint",
                          precision="double", store_particles=False, keep_final=False,
                          track_quantiles=True, keep_indices=False, debug_checks=False,
                          noise=None):
    """Joint state and parameter filtering (filtering.py:178-197).

    ``noise`` (extension, oracle mode): a dict of [T+1, n] float64 arrays
    ``z``, ``g_sigma``, ``g_tau`` (and optionally ``w``, rows 1..T) that replace
    the device's ndtri / gammaincinv outputs (and weights) with externally
    supplied draws -- the reference's own, in the parity tests.
    """
    if not isinstance(priors, Priors):
        raise TypeError("run_particle_learning expects a Priors instance")
    return _run_loop(model=None, priors=priors, y=y, n=n, seed=seed, backend=backend,
                     resampler=resampler, precision=precision, store_particles=store_particles,
                     keep_final=keep_final, track_quantiles=track_quantiles,
                     keep_indices=keep_indices, debug_checks=debug_checks, noise=noise)


def _build_config(model, priors, n, seed, precision, flags, device, resampler="cutpoint"):
    learn = priors is not None
    if learn:
        ls, lt = priors.learns_sigma2, priors.learns_tau2
        kw = dict(x0_mean=priors.x0_mean, x0_var=priors.x0_var,
                  sigma2_shape=priors.sigma2.shape if ls else 0.0,
                  sigma2_scale=priors.sigma2.scale if ls else 0.0,
                  tau2_shape=priors.tau2.shape if lt else 0.0,
                  tau2_scale=priors.tau2.scale if lt else 0.0,
                  sigma2_fixed=1.0 if ls else float(priors.sigma2),
                  tau2_fixed=1.0 if lt else float(priors.tau2))
    else:
        ls = lt = False
        kw = dict(x0_mean=model.x0_mean, x0_var=model.x0_var,
                  sigma2_fixed=float(model.sigma2), tau2_fixed=float(model.tau2))
    return make_config(n, seed, learn=learn, learn_sigma2=ls, learn_tau2=lt,
                       precision=precision, device=device, resampler=resampler, **flags, **kw), ls, lt


def _run_loop(model, priors, y, n, seed, backend, resampler, precision, store_particles,
              keep_final, track_quantiles, keep_indices, debug_checks, noise=None):
    y = check_observations(y)
    n = int(n)
    if n < 1:
        raise ValueError("particle count must be >= 1")
    if resampler not in RESAMPLERS:
        raise ValueError(f"unknown resampler {resampler!r}; choose from {RESAMPLERS}")
    if resampler == "cutpoint":
        check_power_of_two(n)
    dtype = _dtype_for(precision)
    # debug_checks: the device gathers each particle's tuple as one 32-byte
    # record, so a torn tuple cannot occur; the flag is accepted and inert.
    del debug_checks
    learn = priors is not None
    t_len = len(y)
    flags = dict(track_quantiles=track_quantiles, keep_indices=keep_indices,
                 keep_final=keep_final, store_particles=store_particles, phase_timing=True)
    own = backend is None
    if own:
        backend = Backend()
    try:
        cfg, ls, lt = _build_config(model, priors, n, seed, precision, flags, backend.device, resampler)
        shards = getattr(backend, "shards", 1)
        if getattr(backend, "distributed", False):
            if store_particles:
                raise NotImplementedError("store_particles is not supported by sharded runs")
            if resampler != "cutpoint":
                raise NotImplementedError("sharded runs use the cut-point resampler")
            if noise is not None:
                raise NotImplementedError("oracle feeds are not supported by sharded runs")
            key = ("rank", n, precision, backend.device, bool(track_quantiles), learn, ls, lt)

            def factory():
                from .distributed import ShardRank

                return ShardRank(cfg, backend.process_group)
        elif shards > 1:
            if store_particles:
                raise NotImplementedError("store_particles is not supported by sharded runs")
            if resampler != "cutpoint":
                raise NotImplementedError("sharded runs use the cut-point resampler")
            key = ("group", n, precision, tuple(backend.devices))

            def factory():
                return Group(cfg, backend.devices)
        else:
            key = ("engine", n, precision, backend.device, resampler)

            def factory():
                return Engine(cfg)

        eng = backend.engine(key, factory)
        eng.reconfigure(cfg)
        out, arrays = _alloc_outputs(t_len, n, learn, ls, lt, track_quantiles, keep_indices,
                                     keep_final, store_particles)
        feed = None
        if noise is not None:
            feed = {k: np.ascontiguousarray(np.asarray(v, dtype=np.float64))
                    for k, v in noise.items() if v is not None}
        if getattr(backend, "distributed", False):
            eng.run_arrays(np.ascontiguousarray(y, dtype=np.float64), arrays, n)
        else:
            eng.run(y, out, feed)
    finally:
        if own:
            backend.close()
    return _assemble(out, arrays, t_len, n, dtype, learn, ls, lt, store_particles)


def _alloc_outputs(t_len, n, learn, ls, lt, track_quantiles, keep_indices, keep_final, store):
    out = _lib.PfOutputs()
    a = {"filtered_mean": np.empty(t_len), "ess": np.empty(t_len)}
    if track_quantiles:
        a["filtered_quantiles"] = np.empty((t_len, 3))
    if learn and ls:
        a["sigma2_mean"], a["sigma2_sd"] = np.empty(t_len), np.empty(t_len)
        a["sigma2_quantiles"] = np.empty((t_len, 5))
    if learn and lt:
        a["tau2_mean"], a["tau2_sd"] = np.empty(t_len), np.empty(t_len)
        a["tau2_quantiles"] = np.empty((t_len, 5))
    if keep_indices:
        a["indices"] = np.empty((t_len, n), dtype=np.int64)
    names = ("states", "sigma2", "tau2", "a_sigma", "b_sigma", "a_tau", "b_tau")
    if keep_final:
        for nm in names:
            a["final_" + nm] = np.empty(n)
    if store and t_len:
        for nm in names:
            a["hist_" + nm] = np.empty((t_len, n))
    for k, v in a.items():
        setattr(out, k, _lib.ptr(v, _lib.C.c_int64 if v.dtype == np.int64 else _lib.C.c_double))
    return out, a


def _system(get, n, dtype, learn):
    states = get("states").astype(dtype)
    weights = np.full(n, 1.0 / n, dtype=dtype)
    params = suff = None
    if learn:
        params = ParamDraws(sigma2=get("sigma2").copy(), tau2=get("tau2").copy())
        suff = SuffStats(a_sigma=get("a_sigma").copy(), b_sigma=get("b_sigma").copy(),
                         a_tau=get("a_tau").copy(), b_tau=get("b_tau").copy())
    return ParticleSystem(states=states, weights=weights, params=params, suffstats=suff)


def _assemble(out, a, t_len, n, dtype, learn, ls, lt, store):
    ph = list(out.phase_ns)
    timings = PhaseTimings(initialize=ph[0], cdf=ph[1], resample=ph[2],
                           resample_sort_only=ph[3], propagate=ph[4], store=ph[5], other=ph[6])
    summaries = None
    if learn:
        summaries = {}
        for name, on in (("sigma2", ls), ("tau2", lt)):
            if on:
                summaries[name] = ParamSummary(mean=a[name + "_mean"], sd=a[name + "_sd"],
                                               quantiles=a[name + "_quantiles"])
    final = None
    if "final_states" in a:
        final = _system(lambda k: a["final_" + k], n, dtype, learn)
    history = None
    if store:
        history = [_system(lambda k, t=t: a["hist_" + k][t], n, dtype, learn) for t in range(t_len)]
    return FilterOutput(filtered_mean=a["filtered_mean"],
                        filtered_quantiles=a.get("filtered_quantiles"),
                        param_posterior=summaries, timings=timings, final_particles=final,
                        particle_history=history, resampled_indices=a.get("indices"), ess=a.get("ess"))
