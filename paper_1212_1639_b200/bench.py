"""Particle-count sweeps (the reference's benchmark harness, ``parsmc.bench``).

Same surface as the reference module (bench.py:1-288 of ``parsmc``): the
``ALGORITHMS`` table, ``BenchConfig`` / ``BenchRecord`` / ``AggregateRecord``,
the CSV schema ``CSV_COLUMNS``, ``run_benchmark``, the trimmed-mean
aggregation, CSV / JSON emitters and loaders, the pairwise ratio table and the
log-log scaling report -- so Table 3/4-style sweeps run unchanged against this
package.

What differs is where the cells run.  The reference's five algorithms name a
resampler and a CPU backend mode; here every mode executes on the device, so
those names are kept (callers that pass them keep working) and the explicit
``gpu_*`` entries name the same resamplers on ``Backend("cuda")``.  One
engine per (algorithm, n) is kept resident across that cell's trials: the
timings are the device phase times of each run (CUDA events, ``PhaseTimings``),
which never include engine creation, exactly as the reference keeps its JIT
warm-up out of the records (bench.py:153-161 there).
"""

from __future__ import annotations

import csv
import json
import math
import statistics
from dataclasses import asdict, dataclass, fields

import numpy as np

from .backend import Backend
from .core import is_power_of_two
from .errors import BenchConfigError, InsufficientPointsError
from .filtering import run_particle_filter, run_particle_learning
from .models import Priors, TrendNoiseModel, simulate
from .rng import AUX_STREAM_BASE, RngStream

#: algorithm -> (resampler, backend mode).  The first five are the
#: reference's names (bench.py:28-34 there); all of them run on the device.
ALGORITHMS = {
    "cpu_naive": ("naive", "sequential"),
    "cpu_sorted": ("sorted", "sequential"),
    "cpu_stratified": ("stratified", "sequential"),
    "cpu_systematic": ("systematic", "sequential"),
    "par_cutpoint": ("cutpoint", "parallel"),
    "gpu_cutpoint": ("cutpoint", "cuda"),
    "gpu_sorted": ("sorted", "cuda"),
    "gpu_systematic": ("systematic", "cuda"),
    "gpu_stratified": ("stratified", "cuda"),
    "gpu_naive": ("naive", "cuda"),
}

#: the observation path comes from aux stream 2^62 + 1 (the reference's data stream)
DATA_STREAM_ID = AUX_STREAM_BASE + 1


@dataclass
class BenchConfig:
    n_list: tuple = (1024, 4096)
    t_len: int = 100
    trials: int = 10
    algorithms: tuple = ("gpu_cutpoint",)
    precision: str = "double"
    seed: int = 0
    store_particles: bool = False
    output_path: str | None = None
    lanes: int = 4
    task: str = "learn"  # "learn": unknown variances; "filter": known parameters
    device: int = 0

    def validate(self):
        problems = []
        if not self.n_list:
            problems.append("n_list must not be empty")
        problems += [f"particle count must be >= 1, got {n}" for n in self.n_list if n < 1]
        for name in ("trials", "t_len", "lanes"):
            if getattr(self, name) < 1:
                problems.append(f"{name} must be >= 1")
        if self.precision not in ("single", "double"):
            problems.append(f"unknown precision {self.precision!r}")
        if self.task not in ("learn", "filter"):
            problems.append(f"unknown task {self.task!r}")
        unknown = sorted(set(self.algorithms) - set(ALGORITHMS))
        if unknown:
            problems.append(f"unknown algorithms {unknown}; choose from {sorted(ALGORITHMS)}")
        if any(ALGORITHMS.get(a, ("",))[0] == "cutpoint" for a in self.algorithms):
            odd = [n for n in self.n_list if n >= 1 and not is_power_of_two(n)]
            if odd:
                problems.append(f"cutpoint algorithms need power-of-two particle counts, got {odd}")
        if problems:
            raise BenchConfigError(problems[0])
        return self


@dataclass
class BenchRecord:
    algorithm: str
    n: int
    precision: str
    trial: int
    initialize_ns: int
    cdf_ns: int
    resample_ns: int
    resample_sort_only_ns: int
    propagate_ns: int
    store_ns: int
    other_ns: int
    total_ns: int
    posterior_sigma2_mean: float
    posterior_tau2_mean: float


CSV_COLUMNS = [f.name for f in fields(BenchRecord)]
TIMING_FIELDS = tuple(c for c in CSV_COLUMNS if c.endswith("_ns"))


@dataclass
class AggregateRecord:
    """One (algorithm, n, precision) cell: each timing field trimmed independently."""

    algorithm: str
    n: int
    precision: str
    trials: int
    initialize_ns: float
    cdf_ns: float
    resample_ns: float
    resample_sort_only_ns: float
    propagate_ns: float
    store_ns: float
    other_ns: float
    total_ns: float
    posterior_sigma2_mean: float
    posterior_tau2_mean: float


def trimmed_mean(values):
    """Mean of the middle ``len // 2`` order statistics (the middle 5 of 10)."""
    ordered = sorted(values)
    keep = max(1, len(ordered) // 2)
    start = (len(ordered) - keep) // 2
    return float(statistics.fmean(ordered[start:start + keep]))


def _cell_run(config, algorithm, n, y, backend):
    resampler = ALGORITHMS[algorithm][0]
    common = dict(seed=config.seed, backend=backend, resampler=resampler, precision=config.precision,
                  store_particles=config.store_particles, track_quantiles=False)
    if config.task == "learn":
        return run_particle_learning(Priors(), y, n, **common)
    return run_particle_filter(TrendNoiseModel(), y, n, **common)


def _posterior_means(out):
    post = out.param_posterior or {}
    return tuple(float(post[k].mean[-1]) if k in post else math.nan for k in ("sigma2", "tau2"))


def run_benchmark(config, progress=None):
    """Run the sweep; returns ``(records, aggregates)``."""
    config.validate()
    _, y = simulate(TrendNoiseModel(), config.t_len, RngStream(config.seed, DATA_STREAM_ID))
    records = []
    for algorithm in config.algorithms:
        mode = ALGORITHMS[algorithm][1]
        for n in config.n_list:
            with Backend(mode=mode, lanes=config.lanes, device=config.device) as backend:
                _cell_run(config, algorithm, n, y, backend)  # engine + tables: outside the records
                for trial in range(1, config.trials + 1):
                    out = _cell_run(config, algorithm, n, y, backend)
                    sig, tau = _posterior_means(out)
                    t = out.timings
                    rec = BenchRecord(algorithm=algorithm, n=n, precision=config.precision, trial=trial,
                                      total_ns=t.total, posterior_sigma2_mean=sig, posterior_tau2_mean=tau,
                                      **t.as_dict())
                    records.append(rec)
                    if progress is not None:
                        progress(rec)
    if config.output_path:
        emit_csv(records, config.output_path)
    return records, aggregate_records(records)


def aggregate_records(records):
    cells = {}
    for r in records:
        cells.setdefault((r.algorithm, r.n, r.precision), []).append(r)
    out = []
    for (algorithm, n, precision), rs in cells.items():
        timing = {f: trimmed_mean(getattr(r, f) for r in rs) for f in TIMING_FIELDS}
        out.append(AggregateRecord(algorithm=algorithm, n=n, precision=precision, trials=len(rs),
                                   posterior_sigma2_mean=rs[0].posterior_sigma2_mean,
                                   posterior_tau2_mean=rs[0].posterior_tau2_mean, **timing))
    return out


def emit_csv(records, path):
    """Header (``CSV_COLUMNS``) and one row per record."""
    if not records:
        raise ValueError("no records to write")
    try:
        with open(path, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=CSV_COLUMNS)
            w.writeheader()
            w.writerows(asdict(r) for r in records)
    except OSError as exc:
        raise OSError(f"cannot write benchmark CSV to {path}: {exc}") from exc
    return path


def load_csv(path):
    conv = {f.name: f.type for f in fields(BenchRecord)}
    cast = {"int": int, "float": float, "str": str}
    with open(path, newline="") as fh:
        return [BenchRecord(**{k: cast[conv[k]](v) for k, v in row.items()}) for row in csv.DictReader(fh)]


def emit_json(records, path):
    with open(path, "w") as fh:
        json.dump([asdict(r) for r in records], fh, indent=2)
    return path


def ratio_table(aggregates):
    """Trimmed total-time ratios for every ordered pair of algorithms at each n."""
    by_n = {}
    for a in aggregates:
        by_n.setdefault(a.n, {})[a.algorithm] = a.total_ns
    rows = []
    for n in sorted(by_n):
        cell = by_n[n]
        names = sorted(cell)
        rows += [{"numerator": p, "denominator": q, "n": n, "ratio": cell[p] / cell[q]}
                 for p in names for q in names if p != q and cell[q] > 0]
    return rows


def fit_loglog_slope(ns, values):
    if len(ns) < 3:
        raise InsufficientPointsError(f"need >= 3 particle counts for a slope, got {len(ns)}")
    x = np.log(np.asarray(ns, dtype=np.float64))
    yv = np.log(np.asarray(values, dtype=np.float64))
    return float(np.polyfit(x, yv, 1)[0])


def scaling_report(records, min_points=3):
    """Per-algorithm log-log slopes (total and per phase) and the ratio block."""
    aggregates = aggregate_records(records)
    groups = {}
    for a in aggregates:
        groups.setdefault(a.algorithm, []).append(a)
    report = {"algorithms": {}, "ratios": ratio_table(aggregates)}
    for algorithm, aggs in groups.items():
        aggs = sorted(aggs, key=lambda a: a.n)
        ns = [a.n for a in aggs]
        if len(set(ns)) < min_points:
            raise InsufficientPointsError(f"{algorithm}: need >= {min_points} particle counts, got {len(set(ns))}")
        slopes = {}
        for phase in ("total", "cdf", "resample", "propagate"):
            vals = [getattr(a, phase + "_ns") for a in aggs]
            if min(vals) > 0:
                slopes[phase] = fit_loglog_slope(ns, vals)
        report["algorithms"][algorithm] = {"slopes": slopes, "points": {a.n: a.total_ns for a in aggs}}
    return report
