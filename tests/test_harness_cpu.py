"""The sweep harness (paper_1212_1639_b200.bench, mirroring parsmc.bench,
SURVEY §8f row 4) on CPU: trimmed means, the CSV schema and round trip, the
ratio table, log-log slopes and config validation -- the reference's
tests/test_bench.py cases restated against this package."""
import csv
import json

import pytest

from paper_1212_1639_b200 import bench as H
from paper_1212_1639_b200.errors import BenchConfigError, InsufficientPointsError


def rec(algorithm="gpu_cutpoint", n=64, trial=1, total=1000, **kw):
    d = dict(algorithm=algorithm, n=n, precision="double", trial=trial, initialize_ns=10, cdf_ns=200,
             resample_ns=300, resample_sort_only_ns=0, propagate_ns=400, store_ns=0, other_ns=90,
             total_ns=total, posterior_sigma2_mean=1.0, posterior_tau2_mean=0.1)
    d.update(kw)
    return H.BenchRecord(**d)


def test_trimmed_mean_keeps_the_middle_half():
    assert H.trimmed_mean(range(1, 11)) == 5.5 - 0.5
    assert H.trimmed_mean([10, 1, 9, 2, 8, 3, 7, 4, 6, 5]) == 5.0
    assert H.trimmed_mean([42]) == 42.0


def test_fields_are_trimmed_independently():
    rs = [rec(trial=t) for t in range(1, 11)]
    rs[0].cdf_ns = 10**9
    rs[-1].propagate_ns = 10**9
    (a,) = H.aggregate_records(rs)
    assert (a.cdf_ns, a.propagate_ns, a.trials) == (200, 400, 10)


def test_csv_schema_is_the_references(tmp_path):
    p = tmp_path / "b.csv"
    H.emit_csv([rec()], p)
    with open(p) as fh:
        header = next(csv.reader(fh))
    assert header == H.CSV_COLUMNS == [
        "algorithm", "n", "precision", "trial", "initialize_ns", "cdf_ns", "resample_ns",
        "resample_sort_only_ns", "propagate_ns", "store_ns", "other_ns", "total_ns",
        "posterior_sigma2_mean", "posterior_tau2_mean"]
    assert len(p.read_text().strip().splitlines()) == 2


def test_csv_round_trip_is_exact(tmp_path):
    rs = [rec(n=1 << k, trial=t, total=k * 10**6 + t, posterior_sigma2_mean=1 / 3, posterior_tau2_mean=0.1 / 3)
          for k in (6, 8) for t in (1, 2)]
    p = tmp_path / "b.csv"
    H.emit_csv(rs, p)
    assert H.load_csv(p) == rs


def test_emitters_reject_bad_input(tmp_path):
    with pytest.raises(ValueError):
        H.emit_csv([], tmp_path / "x.csv")
    with pytest.raises(OSError, match="no/such/dir"):
        H.emit_csv([rec()], "/no/such/dir/b.csv")
    p = H.emit_json([rec()], tmp_path / "b.json")
    assert json.loads(open(p).read())[0]["total_ns"] == 1000


def test_ratio_table():
    rows = H.ratio_table(H.aggregate_records([rec("gpu_sorted", total=3000), rec("gpu_cutpoint", total=1000)]))
    r = {(x["numerator"], x["denominator"]): x["ratio"] for x in rows}
    assert r[("gpu_sorted", "gpu_cutpoint")] == pytest.approx(3.0)
    assert r[("gpu_cutpoint", "gpu_sorted")] == pytest.approx(1 / 3)


@pytest.mark.parametrize("exponent", [1.0, 2.0])
def test_scaling_report_recovers_power_laws(exponent):
    rs = []
    for k in range(6, 12):
        tot = int(50.0 * (1 << k) ** exponent)
        rs.append(rec(n=1 << k, total=tot, cdf_ns=max(1, tot // 4), resample_ns=max(1, tot // 2),
                      propagate_ns=max(1, tot // 8)))
    rep = H.scaling_report(rs)
    assert rep["algorithms"]["gpu_cutpoint"]["slopes"]["total"] == pytest.approx(exponent, abs=0.01)


def test_scaling_needs_three_particle_counts():
    with pytest.raises(InsufficientPointsError):
        H.scaling_report([rec(n=64), rec(n=128)])
    with pytest.raises(InsufficientPointsError):
        H.fit_loglog_slope([64, 128], [1.0, 2.0])


def test_config_validation():
    for algo in ("par_cutpoint", "gpu_cutpoint"):
        with pytest.raises(BenchConfigError):
            H.BenchConfig(n_list=(100,), algorithms=(algo,)).validate()
    H.BenchConfig(n_list=(100,), algorithms=("gpu_sorted", "cpu_naive")).validate()
    for bad in (dict(algorithms=("gpu_magic",)), dict(trials=0), dict(n_list=()), dict(precision="quad"),
                dict(task="smooth"), dict(t_len=0)):
        with pytest.raises(BenchConfigError):
            H.BenchConfig(**bad).validate()


def test_reference_algorithm_names_are_kept():
    for name in ("cpu_naive", "cpu_sorted", "cpu_stratified", "cpu_systematic", "par_cutpoint"):
        assert name in H.ALGORITHMS
    assert H.ALGORITHMS["gpu_cutpoint"] == ("cutpoint", "cuda")
