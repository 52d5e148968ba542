"""The sweep harness end to end on the device (paper_1212_1639_b200.bench):
records per (algorithm, n, trial) with device phase times that add up to the
total, identical numerics across trials, the sort-only time for `sorted`."""
import math

import pytest

from paper_1212_1639_b200 import bench as H

pytestmark = pytest.mark.gpu


def test_small_sweep_records_and_determinism(gpu):
    cfg = H.BenchConfig(n_list=(64, 4096), t_len=4, trials=3, algorithms=("gpu_sorted", "gpu_cutpoint"), seed=11)
    records, aggs = H.run_benchmark(cfg)
    assert len(records) == 12 and len(aggs) == 4
    for r in records:
        phases = r.initialize_ns + r.cdf_ns + r.resample_ns + r.propagate_ns + r.store_ns + r.other_ns
        assert phases == r.total_ns and r.total_ns > 0
        assert math.isfinite(r.posterior_sigma2_mean)
    cells = {}
    for r in records:
        cells.setdefault((r.algorithm, r.n), []).append(r)
    for rs in cells.values():
        assert len({(r.posterior_sigma2_mean, r.posterior_tau2_mean) for r in rs}) == 1
    assert all(r.resample_sort_only_ns > 0 for r in records if r.algorithm == "gpu_sorted")
    assert all(r.resample_sort_only_ns == 0 for r in records if r.algorithm == "gpu_cutpoint")


def test_filter_task_and_reference_names(gpu, tmp_path):
    out = tmp_path / "sweep.csv"
    cfg = H.BenchConfig(n_list=(256,), t_len=3, trials=1, algorithms=("cpu_systematic", "par_cutpoint"),
                        task="filter", output_path=str(out))
    records, _ = H.run_benchmark(cfg)
    assert all(math.isnan(r.posterior_sigma2_mean) for r in records)
    back = H.load_csv(out)
    assert [(r.algorithm, r.total_ns, r.cdf_ns) for r in back] == [(r.algorithm, r.total_ns, r.cdf_ns) for r in records]
    assert all(math.isnan(r.posterior_tau2_mean) for r in back)


def test_scaling_report_on_a_real_sweep(gpu):
    cfg = H.BenchConfig(n_list=(1 << 12, 1 << 14, 1 << 16), t_len=8, trials=3, algorithms=("gpu_cutpoint",))
    records, _ = H.run_benchmark(cfg)
    rep = H.scaling_report(records)
    assert 0.0 < rep["algorithms"]["gpu_cutpoint"]["slopes"]["total"] < 1.5
