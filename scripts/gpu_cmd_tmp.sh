#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; grep '^{' gpurun_out/bench.log | tail -1 | cut -c1-150
timeout 600 python bench.py --n 1048576 --no-cpu-baseline > gpurun_out/bench_2e20.log 2>&1; grep '^{' gpurun_out/bench_2e20.log | tail -1 | cut -c1-150
timeout 600 python scripts/bench_replications.py --reps 128 > gpurun_out/bench_replications.log 2>&1; tail -1 gpurun_out/bench_replications.log | cut -c1-150
