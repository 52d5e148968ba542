#!/bin/bash
# Iteration check: GPU parity tests, bench, steady-state launch list (steps 290..300).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
cat gpurun_out/bench.log
PF_PROFILE_FROM_STEP=290 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_steady.csv python scripts/prof_run.py 24 300 > gpurun_out/prof_steady.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_steady.csv
echo done
