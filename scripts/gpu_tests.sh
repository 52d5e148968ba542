#!/bin/bash
# GPU parity tests (optionally a subset via $PYTEST_ARGS), then the default bench.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/nvidia_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rA ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|worst|Error|assert" gpurun_out/pytest_gpu.log | tail -30
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
fi
echo done
