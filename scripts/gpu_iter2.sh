#!/bin/bash
# Iteration: bench (no CPU baseline), a parity subset, and memcheck of the fused-draws step kernel.
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("value", d["value"]/1e9, "e2e", d["e2e"]["value"]/1e9, "step_ms", d["roofline"]["step_kernel_ms"], "frac", d["roofline"]["frac"])'
timeout 1200 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-tests/test_gpu_parity_large.py tests/test_gpu_engine.py tests/test_gpu_kernels.py} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
if [ -n "$SAN" ]; then
PF_FUSED_DRAWS=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/prof_run.py 16 3 > gpurun_out/memcheck_default.txt 2>&1; tail -3 gpurun_out/memcheck_default.txt
PARSMC_B200_LIB=$PWD/build_variants/sb1.so PF_FUSED_DRAWS=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/prof_run.py 16 3 > gpurun_out/memcheck_sb1.txt 2>&1; tail -3 gpurun_out/memcheck_sb1.txt
fi
echo done
