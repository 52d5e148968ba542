#!/bin/bash
# tests, then full ncu captures (steady state, step 200) of the kernels named in $1 (regex)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"$1" -c ${2:-3} -o gpurun_out/kprof python scripts/prof_run.py 24 205 > gpurun_out/ncu_k.log 2>&1
python scripts/ncu_summary.py gpurun_out/kprof.ncu-rep
echo done
