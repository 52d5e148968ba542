#!/bin/bash
mkdir -p gpurun_out
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"cdf_expand|cdf_reduce_kernel" -c 2 -o gpurun_out/k4_full python scripts/prof_run.py 24 205 > gpurun_out/ncu_k4.log 2>&1
tail -2 gpurun_out/ncu_k4.log
