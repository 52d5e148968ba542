#!/bin/bash
# Steady-state profiles at configs[2] (N=2^24): full capture of the step kernel
# (source-level), steady launch list with DRAM bytes, full captures of the CDF chain.
mkdir -p gpurun_out
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"step_kernel" -c 1 -o gpurun_out/step_full python scripts/prof_run.py 24 205 > gpurun_out/ncu_step.log 2>&1
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_steady.csv python scripts/prof_run.py 24 210 > gpurun_out/ncu_launch_steady.log 2>&1
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"cdf_|group_build|q_" -c 12 -o gpurun_out/chain_full python scripts/prof_run.py 24 205 > gpurun_out/ncu_chain.log 2>&1
ls -la gpurun_out
echo done
