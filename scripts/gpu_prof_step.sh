#!/bin/bash
mkdir -p gpurun_out
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"step_kernel" -c 1 -o gpurun_out/step_steady python scripts/prof_run.py 24 205 > gpurun_out/ncu_step.log 2>&1
python scripts/ncu_summary.py gpurun_out/step_steady.ncu-rep
echo done
