#!/bin/bash
set -x
mkdir -p gpurun_out
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"cdf_reduce_q|cdf_expand|q_finish|q_hist" -c 4 -o gpurun_out/cdf_full python scripts/prof_run.py 24 205 > gpurun_out/ncu_cdf.log 2>&1
echo done
