#!/bin/bash
set -x
mkdir -p gpurun_out
./scripts/micro/gather > gpurun_out/gather.log 2>&1
./scripts/micro/gather 32 >> gpurun_out/gather.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --csv ./scripts/micro/gather > gpurun_out/gather_ncu.csv 2>&1
PF_PROFILE_FROM_STEP=290 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_steady.csv python scripts/prof_run.py 24 300 > gpurun_out/prof_steady.log 2>&1
timeout 300 python scripts/prof_run.py 24 1000 > gpurun_out/prof_1000.log 2>&1
echo done
