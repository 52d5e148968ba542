#!/bin/bash
mkdir -p gpurun_out
./scripts/micro/gather > gpurun_out/gather2.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --csv ./scripts/micro/gather > gpurun_out/gather2_ncu.csv 2>&1
echo done
