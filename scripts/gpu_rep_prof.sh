#!/bin/bash
# configs[4] (N=2^20, T=100) diagnostics: where the per-step time goes.
mkdir -p gpurun_out
for fd in 0 1; do
  echo "== PF_FUSED_DRAWS=$fd replications"
  PF_FUSED_DRAWS=$fd timeout 300 python scripts/bench_replications.py --reps 32 --concurrency 1 2>&1 | tail -1
done
echo "== resident timing N=2^20 T=100 (graph)"
timeout 300 python scripts/prof_run.py 20 100 2>&1 | tail -2
PF_PROFILE_FROM_STEP=80 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_2e20.csv python scripts/prof_run.py 20 100 > gpurun_out/ncu_2e20.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_2e20.csv
PF_FUSED_DRAWS=1 PF_PROFILE_FROM_STEP=80 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_2e20_fd.csv python scripts/prof_run.py 20 100 > gpurun_out/ncu_2e20_fd.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_2e20_fd.csv
