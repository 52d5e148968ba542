#!/bin/bash
# Round evidence: GPU tests, smoke, the default bench (with CPU baseline), the reference arm,
# perf-mode and small-N lines, the one-process-per-GPU path, the chain split, the ncu launch list
# (steady state) and a full capture of the step kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
timeout 600 python bench.py --resampler spacings --no-cpu-baseline > gpurun_out/bench_spacings.log 2>&1; tail -1 gpurun_out/bench_spacings.log
timeout 600 python bench.py --n 1048576 --t 1000 --no-cpu-baseline > gpurun_out/bench_2e20.log 2>&1; tail -1 gpurun_out/bench_2e20.log
timeout 600 python scripts/bench_replications.py --reps 128 > gpurun_out/bench_replications.log 2>&1; tail -1 gpurun_out/bench_replications.log
timeout 600 python scripts/bench_replications.py --reps 64 --batch 1 > gpurun_out/bench_replications_b1.log 2>&1; tail -1 gpurun_out/bench_replications_b1.log
timeout 600 python bench.py --process-group --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pg.log 2>&1; tail -1 gpurun_out/bench_pg.log
timeout 600 python bench.py --process-group --resampler spacings --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pg_spacings.log 2>&1; tail -1 gpurun_out/bench_pg_spacings.log
PF_CHAIN_DEBUG=1 timeout 300 python scripts/prof_run.py 24 300 > gpurun_out/chain.log 2>&1
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_steady.csv python scripts/prof_run.py 24 210 > gpurun_out/ncu_launch_steady.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --t 20 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"step_kernel" -c 1 -o gpurun_out/step_full python scripts/prof_run.py 24 205 > gpurun_out/ncu_full.log 2>&1
python scripts/ncu_summary.py gpurun_out/step_full.ncu-rep > gpurun_out/step_full_summary.txt 2>&1
echo done
