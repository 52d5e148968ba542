#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -m gpu 2>&1 | tail -4
compute-sanitizer --tool memcheck timeout 600 python -m pytest tests/test_gpu_batch.py -q -x -m gpu -k "pl_matches and 4096 or known_parameters or engine_reuse" > gpurun_out/memcheck_batch.txt 2>&1; tail -3 gpurun_out/memcheck_batch.txt
compute-sanitizer --tool racecheck timeout 600 python -m pytest tests/test_gpu_batch.py -q -x -m gpu -k "known_parameters" > gpurun_out/racecheck_batch.txt 2>&1; tail -3 gpurun_out/racecheck_batch.txt
for r in 32; do timeout 300 python scripts/bench_replications.py --reps 128 --batch $r | tail -1; done
