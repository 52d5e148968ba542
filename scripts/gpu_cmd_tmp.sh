#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -m gpu 2>&1 | tail -15
for b in 1 4 16 32; do echo "== batch $b"; timeout 300 python scripts/bench_replications.py --reps 64 --batch $b 2>&1 | tail -1; done
