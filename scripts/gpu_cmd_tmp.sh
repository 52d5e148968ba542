#!/bin/bash
mkdir -p gpurun_out
for b in 1 16 32 64; do timeout 300 python scripts/bench_replications.py --reps 128 --batch $b | tail -1 | tee -a gpurun_out/bench_replications_batch.jsonl; done
