#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity_large.py tests/test_gpu_batch.py tests/test_gpu_shards.py -q -x -m gpu 2>&1 | tail -3
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
R=$PWD
for d in $R $R/_abhead $R $R/_abhead; do
  echo "== $d"
  (cd $d && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $R/gpurun_out/ab24.log 2>&1); pj 2^24 < gpurun_out/ab24.log
  (cd $d && timeout 300 python bench.py --steps 3 --warmup 3 --n 1048576 --no-cpu-baseline > $R/gpurun_out/ab20.log 2>&1); pj 2^20 < gpurun_out/ab20.log
done
timeout 300 python scripts/bench_replications.py --reps 128 --batch 32 | tail -1 | cut -c1-120
