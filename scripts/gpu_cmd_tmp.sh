#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x -m gpu 2>&1 | tail -2
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
R=$PWD
for d in $R $R/_abhead $R $R/_abhead $R $R/_abhead; do
  echo "== $d"
  (cd $d && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $R/gpurun_out/ab24.log 2>&1); pj 2^24 < gpurun_out/ab24.log
done
