#!/bin/bash
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
for m in 0 8192 16384 0 8192 16384; do
  export PF_FB_MIN=$m; echo "== fbmin $m"
  for n in 1048576 4194304; do
  timeout 300 python bench.py --steps 3 --warmup 3 --n $n --no-cpu-baseline > gpurun_out/ab.log 2>&1; pj $n < gpurun_out/ab.log
  done
done
