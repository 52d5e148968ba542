#!/bin/bash
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
for w in 1 0 1 0 1 0; do
  if [ $w = 1 ]; then export PF_CLS_LATE=1; else unset PF_CLS_LATE; fi; echo "== late $w"
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1; pj 2^24 < gpurun_out/ab.log
done
