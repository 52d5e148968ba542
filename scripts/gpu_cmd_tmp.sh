#!/bin/bash
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
for n in 1048576 2097152 4194304 16777216; do
  timeout 300 python bench.py --steps 3 --warmup 3 --n $n --no-cpu-baseline > gpurun_out/ab.log 2>&1; pj $n < gpurun_out/ab.log
done
timeout 300 python scripts/bench_replications.py --reps 128 --batch 32 | tail -1 | cut -c1-120
