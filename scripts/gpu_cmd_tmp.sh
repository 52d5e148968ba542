#!/bin/bash
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
for f in 1 0 1 0; do
  export PF_FUSED_DRAWS=$f; echo "== fd $f"
  timeout 300 python bench.py --steps 3 --warmup 3 --n 1048576 --no-cpu-baseline > gpurun_out/ab.log 2>&1; pj 2^20 < gpurun_out/ab.log
done
unset PF_FUSED_DRAWS
for b in 32; do for f in 1 0; do PF_FUSED_DRAWS=$f timeout 300 python scripts/bench_replications.py --reps 128 --batch $b | tail -1 | cut -c1-110; done; done
