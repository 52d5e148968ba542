#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity_large.py tests/test_gpu_batch.py tests/test_gpu_spacings.py -q -x -m gpu 2>&1 | tail -3
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
for c in 1 0 1 0; do
  export PF_COND_FALLBACK=$c; echo "== cond $c"
  for n in 1048576 4194304; do
  timeout 300 python bench.py --steps 3 --warmup 3 --n $n --no-cpu-baseline > gpurun_out/ab.log 2>&1; pj $n < gpurun_out/ab.log; tail -2 gpurun_out/ab.log | grep -i error
  done
done
