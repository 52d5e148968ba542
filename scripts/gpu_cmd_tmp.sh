#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity_large.py tests/test_gpu_batch.py tests/test_gpu_spacings.py tests/test_gpu_kernels.py -q -x -m gpu 2>&1 | tail -2
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
for i in 1 2; do
  for n in 1048576 4194304 16777216; do
  timeout 300 python bench.py --steps 3 --warmup 3 --n $n --no-cpu-baseline > gpurun_out/ab.log 2>&1; pj $n < gpurun_out/ab.log
  done
done
timeout 300 python scripts/bench_replications.py --reps 128 | tail -1 | cut -c1-110
