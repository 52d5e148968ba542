#!/bin/bash
pj() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$1', round(d['value']/1e9,3), d.get('roofline',{}).get('step_kernel_ms'))
"; }
for w in 2 0 2 0 2 0; do
  export PF_WBUF=$w; echo "== wbuf $w"
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1; pj 2^24 < gpurun_out/ab.log
done
PF_WBUF=2 timeout 600 python -m pytest tests/test_gpu_parity_large.py -q -x -m gpu 2>&1 | tail -1
