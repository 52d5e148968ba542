#!/bin/bash
# A/B of an environment switch on the 1-GPU bench: gpu_ab_env.sh VAR "v1 v2 ..." [steps]
for v in $2; do
  for rep in 1 2; do
    echo "$1=$v rep $rep: $(env $1=$v timeout 300 python bench.py --steps ${3:-3} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s  ms/step", round(d["ms_per_step"],1), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4))')"
  done
done
