#!/bin/bash
# A/B of variant library builds on the 1-GPU bench: gpu_ab_lib.sh "default build_variants/x.so ..." [steps]
for lib in $1; do
  for rep in 1 2; do
    if [ "$lib" = default ]; then unset PARSMC_B200_LIB; else export PARSMC_B200_LIB=$PWD/$lib; fi
    echo "$lib rep $rep: $(timeout 300 python bench.py --steps ${2:-3} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s  ms/run", round(d["ms_per_step"],1), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4))')"
  done
done
