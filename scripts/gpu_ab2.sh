#!/bin/bash
# A/B of variant builds (bench only) + memcheck/racecheck of a variant.
mkdir -p gpurun_out
for lib in $LIBS; do
  if [ "$lib" = default ]; then unset PARSMC_B200_LIB; else export PARSMC_B200_LIB=$PWD/$lib; fi
  for rep in 1 2; do
    echo "$lib rep $rep: $(timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s  ms/run", round(d["ms_per_step"],1), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4))')"
  done
done
unset PARSMC_B200_LIB
for lib in $SANLIBS; do
  n=$(basename $lib .so)
  PARSMC_B200_LIB=$PWD/$lib PF_FUSED_DRAWS=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python scripts/prof_run.py 16 3 > gpurun_out/memcheck_$n.txt 2>&1; echo "memcheck $n: $(grep 'ERROR SUMMARY' gpurun_out/memcheck_$n.txt)"
  PARSMC_B200_LIB=$PWD/$lib PF_FUSED_DRAWS=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python scripts/prof_run.py 16 3 > gpurun_out/racecheck_$n.txt 2>&1; echo "racecheck $n: $(grep 'ERROR SUMMARY' gpurun_out/racecheck_$n.txt)"
done
echo done
