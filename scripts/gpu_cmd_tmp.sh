b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s e2e", round(d["e2e"]["value"]/1e9,3), "ms/run", round(d["ms_per_step"],2), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4), "frac", round(d["roofline"]["frac"],4))' 2>&1 | tail -1; }
echo "2^24: $(b)"
echo "2^24: $(b)"
echo "2^22: $(b --n 4194304 --t 1000)"
echo "2^23: $(b --n 8388608 --t 1000)"
echo "2^24 spacings: $(b --resampler spacings)"
timeout 1800 python -m pytest -q tests -m gpu 2>&1 | tail -2
PF_FUSED_DRAWS=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python scripts/prof_run.py 16 3 > gpurun_out/memcheck_fd768.txt 2>&1; grep "ERROR SUMMARY" gpurun_out/memcheck_fd768.txt
PF_FUSED_DRAWS=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python scripts/prof_run.py 16 3 > gpurun_out/racecheck_fd768.txt 2>&1; grep "RACECHECK SUMMARY" gpurun_out/racecheck_fd768.txt
PF_PROFILE_FROM_STEP=200 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"step_kernel" -c 1 -o gpurun_out/step_full python scripts/prof_run.py 24 205 > gpurun_out/ncu_full.log 2>&1
python scripts/ncu_summary.py gpurun_out/step_full.ncu-rep
