b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s e2e", round(d["e2e"]["value"]/1e9,3), "ms/run", round(d["ms_per_step"],2), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4))' 2>&1 | tail -1; }
for r in 1 2; do
echo "windows 2^24: $(b)"
echo "no windows 2^24: $(PF_GROUP_WINDOWS=0 b)"
done
echo "windows spacings: $(b --resampler spacings)"
echo "windows 2^22: $(b --n 4194304)"
timeout 1500 python -m pytest -q -x tests/test_gpu_parity_large.py tests/test_gpu_engine.py tests/test_gpu_spacings.py tests/test_gpu_kernels.py 2>&1 | tail -2
