b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s e2e", round(d["e2e"]["value"]/1e9,3), "ms/run", round(d["ms_per_step"],2), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4), "launches", d["gpu_launches"])'; }
echo "2^24: $(b)"
echo "2^23: $(b --n 8388608)"
echo "2^23 fused: $(PF_FUSED_RESOLVE_LOG2N=23 b --n 8388608)"
echo "2^20: $(b --n 1048576 --t 1000)"
echo "2^21: $(b --n 2097152 --t 1000)"
timeout 1500 python -m pytest -q tests/test_gpu_engine.py tests/test_gpu_parity_large.py 2>&1 | tail -1
PF_FUSED_RESOLVE_LOG2N=30 timeout 1500 python -m pytest -q tests/test_gpu_engine.py tests/test_gpu_parity_large.py 2>&1 | tail -1
PF_FUSED_RESOLVE_LOG2N=0 timeout 1500 python -m pytest -q tests/test_gpu_engine.py tests/test_gpu_parity_large.py 2>&1 | tail -1
