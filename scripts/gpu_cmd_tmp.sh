b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s e2e", round(d["e2e"]["value"]/1e9,3), "ms/run", round(d["ms_per_step"],2), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4))' 2>&1 | tail -1; }
for r in 1 2; do
echo "default 2^24: $(b)"
echo "fuse_cls 2^24: $(PF_FUSE_CLASSIFY=1 b)"
done
echo "default 2^20: $(b --n 1048576)"
echo "fuse_cls 2^20: $(PF_FUSE_CLASSIFY=1 b --n 1048576)"
echo "fuse_cls 2^22: $(PF_FUSE_CLASSIFY=1 b --n 4194304)"
echo "default 2^22: $(b --n 4194304)"
PF_FUSE_CLASSIFY=1 timeout 1500 python -m pytest -q -x tests/test_gpu_parity_large.py tests/test_gpu_engine.py 2>&1 | tail -2
