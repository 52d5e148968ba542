b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s e2e", round(d["e2e"]["value"]/1e9,3), "ms/run", round(d["ms_per_step"],2), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4))' 2>&1 | tail -1; }
for n in 1048576 2097152; do
echo "$n default: $(b --n $n)"
echo "$n FD: $(PF_FUSED_DRAWS=1 b --n $n)"
done
echo "4194304 noFD: $(PF_FUSED_DRAWS=0 b --n 4194304)"
echo "4194304 FD: $(b --n 4194304)"
