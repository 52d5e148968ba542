b() { timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s e2e", round(d["e2e"]["value"]/1e9,3), "ms/run", round(d["ms_per_step"],2), "step_kernel_ms", round(d["roofline"].get("step_kernel_ms",0),4))' 2>&1 | tail -1; }
echo "2^24: $(b)"
echo "2^20: $(b --n 1048576 --t 1000)"
echo "2^22: $(b --n 4194304 --t 1000)"
echo "reps: $(timeout 600 python scripts/bench_replications.py --reps 64 --concurrency 1 2>&1 | tail -1)"
timeout 1800 python -m pytest -q -x tests -m gpu 2>&1 | tail -3
