mkdir -p gpurun_out
b() { timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1; }
b > gpurun_out/m_2e24.json; b --resampler spacings > gpurun_out/m_2e24_sp.json
b --n 1048576 --t 1000 > gpurun_out/m_2e20.json; b --n 1048576 --t 100 > gpurun_out/m_2e20_T100.json
b --n 2097152 --t 1000 > gpurun_out/m_2e21.json; b --n 4194304 --t 1000 > gpurun_out/m_2e22.json; b --n 8388608 --t 1000 > gpurun_out/m_2e23.json
b --n 134217728 --t 100 --steps 2 --warmup 3 > gpurun_out/m_2e27_T100.json
b --n 134217728 --t 100 --steps 2 --warmup 3 --resampler spacings > gpurun_out/m_2e27_T100_sp.json
timeout 900 python bench.py --shards 8 --n 134217728 --t 100 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/m_2e27_8shards.json
timeout 900 python bench.py --shards 8 --n 134217728 --t 100 --steps 2 --warmup 3 --no-cpu-baseline --resampler spacings 2>/dev/null | tail -1 > gpurun_out/m_2e27_8shards_sp.json
timeout 600 python bench.py --process-group --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/m_pg.json
timeout 600 python bench.py --process-group --resampler spacings --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/m_pg_sp.json
timeout 600 python scripts/bench_replications.py --reps 64 --concurrency 1 2>/dev/null | tail -1 > gpurun_out/m_reps.json
for f in gpurun_out/m_*.json; do echo "$f: $(python -c "import json; d=json.load(open('$f')); print(round(d['value']/1e9,3), 'G/s', 'e2e', round(d.get('e2e',{}).get('value',0)/1e9,3) if isinstance(d.get('e2e'),dict) else '', 'ms', round(d.get('ms_per_step', d.get('ms_per_replication',0)),2))" 2>&1 | tail -1)"; done
