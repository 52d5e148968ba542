#!/bin/bash
# Full-size oracle-mode validation: configs[1] (N=2^20, T=1000) and the fused-draws path (N=2^22, T=100).
mkdir -p gpurun_out
free -g > gpurun_out/free.txt
timeout 2400 python scripts/validate_oracle_config1.py 20 1000 > gpurun_out/validate_2e20_T1000.json 2> gpurun_out/validate_2e20.err; tail -1 gpurun_out/validate_2e20_T1000.json
timeout 1800 python scripts/validate_oracle_config1.py 22 100 > gpurun_out/validate_2e22_T100.json 2> gpurun_out/validate_2e22.err; tail -1 gpurun_out/validate_2e22_T100.json
