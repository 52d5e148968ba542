#!/bin/bash
nproc
timeout 600 python scripts/bench_store.py 20 30 | tee gpurun_out/bench_store.json
timeout 600 python scripts/bench_store.py 22 10
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -m gpu 2>&1 | tail -1
