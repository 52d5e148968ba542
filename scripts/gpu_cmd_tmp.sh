#!/bin/bash
timeout 600 python scripts/bench_store.py 20 30 | tee gpurun_out/bench_store.json
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_resamplers.py tests/test_gpu_harness.py tests/test_gpu_spacings.py -q -x -m gpu 2>&1 | tail -2
