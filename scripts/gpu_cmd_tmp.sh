./scripts/micro/div_check
LIBS="default" bash scripts/gpu_ab2.sh
echo "chain: $(PF_CHAIN_DEBUG=1 timeout 300 python scripts/prof_run.py 24 300 2>&1 | grep chain | tr '\n' ' ')"
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_parity_large.py tests/test_gpu_shards.py tests/test_gpu_engine.py tests/test_gpu_resamplers.py 2>&1 | tail -2
