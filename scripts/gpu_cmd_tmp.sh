LIBS="default build_variants/ilf.so default build_variants/ilf.so" bash scripts/gpu_ab2.sh 2>&1 | grep -v "^done"
export PARSMC_B200_LIB=$PWD/build_variants/ilf.so
echo "ilf chain: $(PF_CHAIN_DEBUG=1 timeout 300 python scripts/prof_run.py 24 300 2>&1 | grep chain | tr '\n' ' ')"
timeout 1500 python -m pytest -q -x tests/test_gpu_parity_large.py tests/test_gpu_engine.py tests/test_gpu_kernels.py tests/test_gpu_shards.py 2>&1 | tail -2
