# the bounds-checked build (ISR_ASSERT traps) through the GPU parity / feature / exchange / strip tests
ISING_SR_LIB=build_variants/checked.so timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_exchange.py tests/test_gpu_shards.py -q -x > gpurun_out/checked_tests.log 2>&1
tail -3 gpurun_out/checked_tests.log
