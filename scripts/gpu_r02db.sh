# round 2: cross-rank pilot keys in the sharded int8 lookup — sharded C-ABI tests (2 ranks, host transport; NCCL world 1) + lookup tests
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1800 python -m pytest tests/test_gpu_sharded_capi.py tests/test_gpu_lookup_i8.py tests/test_gpu_lookup.py -q -x > gpurun_out/r02db_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02db_tests.log
timeout -s KILL 300 python scripts/time_lookup.py 1000000 32 768 2>&1 | tail -1
