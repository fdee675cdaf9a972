# round 2: sharded C-ABI tests incl. int8 two-phase and a skewed shard
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_sharded_capi.py tests/test_gpu_store.py -q -x > gpurun_out/r02ae_tests.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed|Error" gpurun_out/r02ae_tests.log | tail -8
