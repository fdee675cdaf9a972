# round 2: fixed-threshold int8 tier for near-tied clusters — tests (+ the 1M clustered timing test)
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup_i8.py tests/test_gpu_lookup.py -q -x -s > gpurun_out/r02ab_tests.log 2>&1; echo "tests rc=$?"; grep -E "clustered vs plain|passed|failed|Error" gpurun_out/r02ab_tests.log | tail -8
