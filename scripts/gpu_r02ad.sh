# round 2: threshold tier tests + two-phase sharded lookup (gloo, 2 ranks on one GPU) + full lookup tests
export CUDA_MODULE_LOADING=EAGER
timeout -s KILL 1500 python -m pytest tests/test_gpu_lookup_i8.py tests/test_gpu_sharded_capi.py tests/test_gpu_lookup.py -q -x -s > gpurun_out/r02ad_tests.log 2>&1; echo "tests rc=$?"; grep -E "clustered vs plain|passed|failed|Error" gpurun_out/r02ad_tests.log | tail -8
