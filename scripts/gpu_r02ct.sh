# round 2: select_keyframes with the item's Gram staged in shared memory; timing + codec tests
export CUDA_MODULE_LOADING=EAGER
FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | sed -n 2,3p
FC_SELECT_STAGED=0 FC_COMPRESS_SPLIT=1 timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | sed -n 2,3p
timeout -s KILL 300 python scripts/time_codec.py 256 2>&1 | sed -n 2,3p
timeout -s KILL 1500 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py tests/test_engine.py tests/test_capi.py -q -x -m gpu > gpurun_out/r02ct_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02ct_tests.log
